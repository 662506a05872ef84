# round 2, call 41 (1 GPU): bench at HEAD (e2e floor measured on the simulation's own transfer pattern)
mkdir -p gpurun_out/r02
timeout 900 python bench.py > gpurun_out/r02/g41_bench_n1.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g41_bench_n1.log
