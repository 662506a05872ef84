# round 2, call 62 (1 GPU): e2e batches after caching the flag buffers; bench N=1
mkdir -p gpurun_out/r02
timeout 600 python scripts/r02/e2e_batches.py > gpurun_out/r02/g62_e2e_batches.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g62_e2e_batches.log
timeout 900 python bench.py > gpurun_out/r02/g62_bench_n1.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g62_bench_n1.log
