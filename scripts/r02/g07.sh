# round 2, call 7: full GPU test suite, smoke, bench (all legs), reference arm
mkdir -p gpurun_out/r02
timeout 1800 python -m pytest tests/ -q -m gpu -x > gpurun_out/r02/g07_gpu_tests.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g07_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02/g07_smoke.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g07_smoke.log
timeout 900 python bench.py > gpurun_out/r02/g07_bench.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g07_bench.log
timeout 900 python bench.py --impl reference > gpurun_out/r02/g07_bench_ref.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g07_bench_ref.log
