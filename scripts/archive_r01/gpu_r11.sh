mkdir -p gpurun_out
timeout 1200 python -m pytest tests/ -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1; echo "exit=$?" >> gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo "exit=$?" >> gpurun_out/bench_full.log
