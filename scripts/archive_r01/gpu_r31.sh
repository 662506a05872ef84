mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "run_batch or fused or graph" > gpurun_out/gpu_tests_r31.log 2>&1; echo "exit=$?" >> gpurun_out/gpu_tests_r31.log
timeout 900 python bench.py --no-kernels > gpurun_out/bench_r31.log 2>&1; echo "exit=$?" >> gpurun_out/bench_r31.log
