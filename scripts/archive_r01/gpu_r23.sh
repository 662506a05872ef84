mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "fused or wave or graph" > gpurun_out/gpu_tests_r23.log 2>&1; echo "exit=$?" >> gpurun_out/gpu_tests_r23.log
timeout 900 python bench.py --no-cpu > gpurun_out/bench_r23.log 2>&1; echo "exit=$?" >> gpurun_out/bench_r23.log
