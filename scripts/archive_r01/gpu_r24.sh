mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "fused or wave" > gpurun_out/gpu_tests_r24.log 2>&1; echo "exit=$?" >> gpurun_out/gpu_tests_r24.log
timeout 900 python bench.py > gpurun_out/bench_r24.log 2>&1; echo "exit=$?" >> gpurun_out/bench_r24.log
