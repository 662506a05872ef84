mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "graph or saxpy" > gpurun_out/gpu_tests_r12.log 2>&1; echo "exit=$?" >> gpurun_out/gpu_tests_r12.log
timeout 900 python bench.py > gpurun_out/bench_r12.log 2>&1; echo "exit=$?" >> gpurun_out/bench_r12.log
