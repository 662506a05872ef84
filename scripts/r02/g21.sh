# round 2, call 21: e2e with the shared pulse uploaded once (device copy for the second buffer); GPU parity of the executor paths
mkdir -p gpurun_out/r02
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_negative_control.py -q -m gpu -x > gpurun_out/r02/g21_gpu_tests.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g21_gpu_tests.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-kernels --no-cpu --no-energy > gpurun_out/r02/g21_bench.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g21_bench.log
