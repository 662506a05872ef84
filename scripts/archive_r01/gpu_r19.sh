mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "fused or wave or graph" > gpurun_out/gpu_tests_r19.log 2>&1; echo "exit=$?" >> gpurun_out/gpu_tests_r19.log
timeout 900 python bench.py --no-kernels --no-cpu > gpurun_out/bench_r19.log 2>&1; echo "exit=$?" >> gpurun_out/bench_r19.log
CQ_WAVE_FUSE=0 timeout 900 python bench.py --no-kernels --no-cpu --no-energy > gpurun_out/bench_r19_nofuse.log 2>&1; echo "exit=$?" >> gpurun_out/bench_r19_nofuse.log
