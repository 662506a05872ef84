mkdir -p gpurun_out/r02
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "piece_layouts or fused" > gpurun_out/r02/g22_gpu_tests.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g22_gpu_tests.log
