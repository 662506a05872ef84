mkdir -p gpurun_out
timeout 600 python examples/quickstart.py > gpurun_out/quickstart.log 2>&1; echo "exit=$?" >> gpurun_out/quickstart.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "huge" >> gpurun_out/quickstart.log 2>&1; echo "exit=$?" >> gpurun_out/quickstart.log
