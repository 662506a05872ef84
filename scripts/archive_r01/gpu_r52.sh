mkdir -p gpurun_out
timeout 1500 python -m pytest tests/ -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1; echo "exit=$?" >> gpurun_out/gpu_tests.log
timeout 600 python scripts/fused_check.py > gpurun_out/fused_check_r52.log 2>&1; echo "exit=$?" >> gpurun_out/fused_check_r52.log
timeout 900 python bench.py --no-cpu --no-energy --no-kernels > gpurun_out/bench_r52.log 2>&1; echo "exit=$?" >> gpurun_out/bench_r52.log
CQ_WAVE_FAST=0 timeout 900 python bench.py --no-cpu --no-energy --no-kernels > gpurun_out/bench_r52_nofast.log 2>&1; echo "exit=$?" >> gpurun_out/bench_r52_nofast.log
