mkdir -p gpurun_out
timeout 600 python scripts/fused_seg_sweep.py > gpurun_out/fused_seg_sweep2.log 2>&1; echo "exit=$?" >> gpurun_out/fused_seg_sweep2.log
timeout 1500 python -m pytest tests/ -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1; echo "exit=$?" >> gpurun_out/gpu_tests.log
timeout 900 python bench.py --no-cpu --no-energy > gpurun_out/bench_r43.log 2>&1; echo "exit=$?" >> gpurun_out/bench_r43.log
