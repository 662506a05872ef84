mkdir -p gpurun_out
timeout 600 python scripts/fused_seg_ab.py > gpurun_out/fused_seg_ab.log 2>&1; echo "exit=$?" >> gpurun_out/fused_seg_ab.log
timeout 1500 python -m pytest tests/ -q -m gpu -x -k "fused or wave or smoke" > gpurun_out/gpu_tests_seg.log 2>&1; echo "exit=$?" >> gpurun_out/gpu_tests_seg.log
timeout 900 python bench.py --no-cpu --no-energy > gpurun_out/bench_r41.log 2>&1; echo "exit=$?" >> gpurun_out/bench_r41.log
