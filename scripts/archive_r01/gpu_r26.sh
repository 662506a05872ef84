mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "fused or wave or graph" > gpurun_out/gpu_tests_r26.log 2>&1; echo "exit=$?" >> gpurun_out/gpu_tests_r26.log
timeout 300 python scripts/fused_prof.py 8 > gpurun_out/fused_prof8.log 2>&1; echo "exit=$?" >> gpurun_out/fused_prof8.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:wave5_fused -s 1 -c 1 -o gpurun_out/fused8_full python scripts/fused_prof.py 8 >> gpurun_out/fused_prof8.log 2>&1; echo "exit=$?" >> gpurun_out/fused_prof8.log
timeout 900 python bench.py > gpurun_out/bench_r26.log 2>&1; echo "exit=$?" >> gpurun_out/bench_r26.log
