mkdir -p gpurun_out
timeout 1500 python -m pytest tests/ -q -m gpu -x -k "fused or wave or smoke or batch" > gpurun_out/gpu_tests_r56.log 2>&1; echo "exit=$?" >> gpurun_out/gpu_tests_r56.log
timeout 600 python scripts/fused_check.py > gpurun_out/fused_check_r56.log 2>&1; echo "exit=$?" >> gpurun_out/fused_check_r56.log
for i in 1 2; do
timeout 900 python bench.py --no-cpu --no-energy --no-kernels > gpurun_out/bench_r56_$i.log 2>&1; echo "exit=$?" >> gpurun_out/bench_r56_$i.log
done
timeout 300 python scripts/fused_prof.py 8 fast > gpurun_out/fused_prof_r56.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:wave5_fused -s 1 -c 1 -o gpurun_out/fused8fast_r56 python scripts/fused_prof.py 8 fast > gpurun_out/ncu_fused8fast_r56.log 2>&1
