mkdir -p gpurun_out
timeout 300 python scripts/fused_prof.py 8 fast > gpurun_out/fused_prof_r53.log 2>&1 || exit 1
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu --no-energy --no-kernels > gpurun_out/bench_small_r53.log 2>&1 || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:wave5_fused -s 1 -c 1 -o gpurun_out/fused8fast_r53 python scripts/fused_prof.py 8 fast > gpurun_out/ncu_fused8fast_r53.log 2>&1; echo "exit=$?" >> gpurun_out/ncu_fused8fast_r53.log
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r53.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-energy --no-kernels > gpurun_out/ncu_list_r53.log 2>&1; echo "exit=$?" >> gpurun_out/ncu_list_r53.log
timeout 900 python bench.py > gpurun_out/bench_r53_full.log 2>&1; echo "exit=$?" >> gpurun_out/bench_r53_full.log
