mkdir -p gpurun_out/r02
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "fused or wave" > gpurun_out/r02/g24_gpu_tests.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g24_gpu_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-kernels --no-cpu --no-energy > gpurun_out/r02/g24_bench.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g24_bench.log
timeout 300 python scripts/r02/prof_one.py 8 > /dev/null 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:wave5_fused -s 2 -c 1 --csv python scripts/r02/prof_one.py 8 > gpurun_out/r02/g24_ncu.csv 2>&1
