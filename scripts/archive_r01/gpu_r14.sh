mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sgemm_3xtf32_2sm -c 1 -o gpurun_out/tf32_2sm_full python scripts/tf32_once.py 8192 > gpurun_out/ncu_tf32_2sm.log 2>&1
echo "exit=$?" >> gpurun_out/ncu_tf32_2sm.log
timeout 900 python bench.py > gpurun_out/bench_r14.log 2>&1; echo "exit=$?" >> gpurun_out/bench_r14.log
