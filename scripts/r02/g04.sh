# round 2, call 4: one-warp blocks, strip-minor ranges: rows-per-warp and ring-depth sweep; ncu of the best
mkdir -p gpurun_out/r02
timeout 900 python scripts/r02/fused_ab.py > gpurun_out/r02/g04_fused_ab.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g04_fused_ab.log
for cfg in "4,9" "4,12"; do
  CQ_WAVE_FUSED_CFG=$cfg SKIP_PARITY=1 timeout 600 python scripts/r02/fused_ab.py >> gpurun_out/r02/g04_fused_ab.log 2>&1
done
M=gpu__time_duration.sum,smsp__warps_launched.sum,smsp__warps_launched.min,smsp__warps_launched.max,smsp__inst_executed.sum,smsp__inst_executed.min,smsp__inst_executed.max,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__cycles_active.avg,sm__cycles_elapsed.avg,dram__bytes_read.sum,dram__bytes_write.sum,smsp__cycles_active.min,smsp__cycles_active.max,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct
for rows in 224 1366; do
  CQ_FUSED_WPB=1 CQ_FUSED_MAP=2 CQ_FUSED_ROWS=$rows timeout 300 ncu --metrics $M --clock-control none -k regex:wave5_fused -s 2 -c 1 --csv python scripts/r02/prof_one.py 8 > gpurun_out/r02/g04_ncu_map2_rows$rows.csv 2>&1
done
