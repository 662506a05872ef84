# round 2, call 3: fused pass layouts A/B (one-warp vs 12-warp blocks, range maps), SMSP balance metrics
mkdir -p gpurun_out/r02
timeout 1200 python scripts/r02/fused_ab.py > gpurun_out/r02/g03_fused_ab.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g03_fused_ab.log
M=gpu__time_duration.sum,smsp__warps_launched.sum,smsp__warps_launched.min,smsp__warps_launched.max,smsp__inst_executed.sum,smsp__inst_executed.min,smsp__inst_executed.max,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__cycles_active.avg,sm__cycles_elapsed.avg,dram__bytes_read.sum,dram__bytes_write.sum,smsp__cycles_active.min,smsp__cycles_active.max
for cfg in "1 0 x" "12 2 224" "12 0 x"; do
  set -- $cfg
  if [ "$3" = x ]; then unset CQ_FUSED_ROWS; else export CQ_FUSED_ROWS=$3; fi
  CQ_FUSED_WPB=$1 CQ_FUSED_MAP=$2 timeout 300 ncu --metrics $M --clock-control none -k regex:wave5_fused -s 2 -c 1 --csv python scripts/r02/prof_one.py 8 > gpurun_out/r02/g03_ncu_wpb$1_map$2_rows$3.csv 2>&1
done
