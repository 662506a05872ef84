# round 2, call 13: branch-free ring loop (predicated cp.async / stores) vs default: parity + interleaved timing + ncu
mkdir -p gpurun_out/r02
PARITY_CFGS="4,56;4,59" timeout 1200 python scripts/r02/fused_ab.py > gpurun_out/r02/g16_fused_ab.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g16_fused_ab.log
M=gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_active.avg,sm__cycles_elapsed.avg,dram__bytes_read.sum,dram__bytes_write.sum
for cfg in "4,6" "4,56" "4,59"; do
  CQ_WAVE_FUSED_CFG=$cfg timeout 300 ncu --metrics $M --clock-control none -k regex:wave5_fused -s 2 -c 1 --csv python scripts/r02/prof_one.py 8 > gpurun_out/r02/g16_ncu_$cfg.csv 2>&1
done
