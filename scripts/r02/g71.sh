# round 2, call 71 (1 GPU): re-tune of the KL=8 pass after the FFMA2(c, lap, +0) form -- rows per piece and ring depth
mkdir -p gpurun_out/r02
for r in 1 2; do
for rows in 160 224 288 456; do
  CQ_FUSED_ROWS=$rows timeout 300 python scripts/r02/lib_ab.py 2>&1 | sed "s/^/rows=$rows /" >> gpurun_out/r02/g71_tune.log
done
for cfg in 4,9 4,12; do
  CQ_WAVE_FUSED_CFG=$cfg timeout 300 python scripts/r02/lib_ab.py 2>&1 | sed "s/^/cfg=$cfg /" >> gpurun_out/r02/g71_tune.log
done
done
echo "exit=$?" >> gpurun_out/r02/g71_tune.log
