mkdir -p gpurun_out
: > gpurun_out/fused_w12.log
for cfg in "4,6,256" "4,6,128"; do
echo "== CQ_WAVE_FUSED_CFG=$cfg (KL8: 12 warps/block)" >> gpurun_out/fused_w12.log
CQ_WAVE_FUSED_CFG=$cfg timeout 600 python scripts/fused_check.py 2>&1 | grep -E "KL=8 96|ALL|MISMATCH|FAIL" >> gpurun_out/fused_w12.log
done
