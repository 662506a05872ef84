mkdir -p gpurun_out
: > gpurun_out/fused_rb.log
for cfg in "4,6,256" "4,6,224" "4,6,192" "4,6,128"; do
echo "== CQ_WAVE_FUSED_CFG=$cfg" >> gpurun_out/fused_rb.log
CQ_WAVE_FUSED_CFG=$cfg timeout 600 python scripts/fused_check.py 2>&1 | grep -E "KL=8 96|ALL|MISMATCH|FAIL|Error" >> gpurun_out/fused_rb.log
done
