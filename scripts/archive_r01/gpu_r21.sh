mkdir -p gpurun_out
: > gpurun_out/fused_cfg.log
for cfg in "4,6,128" "4,12,128" "4,12,256" "4,9,256" "4,6,256"; do
echo "== CQ_WAVE_FUSED_CFG=$cfg" >> gpurun_out/fused_cfg.log
CQ_WAVE_FUSED_CFG=$cfg timeout 600 python scripts/fused_check.py 2>&1 | grep -v bit-identical >> gpurun_out/fused_cfg.log; echo "exit=$?" >> gpurun_out/fused_cfg.log
done
