mkdir -p gpurun_out
: > gpurun_out/fused_check.log
for cfg in "4 12" "4 6" "2 12"; do
set -- $cfg
echo "== CQ_WAVE_FUSED_V=$1 D=$2" >> gpurun_out/fused_check.log
CQ_WAVE_FUSED_V=$1 CQ_WAVE_FUSED_D=$2 timeout 600 python scripts/fused_check.py >> gpurun_out/fused_check.log 2>&1; echo "exit=$?" >> gpurun_out/fused_check.log
done
