mkdir -p gpurun_out
: > gpurun_out/fused_r36.log
timeout 600 python scripts/fused_check.py 2>&1 | grep -E "96 steps|ALL|MISMATCH|FAIL|huge|Error" >> gpurun_out/fused_r36.log
echo "== CQ_WAVE_FUSED_EXACT=1" >> gpurun_out/fused_r36.log
CQ_WAVE_FUSED_EXACT=1 timeout 600 python scripts/fused_check.py 2>&1 | grep -E "KL=. 96 steps|ALL|MISMATCH" >> gpurun_out/fused_r36.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "fused or wave" >> gpurun_out/fused_r36.log 2>&1; echo "exit=$?" >> gpurun_out/fused_r36.log
