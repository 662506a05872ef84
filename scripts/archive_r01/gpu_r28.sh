mkdir -p gpurun_out
: > gpurun_out/fused_r28.log
timeout 600 python scripts/fused_check.py 2>&1 | grep -E "96 steps|ALL|MISMATCH|FAIL" >> gpurun_out/fused_r28.log
