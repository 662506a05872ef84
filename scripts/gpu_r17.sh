mkdir -p gpurun_out
timeout 600 python scripts/fused_check.py > gpurun_out/fused_check.log 2>&1; echo "exit=$?" >> gpurun_out/fused_check.log
