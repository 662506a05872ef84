# round 2, call 68 (1 GPU): 3xTF32 MN-major B diagnostic
mkdir -p gpurun_out/r02
timeout 300 python scripts/r02/tf32_mnb_diag.py > gpurun_out/r02/g68_diag.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g68_diag.log
