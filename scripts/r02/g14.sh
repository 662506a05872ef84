mkdir -p gpurun_out/r02
timeout 900 python scripts/r02/e2e_diag2.py > gpurun_out/r02/g14_e2e_diag2.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g14_e2e_diag2.log
