mkdir -p gpurun_out/r02
timeout 900 python scripts/r02/e2e_diag.py > gpurun_out/r02/g12_e2e_diag.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g12_e2e_diag.log
