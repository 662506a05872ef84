# round 2, call 59 (1 GPU): e2e batch variance diagnostic
mkdir -p gpurun_out/r02
timeout 600 python scripts/r02/e2e_batches.py > gpurun_out/r02/g59_e2e_batches.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g59_e2e_batches.log
