# round 2, call 61 (1 GPU): which libcq call makes a session close slow
mkdir -p gpurun_out/r02
timeout 600 python scripts/r02/e2e_batches.py > gpurun_out/r02/g61_e2e_batches.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g61_e2e_batches.log
