# round 2, call 60 (1 GPU): e2e batch variance -- session close times, gen-2 GC, with and without GC
mkdir -p gpurun_out/r02
timeout 600 python scripts/r02/e2e_batches.py > gpurun_out/r02/g60_e2e_batches.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g60_e2e_batches.log
timeout 600 python scripts/r02/e2e_batches.py nogc > gpurun_out/r02/g60_e2e_batches_nogc.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g60_e2e_batches_nogc.log
