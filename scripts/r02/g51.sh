# round 2, call 51 (1 GPU): e2e pipeline depth sweep on another box
mkdir -p gpurun_out/r02
timeout 600 python scripts/r02/e2e_depth.py > gpurun_out/r02/g51_e2e_depth.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g51_e2e_depth.log
