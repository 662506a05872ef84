mkdir -p gpurun_out/r02
timeout 600 python scripts/r02/nbody_ab.py > gpurun_out/r02/g28_nbody_ab.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g28_nbody_ab.log
