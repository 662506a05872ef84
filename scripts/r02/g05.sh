# round 2, call 5: interleaved timing sweep of the fused pass; bench with the new defaults
mkdir -p gpurun_out/r02
SKIP_PARITY=1 timeout 900 python scripts/r02/fused_ab.py > gpurun_out/r02/g05_fused_ab.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g05_fused_ab.log
timeout 600 python bench.py --no-cpu --no-energy --no-kernels > gpurun_out/r02/g05_bench.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g05_bench.log
