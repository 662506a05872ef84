# round 2, call 2: balanced one-warp-block fused pass -- parity + A/B timings, wave GPU tests, bench line
mkdir -p gpurun_out/r02
timeout 900 python scripts/r02/fused_ab.py > gpurun_out/r02/g02_fused_ab.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g02_fused_ab.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu > gpurun_out/r02/g02_gpu_parity.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g02_gpu_parity.log
timeout 600 python bench.py --no-cpu --no-energy --no-kernels > gpurun_out/r02/g02_bench.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g02_bench.log
