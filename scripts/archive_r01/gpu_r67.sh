mkdir -p gpurun_out
rm -f gpurun_out/r67_*
timeout 1500 python -m pytest tests/ -q -m gpu -x > gpurun_out/r67_gpu_tests.log 2>&1; echo "exit=$?" >> gpurun_out/r67_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r67_smoke.log 2>&1; echo "exit=$?" >> gpurun_out/r67_smoke.log
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > gpurun_out/r67_bench.log 2>&1; echo "exit=$?" >> gpurun_out/r67_bench.log
CUDA_VISIBLE_DEVICES=0 timeout 300 python scripts/fused_prof.py 8 fast > gpurun_out/r67_prof.log 2>&1 && CUDA_VISIBLE_DEVICES=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:wave5_fused -s 1 -c 1 -o gpurun_out/r67_fused8fast python scripts/fused_prof.py 8 fast > gpurun_out/r67_ncu.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 300 python scripts/fused_prof.py 4 > gpurun_out/r67_prof4.log 2>&1 && CUDA_VISIBLE_DEVICES=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:wave5_fused -s 1 -c 1 -o gpurun_out/r67_fused4 python scripts/fused_prof.py 4 > gpurun_out/r67_ncu4.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu --no-energy --no-kernels > gpurun_out/r67_small.log 2>&1 && CUDA_VISIBLE_DEVICES=0 timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r67_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-energy --no-kernels > gpurun_out/r67_ncu_list.log 2>&1
