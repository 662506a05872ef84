mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu > gpurun_out/gpu_tests.log 2>&1
echo "exit=$?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "exit=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py --size 2048 --wave-steps 20 --steps 3 --warmup 3 --nbody 16384 --sgemm 1024 --no-cpu > gpurun_out/bench_small.log 2>&1
echo "exit=$?" >> gpurun_out/bench_small.log
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1
echo "exit=$?" >> gpurun_out/bench_full.log
