mkdir -p gpurun_out
timeout 1200 python -m pytest tests/ -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo "exit=$?" >> gpurun_out/gpu_tests.log
timeout 900 python bench.py --no-cpu --sgemm-variants 3xtf32,ffma > gpurun_out/bench_full.log 2>&1; echo "exit=$?" >> gpurun_out/bench_full.log
timeout 300 python bench.py --no-cpu --no-energy --size 2048 --wave-steps 4 --steps 2 --warmup 3 --sgemm 1024 --sgemm-variants 3xtf32 > gpurun_out/plain_small.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:nbody_kick -s 1 -c 1 -o gpurun_out/nbody_full python bench.py --no-cpu --no-energy --size 2048 --wave-steps 4 --steps 2 --warmup 3 --sgemm 1024 --sgemm-variants 3xtf32 > gpurun_out/ncu_nbody.log 2>&1
echo "exit=$?" >> gpurun_out/ncu_nbody.log
