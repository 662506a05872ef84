# round 2, call 20: round-end rehearsal -- GPU tests, smoke, bench, reference arm, launch list
mkdir -p gpurun_out/r02
timeout 1800 python -m pytest tests/ -q -m gpu -x > gpurun_out/r02/g20_gpu_tests.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g20_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02/g20_smoke.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g20_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02/g20_bench.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g20_bench.log
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02/g20_bench_ref.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g20_bench_ref.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02/g20_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-energy --no-kernels > gpurun_out/r02/g20_ncu.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g20_ncu.log
