# round-end rehearsal: the driver's GPU tiers in order (tests, smoke, bench, reference arm)
mkdir -p gpurun_out
rm -f gpurun_out/final_*.log
timeout 1500 python -m pytest tests/ -q -m gpu -x > gpurun_out/final_gpu_tests.log 2>&1; echo "exit=$?" >> gpurun_out/final_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "exit=$?" >> gpurun_out/final_smoke.log
timeout 900 python bench.py > gpurun_out/final_bench.log 2>&1; echo "exit=$?" >> gpurun_out/final_bench.log
timeout 600 python bench.py --impl reference > gpurun_out/final_bench_ref.log 2>&1; echo "exit=$?" >> gpurun_out/final_bench_ref.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-energy > gpurun_out/final_ncu.log 2>&1; echo "exit=$?" >> gpurun_out/final_ncu.log
