mkdir -p gpurun_out
timeout 1500 python -m pytest tests/ -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1; echo "exit=$?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "exit=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_r34.log 2>&1; echo "exit=$?" >> gpurun_out/bench_r34.log
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r34.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-energy > gpurun_out/ncu_list_r34.log 2>&1; echo "exit=$?" >> gpurun_out/ncu_list_r34.log
