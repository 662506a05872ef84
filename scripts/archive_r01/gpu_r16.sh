mkdir -p gpurun_out
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu --no-energy > gpurun_out/bench_plain_r16.log 2>&1; echo "exit=$?" >> gpurun_out/bench_plain_r16.log
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r16.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-energy > gpurun_out/ncu_list_r16.log 2>&1; echo "exit=$?" >> gpurun_out/ncu_list_r16.log
