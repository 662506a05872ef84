mkdir -p gpurun_out
timeout 300 python scripts/tf32_check.py > gpurun_out/tf32.log 2>&1; echo "exit=$?" >> gpurun_out/tf32.log
timeout 600 python bench.py --no-kernels --no-cpu --steps 2 --warmup 3 > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --no-kernels --no-cpu --steps 2 --warmup 3 > gpurun_out/ncu_list.log 2>&1
echo "exit=$?" >> gpurun_out/ncu_list.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:wave5_rows -s 5 -c 1 -o gpurun_out/wave5_full python bench.py --no-kernels --no-cpu --steps 2 --warmup 3 > gpurun_out/ncu_full.log 2>&1
echo "exit=$?" >> gpurun_out/ncu_full.log
