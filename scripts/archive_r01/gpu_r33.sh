mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_r33.log 2>&1; echo "exit=$?" >> gpurun_out/bench_r33.log
