mkdir -p gpurun_out
timeout 1200 python -m pytest tests/ -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo "exit=$?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "exit=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo "exit=$?" >> gpurun_out/bench_full.log
timeout 300 python scripts/tf32_check.py 8192 > gpurun_out/tf32_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sgemm_3xtf32 -s 2 -c 1 -o gpurun_out/tf32_full python scripts/tf32_check.py 8192 > gpurun_out/ncu_tf32.log 2>&1
echo "exit=$?" >> gpurun_out/ncu_tf32.log
