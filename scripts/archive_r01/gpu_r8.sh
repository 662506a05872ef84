mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "jit" > gpurun_out/gpu_jit.log 2>&1; echo "exit=$?" >> gpurun_out/gpu_jit.log
timeout 300 python scripts/tf32_once.py 8192 > gpurun_out/tf32_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sgemm_3xtf32_kernel -c 1 -o gpurun_out/tf32_full python scripts/tf32_once.py 8192 > gpurun_out/ncu_tf32.log 2>&1
echo "exit=$?" >> gpurun_out/ncu_tf32.log
