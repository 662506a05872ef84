mkdir -p gpurun_out
L=gpurun_out/tf32_2sm.log
: > $L
md5sum paper_2505_06022_b200/libcq.so >> $L
timeout 300 python scripts/tf32_check.py 4096 >> $L 2>&1; echo "exit=$? (2sm check)" >> $L
timeout 400 python scripts/tf32_ab.py 16384 >> $L 2>&1; echo "exit=$? (ab)" >> $L
nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv >> $L
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "sgemm" >> $L 2>&1; echo "exit=$? (pytest)" >> $L
