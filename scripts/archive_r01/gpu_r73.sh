mkdir -p gpurun_out
CQ_LIB=$PWD/paper_2505_06022_b200/libcq_old.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "fast_form" > gpurun_out/zeros_old.log 2>&1; echo "exit=$?" >> gpurun_out/zeros_old.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "fast_form" > gpurun_out/zeros_new.log 2>&1; echo "exit=$?" >> gpurun_out/zeros_new.log
