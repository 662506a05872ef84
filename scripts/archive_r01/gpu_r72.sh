mkdir -p gpurun_out
CQ_LIB=$PWD/paper_2505_06022_b200/libcq_old.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "signed_zeros" > gpurun_out/zeros_old.log 2>&1; echo "exit=$?" >> gpurun_out/zeros_old.log
timeout 1500 python -m pytest tests/ -q -m gpu -x > gpurun_out/r72_gpu_tests.log 2>&1; echo "exit=$?" >> gpurun_out/r72_gpu_tests.log
timeout 600 python scripts/fused_check.py > gpurun_out/r72_check.log 2>&1; echo "exit=$?" >> gpurun_out/r72_check.log
: > gpurun_out/r72_ab.log
for i in 1 2; do
timeout 600 python bench.py --no-cpu --no-energy --no-kernels 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],3), round(d['roofline']['achieved']))" >> gpurun_out/r72_ab.log
done
