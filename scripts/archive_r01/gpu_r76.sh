mkdir -p gpurun_out
CQ_LIB=$PWD/paper_2505_06022_b200/libcq_w16.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "fast_form or baseline" > gpurun_out/w16_tests.log 2>&1; echo "exit=$?" >> gpurun_out/w16_tests.log
: > gpurun_out/w16_ab.log
for v in w16 w12 w16 w12; do
  if [ $v = w16 ]; then export CQ_LIB=$PWD/paper_2505_06022_b200/libcq_w16.so; else unset CQ_LIB; fi
  timeout 600 python bench.py --no-cpu --no-energy --no-kernels 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value']), round(d['ms_per_step'],3), round(d['roofline']['achieved']))" >> gpurun_out/w16_ab.log
done
