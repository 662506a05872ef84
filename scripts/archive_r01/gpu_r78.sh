mkdir -p gpurun_out
timeout 1500 python -m pytest tests/ -q -m gpu -x > gpurun_out/r78_gpu_tests.log 2>&1; echo "exit=$?" >> gpurun_out/r78_gpu_tests.log
: > gpurun_out/order_ab.log
for v in new old new old; do
  timeout 600 python scripts/order_ab.py $v --no-cpu --no-energy --no-kernels 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value']), round(d['ms_per_step'],3), d['config']['execution'][:60])" >> gpurun_out/order_ab.log
done
