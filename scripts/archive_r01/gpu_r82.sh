mkdir -p gpurun_out
timeout 1500 python -m pytest tests/ -q -m gpu -x > gpurun_out/r82_gpu_tests.log 2>&1; echo "exit=$?" >> gpurun_out/r82_gpu_tests.log
: > gpurun_out/r82_ab.log
for i in 1 2; do
timeout 600 python bench.py --no-cpu --no-energy --no-kernels 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],3), round(d['roofline']['achieved']), d['config']['execution'][:80], d['gpu_launches'])" >> gpurun_out/r82_ab.log
done
