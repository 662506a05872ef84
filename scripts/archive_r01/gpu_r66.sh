mkdir -p gpurun_out
timeout 600 python scripts/fused_check.py > gpurun_out/lin_check.log 2>&1; echo "exit=$?" >> gpurun_out/lin_check.log
timeout 900 python -m pytest tests/ -q -m gpu -x -k "fused or wave or smoke" > gpurun_out/lin_tests.log 2>&1; echo "exit=$?" >> gpurun_out/lin_tests.log
: > gpurun_out/lin_ab.log
for v in lin w12 lin w12; do
  if [ $v = w12 ]; then export CQ_LIB=$PWD/paper_2505_06022_b200/libcq_w12.so; else unset CQ_LIB; fi
  timeout 600 python bench.py --no-cpu --no-energy 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print('$v', round(d['value']), round(d['ms_per_step'],3), round(d['roofline']['achieved']), 'strong', round(k['wave_f32_strong']['value']), 'f64', round(k['wave_f64_weak']['value']))" >> gpurun_out/lin_ab.log
done
unset CQ_LIB
timeout 600 python scripts/seg_check.py > gpurun_out/seg_check3.log 2>&1
