mkdir -p gpurun_out
timeout 600 python scripts/fused_check.py > gpurun_out/w12_check.log 2>&1; echo "exit=$?" >> gpurun_out/w12_check.log
timeout 900 python -m pytest tests/ -q -m gpu -x -k "fused or wave" > gpurun_out/w12_tests.log 2>&1; echo "exit=$?" >> gpurun_out/w12_tests.log
CQ_LIB=$PWD/paper_2505_06022_b200/libcq_w8.so timeout 900 python -m pytest tests/ -q -m gpu -x -k "fused or wave" > gpurun_out/w8_tests.log 2>&1; echo "exit=$?" >> gpurun_out/w8_tests.log
: > gpurun_out/w_ab.log
for v in w12 w8 w12 w8; do
  if [ $v = w8 ]; then export CQ_LIB=$PWD/paper_2505_06022_b200/libcq_w8.so; else unset CQ_LIB; fi
  timeout 600 python bench.py --no-cpu --no-energy --no-kernels 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value']), round(d['ms_per_step'],3), round(d['roofline']['achieved']))" >> gpurun_out/w_ab.log
done
unset CQ_LIB
timeout 300 python scripts/fused_prof.py 8 fast > gpurun_out/w12_prof.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:wave5_fused -s 1 -c 1 -o gpurun_out/w12_r65 python scripts/fused_prof.py 8 fast > gpurun_out/ncu_w12.log 2>&1
