mkdir -p gpurun_out
CQ_WAVE_SPLIT=1 timeout 600 python scripts/fused_check.py > gpurun_out/split_check.log 2>&1; echo "exit=$?" >> gpurun_out/split_check.log
CQ_WAVE_SPLIT=1 timeout 900 python -m pytest tests/ -q -m gpu -x -k "fused or wave" > gpurun_out/split_tests.log 2>&1; echo "exit=$?" >> gpurun_out/split_tests.log
: > gpurun_out/split_ab.log
for sp in 1 0 1 0; do
CQ_WAVE_SPLIT=$sp timeout 600 python bench.py --no-cpu --no-energy --no-kernels 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('split=$sp', round(d['value']), round(d['ms_per_step'],3), round(d['roofline']['achieved']))" >> gpurun_out/split_ab.log
done
