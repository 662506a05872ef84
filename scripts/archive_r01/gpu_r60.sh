mkdir -p gpurun_out
: > gpurun_out/cfg_fast.log
for cfg in 4,3,256 4,6,256 4,3,256 4,6,256; do
  CQ_WAVE_FUSED_CFG=$cfg timeout 600 python bench.py --no-cpu --no-energy --no-kernels 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', round(d['value']), round(d['ms_per_step'],3), round(d['roofline']['achieved']))" >> gpurun_out/cfg_fast.log
done
