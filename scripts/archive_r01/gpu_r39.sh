mkdir -p gpurun_out
: > gpurun_out/batch_depth.log
for d in 2 3 4; do
CQ_BATCH_DEPTH=$d timeout 900 python bench.py --no-kernels --no-cpu --no-energy 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('depth', $d, json.dumps(d['e2e']))" >> gpurun_out/batch_depth.log
done
