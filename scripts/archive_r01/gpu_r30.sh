mkdir -p gpurun_out
: > gpurun_out/nbody_np.log
for np in 4 6 8; do
  echo "== NP=$np" >> gpurun_out/nbody_np.log
  CQ_NBODY_NP=$np timeout 300 python bench.py --no-cpu --no-energy --size 2048 --wave-steps 4 --steps 2 --warmup 3 --sgemm 1024 --sgemm-variants ffma 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps(d['kernels']['nbody_262144']['roofline']))" >> gpurun_out/nbody_np.log 2>&1
done
timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k nbody >> gpurun_out/nbody_np.log 2>&1
