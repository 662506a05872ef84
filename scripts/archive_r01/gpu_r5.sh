mkdir -p gpurun_out
for args in "2 16384" "2 16384 --torch" "1 16384" "2 4096" "4 8192"; do
  echo "== $args" >> gpurun_out/pin.log
  timeout 300 python scripts/pin_repro.py $args >> gpurun_out/pin.log 2>&1
done
for np in 1 2 3 4; do
  echo "== NP=$np" >> gpurun_out/nbody_np.log
  CQ_NBODY_NP=$np timeout 300 python bench.py --no-cpu --no-energy --size 2048 --wave-steps 4 --steps 2 --warmup 3 --sgemm 1024 --sgemm-variants ffma 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps(d['kernels']['nbody_262144']['roofline']))" >> gpurun_out/nbody_np.log 2>&1
done
for mc in 1 2; do
  echo "== MC=$mc" >> gpurun_out/tf32.log
  CQ_TF32_MC=$mc timeout 300 python scripts/tf32_check.py >> gpurun_out/tf32.log 2>&1; echo "exit=$?" >> gpurun_out/tf32.log
done
