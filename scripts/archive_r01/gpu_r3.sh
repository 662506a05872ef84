mkdir -p gpurun_out
for bn in 256 128; do
  for g in 4 16; do
    echo "== BN=$bn GROUP_KB=$g" >> gpurun_out/tf32.log
    CQ_TF32_BN=$bn CQ_TF32_GROUP_KB=$g timeout 300 python scripts/tf32_check.py >> gpurun_out/tf32.log 2>&1; echo "exit=$?" >> gpurun_out/tf32.log
  done
done
timeout 600 python bench.py --no-cpu --sgemm-variants 3xtf32,ffma > gpurun_out/bench_full.log 2>&1; echo "exit=$?" >> gpurun_out/bench_full.log
