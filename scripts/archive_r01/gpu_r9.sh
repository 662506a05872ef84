mkdir -p gpurun_out
for bk in 16 32; do
  echo "== BK=$bk" >> gpurun_out/tf32.log
  CQ_TF32_BK=$bk timeout 300 python scripts/tf32_check.py >> gpurun_out/tf32.log 2>&1; echo "exit=$?" >> gpurun_out/tf32.log
done
