# round 2, call 39 (1 GPU): two-warp KL=8 pass (CQ_WAVE_FUSED_CFG=8,6) vs the one-warp pass: parity + A/B
mkdir -p gpurun_out/r02
for r in 1 2 3; do
  timeout 300 python scripts/r02/lib_ab.py >> gpurun_out/r02/g39_ab.log 2>&1
  CQ_WAVE_FUSED_CFG=8,6 timeout 300 python scripts/r02/lib_ab.py >> gpurun_out/r02/g39_ab.log 2>&1
done
echo "exit=$?" >> gpurun_out/r02/g39_ab.log
