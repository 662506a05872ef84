# round 2, call 38 (1 GPU): ncu of the two-warp KL=8 pass (source-level stalls)
mkdir -p gpurun_out/r02
CQ_WAVE_FUSED_CFG=8,6 timeout 900 ncu --set full --clock-control none --import-source on -k regex:pair -s 2 -c 1 \
  -o gpurun_out/r02/g38_pair python scripts/r02/prof_one.py 8 > gpurun_out/r02/g38_ncu.log 2>&1
echo "exit=$?" >> gpurun_out/r02/g38_ncu.log
