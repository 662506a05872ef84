# round 2, call 32 (1 GPU): ncu --set full with source counters of the KL=8 pass (per-instruction stall samples)
mkdir -p gpurun_out/r02
timeout 300 python scripts/r02/prof_one.py 8 > gpurun_out/r02/g32_prof.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:wave5_fused -s 2 -c 1 \
  -o gpurun_out/r02/g32_fused8 python scripts/r02/prof_one.py 8 > gpurun_out/r02/g32_ncu.log 2>&1
echo "exit=$?" >> gpurun_out/r02/g32_ncu.log
