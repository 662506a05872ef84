# round 2, call 6: ncu --set full (source-level) of the current KL=8 pass (one-warp blocks, 224-row strip-minor ranges)
mkdir -p gpurun_out/r02
timeout 300 python scripts/r02/prof_one.py 8 > gpurun_out/r02/g06_prof.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:wave5_fused -s 2 -c 1 \
  -o gpurun_out/r02/fused8_map2 python scripts/r02/prof_one.py 8 > gpurun_out/r02/g06_ncu.log 2>&1
timeout 300 python scripts/r02/prof_one.py 4 > gpurun_out/r02/g06_prof4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none -k regex:wave5_fused -s 2 -c 1 \
  -o gpurun_out/r02/fused4_map2 python scripts/r02/prof_one.py 4 > gpurun_out/r02/g06_ncu4.log 2>&1
echo done
