# round 2, call 40 (1 GPU): two-warp KL=8 pass, lock-step barrier vs mbarrier hand-off, vs the one-warp pass
mkdir -p gpurun_out/r02
for r in 1 2; do
  timeout 300 python scripts/r02/lib_ab.py >> gpurun_out/r02/g40_ab.log 2>&1
  CQ_LIB=build/exp/libcq_pair_bar.so CQ_WAVE_FUSED_CFG=8,6 timeout 300 python scripts/r02/lib_ab.py >> gpurun_out/r02/g40_ab.log 2>&1
  CQ_LIB=build/exp/libcq_pair_mbar.so CQ_WAVE_FUSED_CFG=8,6 timeout 300 python scripts/r02/lib_ab.py >> gpurun_out/r02/g40_ab.log 2>&1
done
echo "exit=$?" >> gpurun_out/r02/g40_ab.log
