# round 2, call 46 (1 GPU): steady-turn mode (no store / prefetch window tests in the body's middle turns) vs HEAD
mkdir -p gpurun_out/r02
for r in 1 2 3; do
  CQ_LIB=build/exp/libcq_head2.so timeout 300 python scripts/r02/lib_ab.py >> gpurun_out/r02/g46_ab.log 2>&1
  timeout 300 python scripts/r02/lib_ab.py >> gpurun_out/r02/g46_ab.log 2>&1
done
echo "exit=$?" >> gpurun_out/r02/g46_ab.log
