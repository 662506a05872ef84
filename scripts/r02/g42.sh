# round 2, call 42 (1 GPU): fast form with c*lap as FFMA2(c, lap, +0) + FADD2 (2 fewer instructions per level-row)
# vs HEAD; parity of both; then the GPU test suite with the new library
mkdir -p gpurun_out/r02
for r in 1 2 3; do
  CQ_LIB=build/exp/libcq_head.so timeout 300 python scripts/r02/lib_ab.py >> gpurun_out/r02/g42_ab.log 2>&1
  timeout 300 python scripts/r02/lib_ab.py >> gpurun_out/r02/g42_ab.log 2>&1
done
echo "exit=$?" >> gpurun_out/r02/g42_ab.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02/g42_gpu_tests.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g42_gpu_tests.log
