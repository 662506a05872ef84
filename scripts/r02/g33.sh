# round 2, call 33 (1 GPU): A/B of the FMA-form wave arithmetic -- packed FP32x2 (libcq.so) vs all-scalar
# with immediate-form FFMA (build/exp/libcq_scalar.so); alternating processes
mkdir -p gpurun_out/r02
for r in 1 2 3; do
  timeout 300 python scripts/r02/lib_ab.py >> gpurun_out/r02/g33_ab.log 2>&1
  CQ_LIB=build/exp/libcq_scalar.so timeout 300 python scripts/r02/lib_ab.py >> gpurun_out/r02/g33_ab.log 2>&1
done
echo "exit=$?" >> gpurun_out/r02/g33_ab.log
