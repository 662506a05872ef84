# round 2, call 67 (1 GPU): 3xTF32 with B MN-major straight from [k, n] -- bit-equality vs transposed, tolerance,
# sgemm tests, timing A/B (every command bounded by timeout)
mkdir -p gpurun_out/r02
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "mn_major" > gpurun_out/r02/g67_mnb.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g67_mnb.log
if grep -q "passed" gpurun_out/r02/g67_mnb.log && ! grep -q "failed" gpurun_out/r02/g67_mnb.log; then
  timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "tf32 or sgemm" > gpurun_out/r02/g67_tests.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g67_tests.log
  sed -i 's/CQ_TF32_RAW_HI/CQ_TF32_MNB/' scripts/r02/tf32_raw_ab.py
  timeout 600 python scripts/r02/tf32_raw_ab.py > gpurun_out/r02/g67_ab.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g67_ab.log
fi
