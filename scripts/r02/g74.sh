# round 2, call 74 (1 GPU): 3xTF32 B MN-major (SWIZZLE_128B_BASE32B) -- bit-equality vs transposed, sgemm tests,
# timing A/B (every command bounded by timeout)
mkdir -p gpurun_out/r02
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "mn_major" > gpurun_out/r02/g74_mnb.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g74_mnb.log
if grep -q "passed" gpurun_out/r02/g74_mnb.log && ! grep -q "failed" gpurun_out/r02/g74_mnb.log; then
  timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "tf32 or sgemm" > gpurun_out/r02/g74_tests.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g74_tests.log
  timeout 600 python scripts/r02/tf32_mnb_ab.py > gpurun_out/r02/g74_ab.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g74_ab.log
fi
tail -3 gpurun_out/r02/g74_*.log
