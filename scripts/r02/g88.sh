# round 2, call 88 (1 GPU): 3xTF32 with the lo split inside the CTA-pair kernel (CQ_TF32_INSPLIT=1, 4 converter warps) -- bit-equality,
# then an interleaved timing A/B (every command bounded by timeout)
mkdir -p gpurun_out/r02
timeout 180 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "in_kernel_split" > gpurun_out/r02/g88_ins.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g88_ins.log
if grep -q "passed" gpurun_out/r02/g88_ins.log && ! grep -q "failed" gpurun_out/r02/g88_ins.log; then
  timeout 600 python scripts/r02/tf32_env_ab.py CQ_TF32_INSPLIT 1 0 > gpurun_out/r02/g88_ab.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g88_ab.log
fi
tail -n 5 gpurun_out/r02/g88_ins.log; cat gpurun_out/r02/g88_ab.log 2>/dev/null
