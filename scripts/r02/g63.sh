# round 2, call 63 (1 GPU): 3xTF32 with A as its own hi part -- bit-equality test, sgemm tests, timing A/B
mkdir -p gpurun_out/r02
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "tf32 or sgemm" > gpurun_out/r02/g63_tests.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g63_tests.log
timeout 600 python scripts/r02/tf32_raw_ab.py > gpurun_out/r02/g63_ab.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g63_ab.log
