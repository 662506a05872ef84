mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "graph or saxpy_f32 or wave_bit" > gpurun_out/gpu_tests.log 2>&1; echo "exit=$?" >> gpurun_out/gpu_tests.log
timeout 900 python bench.py --no-cpu --sgemm-variants 3xtf32 > gpurun_out/bench_full.log 2>&1; echo "exit=$?" >> gpurun_out/bench_full.log
