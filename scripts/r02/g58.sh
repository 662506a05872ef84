# round 2, call 58 (2 GPUs): rehearsal at HEAD -- pytest -m gpu on 2 GPUs (multi-rank tests included), smoke, bench N=1
mkdir -p gpurun_out/r02
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02/g58_gpu_tests_2gpu.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g58_gpu_tests_2gpu.log
CUDA_VISIBLE_DEVICES=0 timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02/g58_gpu_tests_1gpu.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g58_gpu_tests_1gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02/g58_smoke.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g58_smoke.log
timeout 900 python bench.py > gpurun_out/r02/g58_bench_n1.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g58_bench_n1.log
