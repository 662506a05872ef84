# round 2, call 85 (1 GPU): final code -- pytest -m gpu, smoke, bench N=1, reference arm N=1
mkdir -p gpurun_out/r02
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02/g85_gpu_tests.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g85_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02/g85_smoke.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g85_smoke.log
timeout 900 python bench.py > gpurun_out/r02/g85_bench_n1.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g85_bench_n1.log
timeout 900 python bench.py --impl reference > gpurun_out/r02/g85_bench_ref_n1.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g85_bench_ref_n1.log
tail -n 2 gpurun_out/r02/g85_gpu_tests.log gpurun_out/r02/g85_smoke.log
