# round 2, call 29 (1 GPU): round-end rehearsal at HEAD after the container was re-created --
# pytest -m gpu, smoke(), default bench, reference arm, launch list of the bench
mkdir -p gpurun_out/r02
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02/g29_gpu_tests.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g29_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02/g29_smoke.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g29_smoke.log
timeout 900 python bench.py > gpurun_out/r02/g29_bench_n1.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g29_bench_n1.log
timeout 900 python bench.py --impl reference > gpurun_out/r02/g29_bench_ref_n1.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g29_bench_ref_n1.log
