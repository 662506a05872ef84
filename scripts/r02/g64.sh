# round 2, call 64 (1 GPU): final-code records -- pytest -m gpu, smoke, bench, reference arm, launch list, ncu of the passes
mkdir -p gpurun_out/r02
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02/g64_gpu_tests.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g64_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02/g64_smoke.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g64_smoke.log
timeout 900 python bench.py > gpurun_out/r02/g64_bench_n1.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g64_bench_n1.log
timeout 900 python bench.py --impl reference > gpurun_out/r02/g64_bench_ref_n1.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g64_bench_ref_n1.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02/g64_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-energy --no-kernels > gpurun_out/r02/g64_ncu_launch.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g64_ncu_launch.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:wave5_fused -s 2 -c 1 \
  -o gpurun_out/r02/g64_fused8 python scripts/r02/prof_one.py 8 > gpurun_out/r02/g64_ncu8.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:wave5_fused -s 2 -c 1 \
  -o gpurun_out/r02/g64_fused4 python scripts/r02/prof_one.py 4 > gpurun_out/r02/g64_ncu4.log 2>&1
echo done
