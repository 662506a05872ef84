# round 2, call 65 (1 GPU): final-code records (g64 again; ncu reports reduced to CSV on the box: the reports
# themselves exceed the 64 MiB copy-back limit)
mkdir -p gpurun_out/r02
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02/g65_gpu_tests.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g65_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02/g65_smoke.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g65_smoke.log
timeout 900 python bench.py > gpurun_out/r02/g65_bench_n1.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g65_bench_n1.log
timeout 900 python bench.py --impl reference > gpurun_out/r02/g65_bench_ref_n1.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g65_bench_ref_n1.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02/g65_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-energy --no-kernels > gpurun_out/r02/g65_ncu_launch.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g65_ncu_launch.log
for k in 8 4; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:wave5_fused -s 2 -c 1 \
    -o /tmp/g65_fused$k python scripts/r02/prof_one.py $k > gpurun_out/r02/g65_ncu$k.log 2>&1
  ncu -i /tmp/g65_fused$k.ncu-rep --page raw --csv > gpurun_out/r02/g65_fused${k}_raw.csv 2>/dev/null
  ncu -i /tmp/g65_fused$k.ncu-rep --page source --csv --print-source sass > gpurun_out/r02/g65_fused${k}_source.csv 2>/dev/null
done
ls -la gpurun_out/r02 | tail -5
echo done
