# round 2, call 45 (1 GPU): records at the final code -- bench, reference arm, launch list, ncu of the KL=8 pass
mkdir -p gpurun_out/r02
timeout 900 python bench.py > gpurun_out/r02/g45_bench_n1.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g45_bench_n1.log
timeout 900 python bench.py --impl reference > gpurun_out/r02/g45_bench_ref_n1.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g45_bench_ref_n1.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02/g45_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-energy --no-kernels > gpurun_out/r02/g45_ncu_launch.log 2>&1
echo "exit=$?" >> gpurun_out/r02/g45_ncu_launch.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:wave5_fused -s 2 -c 1 \
  -o gpurun_out/r02/g45_fused8 python scripts/r02/prof_one.py 8 > gpurun_out/r02/g45_ncu8.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:wave5_fused -s 2 -c 1 \
  -o gpurun_out/r02/g45_fused4 python scripts/r02/prof_one.py 4 > gpurun_out/r02/g45_ncu4.log 2>&1
echo done
