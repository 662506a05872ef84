# round 2, call 75 (1 GPU): records at the MN-major-B code -- pytest -m gpu, smoke, bench N=1, and an ncu --set full
# of the CTA-pair SGEMM (MN-major B instantiation) plus the split pass, reduced to CSV on the box
mkdir -p gpurun_out/r02
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02/g75_gpu_tests.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g75_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02/g75_smoke.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g75_smoke.log
timeout 900 python bench.py > gpurun_out/r02/g75_bench_n1.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g75_bench_n1.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sgemm_3xtf32_2sm|split_lo" -s 3 -c 3 \
  -o /tmp/g75_sgemm python scripts/r02/prof_kernels.py sgemm > gpurun_out/r02/g75_ncu_sgemm.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g75_ncu_sgemm.log
ncu -i /tmp/g75_sgemm.ncu-rep --page raw --csv > gpurun_out/r02/g75_sgemm_raw.csv 2>/dev/null
ncu -i /tmp/g75_sgemm.ncu-rep --page details --csv > gpurun_out/r02/g75_sgemm_details.csv 2>/dev/null
ls -la gpurun_out/r02 | grep g75
