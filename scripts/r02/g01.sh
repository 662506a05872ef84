# round 2, call 1: NVML clock-control probe (read-only), baseline bench line, full ncu of the KL=8 pass
mkdir -p gpurun_out/r02
python scripts/nvml_probe.py > gpurun_out/r02/nvml_probe.json 2>&1
nvidia-smi -q -d CLOCK,POWER,PERFORMANCE > gpurun_out/r02/smi_q.txt 2>&1
timeout 600 python bench.py --no-cpu --no-energy --no-kernels > gpurun_out/r02/g01_bench.log 2>&1
timeout 300 python scripts/fused_prof.py 8 fast > gpurun_out/r02/g01_prof.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:wave5_fused -s 2 -c 1 \
  -o gpurun_out/r02/fused8_base python scripts/fused_prof.py 8 fast > gpurun_out/r02/g01_ncu.log 2>&1
echo done
