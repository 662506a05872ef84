mkdir -p gpurun_out
timeout 300 python scripts/fused_prof.py 4 > gpurun_out/fused_prof.log 2>&1; echo "exit=$?" >> gpurun_out/fused_prof.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:wave5_fused -s 1 -c 1 -o gpurun_out/fused4_full python scripts/fused_prof.py 4 >> gpurun_out/fused_prof.log 2>&1; echo "exit=$?" >> gpurun_out/fused_prof.log
