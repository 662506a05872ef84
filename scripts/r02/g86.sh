# round 2, call 86 (1 GPU): 3xTF32 rasterisation / drain-group sweep (no code change; env knobs)
mkdir -p gpurun_out/r02
timeout 900 python scripts/r02/tf32_raster_sweep.py > gpurun_out/r02/g86_tf32_raster.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g86_tf32_raster.log
cat gpurun_out/r02/g86_tf32_raster.log
