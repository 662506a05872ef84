# round 2, call 30 (1 GPU): GPU tests after the NVML-window fix; read-only DVFS probe
mkdir -p gpurun_out/r02
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02/g30_gpu_tests.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g30_gpu_tests.log
timeout 600 python scripts/r02/dvfs_probe.py > gpurun_out/r02/g30_dvfs.json 2> gpurun_out/r02/g30_dvfs.err; echo "exit=$?" >> gpurun_out/r02/g30_dvfs.err
