# round 2, call 31 (1 GPU): read-only DVFS probe v2 (sampler process)
mkdir -p gpurun_out/r02
timeout 600 python scripts/r02/dvfs_probe.py > gpurun_out/r02/g31_dvfs.json 2> gpurun_out/r02/g31_dvfs.err; echo "exit=$?" >> gpurun_out/r02/g31_dvfs.err
