# round 2, call 43 (1 GPU): e2e leg vs NUMA placement (default affinity vs bound to the GPU's local CPUs)
mkdir -p gpurun_out/r02
(nvidia-smi topo -m; lscpu | head -30; numactl -H 2>&1 | head -20) > gpurun_out/r02/g43_topo.log 2>&1
for r in 1 2; do
  timeout 600 python scripts/r02/e2e_numa.py >> gpurun_out/r02/g43_e2e.log 2>&1
  timeout 600 python scripts/r02/e2e_numa.py bind >> gpurun_out/r02/g43_e2e.log 2>&1
done
echo "exit=$?" >> gpurun_out/r02/g43_e2e.log
