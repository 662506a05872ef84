# round 2, call 79 (2 GPUs): e2e at N=2 -- Session setup / close cost vs per-simulation run_batch time
mkdir -p gpurun_out/r02
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 \
  scripts/r02/e2e_setup_n2.py > gpurun_out/r02/g79_e2e_setup_n2.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g79_e2e_setup_n2.log
cat gpurun_out/r02/g79_e2e_setup_n2.log | grep -v Warning | tail -12
