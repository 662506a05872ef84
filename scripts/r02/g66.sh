# round 2, call 66 (2 GPUs): multi-rank check with huge values in a neighbour's halo rows (peer path and NCCL path)
mkdir -p gpurun_out/r02
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 $TR --nproc-per-node 2 --master-port 29641 scripts/mgpu_check.py > gpurun_out/r02/g66_mgpu_check_n2.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g66_mgpu_check_n2.log
CQ_WAVE_P2P=0 timeout 600 $TR --nproc-per-node 2 --master-port 29642 scripts/mgpu_check.py > gpurun_out/r02/g66_mgpu_check_n2_nccl.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g66_mgpu_check_n2_nccl.log
