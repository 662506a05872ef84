# round 2, call 53 (2 GPUs): peer-memory halo rows (CUDA IPC + NVLink copies, device pass counters) --
# multi-rank parity, per-pass timeline, bench N=2 with and without it
mkdir -p gpurun_out/r02
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 $TR --nproc-per-node 2 --master-port 29601 scripts/mgpu_check.py > gpurun_out/r02/g53_mgpu_check_n2.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g53_mgpu_check_n2.log
timeout 300 $TR --nproc-per-node 2 --master-port 29602 scripts/r02/halo_timeline.py > gpurun_out/r02/g53_timeline_n2.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g53_timeline_n2.log
timeout 900 $TR --nproc-per-node 2 --master-port 29603 bench.py --gpus 2 --no-kernels --no-cpu --no-energy > gpurun_out/r02/g53_bench_n2_p2p.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g53_bench_n2_p2p.log
CQ_WAVE_P2P=0 timeout 900 $TR --nproc-per-node 2 --master-port 29604 bench.py --gpus 2 --no-kernels --no-cpu --no-energy > gpurun_out/r02/g53_bench_n2_nccl.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g53_bench_n2_nccl.log
