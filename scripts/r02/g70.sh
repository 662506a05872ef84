# round 2, call 70 (2 GPUs): device-resident re-runs skip the first block's NCCL exchange -- parity, timeline, bench N=2
mkdir -p gpurun_out/r02
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 $TR --nproc-per-node 2 --master-port 29661 scripts/mgpu_check.py > gpurun_out/r02/g70_mgpu_check_n2.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g70_mgpu_check_n2.log
timeout 300 $TR --nproc-per-node 2 --master-port 29662 scripts/r02/halo_timeline.py > gpurun_out/r02/g70_timeline_n2.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g70_timeline_n2.log
timeout 900 python bench.py --no-kernels --no-cpu --no-energy > gpurun_out/r02/g70_bench_n1.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g70_bench_n1.log
timeout 900 $TR --nproc-per-node 2 --master-port 29663 bench.py --gpus 2 --no-kernels --no-cpu --no-energy > gpurun_out/r02/g70_bench_n2.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g70_bench_n2.log
