# round 2, call 56 (2 GPUs): peer halo rows with the wait / signal inside the pass kernel (edge pieces only) --
# multi-rank parity, per-pass timeline, bench N=2 with and without, single-GPU pass timing
mkdir -p gpurun_out/r02
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 $TR --nproc-per-node 2 --master-port 29621 scripts/mgpu_check.py > gpurun_out/r02/g56_mgpu_check_n2.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g56_mgpu_check_n2.log
timeout 300 $TR --nproc-per-node 2 --master-port 29622 scripts/r02/halo_timeline.py > gpurun_out/r02/g56_timeline_n2.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g56_timeline_n2.log
for r in 1 2; do
timeout 900 $TR --nproc-per-node 2 --master-port 29623 bench.py --gpus 2 --no-kernels --no-cpu --no-energy > gpurun_out/r02/g56_bench_n2_p2p_$r.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g56_bench_n2_p2p_$r.log
CQ_WAVE_P2P=0 timeout 900 $TR --nproc-per-node 2 --master-port 29624 bench.py --gpus 2 --no-kernels --no-cpu --no-energy > gpurun_out/r02/g56_bench_n2_nccl_$r.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g56_bench_n2_nccl_$r.log
done
timeout 300 python scripts/r02/lib_ab.py > gpurun_out/r02/g56_ab.log 2>&1
