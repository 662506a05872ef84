# round 2, call 54 (2 GPUs): in-kernel peer stores of the halo rows -- single-GPU A/B of the pass vs HEAD,
# multi-rank parity, per-pass timeline, bench N=2 with and without the peer path
mkdir -p gpurun_out/r02
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for r in 1 2; do
  CQ_LIB=build/exp/libcq_head2.so timeout 300 python scripts/r02/lib_ab.py >> gpurun_out/r02/g54_ab.log 2>&1
  timeout 300 python scripts/r02/lib_ab.py >> gpurun_out/r02/g54_ab.log 2>&1
done
timeout 600 $TR --nproc-per-node 2 --master-port 29611 scripts/mgpu_check.py > gpurun_out/r02/g54_mgpu_check_n2.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g54_mgpu_check_n2.log
timeout 300 $TR --nproc-per-node 2 --master-port 29612 scripts/r02/halo_timeline.py > gpurun_out/r02/g54_timeline_n2.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g54_timeline_n2.log
timeout 900 $TR --nproc-per-node 2 --master-port 29613 bench.py --gpus 2 --no-kernels --no-cpu --no-energy > gpurun_out/r02/g54_bench_n2_p2p.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g54_bench_n2_p2p.log
CQ_WAVE_P2P=0 timeout 900 $TR --nproc-per-node 2 --master-port 29614 bench.py --gpus 2 --no-kernels --no-cpu --no-energy > gpurun_out/r02/g54_bench_n2_nccl.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g54_bench_n2_nccl.log
