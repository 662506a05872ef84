# round 2, call 50 (2 GPUs): per-pass timeline at N=2 with small NCCL CTAs (can they co-reside with the interior pass?)
mkdir -p gpurun_out/r02
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for cfg in "NCCL_NTHREADS=64 NCCL_MAX_NCHANNELS=1 NCCL_MIN_NCHANNELS=1" "NCCL_NTHREADS=128 NCCL_MAX_CTAS=1 NCCL_MIN_CTAS=1" "NCCL_P2P_USE_CUDA_MEMCPY=1"; do
  echo "=== $cfg" >> gpurun_out/r02/g50_timeline_n2.log
  env $cfg timeout 600 $TR --nproc-per-node 2 --master-port 29581 scripts/r02/halo_timeline.py 2>&1 | grep -v "^\*\|OMP_NUM\|^$" | head -30 >> gpurun_out/r02/g50_timeline_n2.log
done
echo "exit=$?" >> gpurun_out/r02/g50_timeline_n2.log
