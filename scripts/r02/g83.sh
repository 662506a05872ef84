# round 2, call 83 (4 GPUs): e2e at N=4 with the peer-memory halo (default) vs the NCCL exchange (CQ_WAVE_P2P=0),
# alternating twice on one box
mkdir -p gpurun_out/r02
for i in 1 2; do
  for p in 1 0; do
    CQ_WAVE_P2P=$p timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
      --master-port 2957$i bench.py --gpus 4 --no-kernels --no-cpu --no-energy > gpurun_out/r02/g83_bench_n4_p2p${p}_$i.log 2>&1
    echo "exit=$?" >> gpurun_out/r02/g83_bench_n4_p2p${p}_$i.log
  done
done
ls gpurun_out/r02 | grep g83
