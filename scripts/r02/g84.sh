# round 2, call 84 (4 GPUs): run / run_batch sessions exchange halo rows over NCCL (peer_halo=False), replayed sessions
# keep the peer-memory path -- the 4-rank check, then bench N=4 default vs CQ_WAVE_P2P=1 (peer forced in run_batch too),
# alternating twice, then bench N=2 default
mkdir -p gpurun_out/r02
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29581 \
  scripts/mgpu_check.py > gpurun_out/r02/g84_mgpu_check_n4.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g84_mgpu_check_n4.log
for i in 1 2; do
  for p in dflt 1; do
    if [ $p = dflt ]; then unset CQ_WAVE_P2P; else export CQ_WAVE_P2P=1; fi
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
      --master-port 2958$((i+1)) bench.py --gpus 4 --no-kernels --no-cpu --no-energy > gpurun_out/r02/g84_bench_n4_p2p${p}_$i.log 2>&1
    echo "exit=$?" >> gpurun_out/r02/g84_bench_n4_p2p${p}_$i.log
  done
done
unset CQ_WAVE_P2P
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29585 \
  bench.py --gpus 2 --no-kernels --no-cpu --no-energy > gpurun_out/r02/g84_bench_n2.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g84_bench_n2.log
tail -n 2 gpurun_out/r02/g84_mgpu_check_n4.log
