# round 2, call 52 (2 GPUs): per-pass timeline at N=2 with more NCCL channels / other protocols (is the exchange
# slow because one starved CTA moves the rows?)
mkdir -p gpurun_out/r02
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for cfg in "NCCL_MIN_NCHANNELS=16 NCCL_MIN_CTAS=16" "NCCL_PROTO=LL" "NCCL_PROTO=LL128" "NCCL_MIN_NCHANNELS=32 NCCL_MIN_CTAS=32 NCCL_PROTO=LL"; do
  echo "=== $cfg" >> gpurun_out/r02/g52_timeline_n2.log
  env $cfg timeout 600 $TR --nproc-per-node 2 --master-port 29591 scripts/r02/halo_timeline.py 2>&1 | grep -E "replay|halo pass  [1-4]:|stream 1 rows      8" | head -8 >> gpurun_out/r02/g52_timeline_n2.log
done
echo "exit=$?" >> gpurun_out/r02/g52_timeline_n2.log
