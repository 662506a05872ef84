# round 2, call 82 (4 GPUs): e2e at N=4 against run_batch depth (CQ_BATCH_DEPTH 2 / 3 / 4, alternating twice)
mkdir -p gpurun_out/r02
for i in 1 2; do
  for dpt in 2 3 4; do
    CQ_BATCH_DEPTH=$dpt timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
      --master-port 2956$i bench.py --gpus 4 --no-kernels --no-cpu --no-energy > gpurun_out/r02/g82_bench_n4_d${dpt}_$i.log 2>&1
    echo "exit=$?" >> gpurun_out/r02/g82_bench_n4_d${dpt}_$i.log
  done
done
ls gpurun_out/r02 | grep g82
