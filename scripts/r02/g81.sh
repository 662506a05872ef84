# round 2, call 81 (4 GPUs): same-box A/B of the containment upload dedup at N=4 -- bench with the previous and the
# new executor, alternating (prev, new, prev, new); e2e, its batches and its measured floor per run
mkdir -p gpurun_out/r02
P=paper_2505_06022_b200/executor.py
for i in 1 2; do
  for v in prev new; do
    cp scripts/r02/ab_tmp/executor_$v.py $P
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2955$i \
      bench.py --gpus 4 --no-kernels --no-cpu --no-energy > gpurun_out/r02/g81_bench_n4_${v}_$i.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g81_bench_n4_${v}_$i.log
  done
done
cp scripts/r02/ab_tmp/executor_new.py $P
ls gpurun_out/r02 | grep g81
