# round 2, call 80 (4 GPUs): final code on 4 GPUs -- the 4-rank check, bench N=4, N=2, N=1 (same box)
mkdir -p gpurun_out/r02
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29541 \
  scripts/mgpu_check.py > gpurun_out/r02/g80_mgpu_check_n4.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g80_mgpu_check_n4.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29542 \
  bench.py --gpus 4 > gpurun_out/r02/g80_bench_n4.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g80_bench_n4.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29543 \
  bench.py --gpus 2 > gpurun_out/r02/g80_bench_n2.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g80_bench_n2.log
timeout 900 python bench.py > gpurun_out/r02/g80_bench_n1.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g80_bench_n1.log
tail -n 2 gpurun_out/r02/g80_mgpu_check_n4.log
