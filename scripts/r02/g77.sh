# round 2, call 77 (2 GPUs): upload dedup by containment (u's slab + halo rows contains up's) -- GPU tests,
# the 2-rank check, bench N=2 (e2e)
mkdir -p gpurun_out/r02
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02/g77_gpu_tests_2gpu.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g77_gpu_tests_2gpu.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29518 \
  scripts/mgpu_check.py > gpurun_out/r02/g77_mgpu_check_n2.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g77_mgpu_check_n2.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 \
  bench.py --gpus 2 > gpurun_out/r02/g77_bench_n2.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g77_bench_n2.log
tail -n 2 gpurun_out/r02/g77_gpu_tests_2gpu.log gpurun_out/r02/g77_mgpu_check_n2.log
