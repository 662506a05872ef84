# round 2, call 76 (2 GPUs): final-code records on two GPUs -- pytest -m gpu (multi-rank tests included), bench N=2
mkdir -p gpurun_out/r02
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02/g76_gpu_tests_2gpu.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g76_gpu_tests_2gpu.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 \
  bench.py --gpus 2 > gpurun_out/r02/g76_bench_n2.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g76_bench_n2.log
tail -n 3 gpurun_out/r02/g76_gpu_tests_2gpu.log
