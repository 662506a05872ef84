mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -q -m gpu -x -k "batch or multirank" > gpurun_out/gpu_tests_batch.log 2>&1; echo "exit=$?" >> gpurun_out/gpu_tests_batch.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 scripts/batch_diag.py > gpurun_out/batch_diag_2c.log 2>&1; echo "exit=$?" >> gpurun_out/batch_diag_2c.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29534 scripts/batch_diag.py > gpurun_out/batch_diag_1c.log 2>&1; echo "exit=$?" >> gpurun_out/batch_diag_1c.log
bash scripts/gpu_bench_multi.sh 2
timeout 900 python bench.py --no-kernels --no-energy --no-cpu > gpurun_out/bench_r51_n1.log 2>&1; echo "exit=$?" >> gpurun_out/bench_r51_n1.log
