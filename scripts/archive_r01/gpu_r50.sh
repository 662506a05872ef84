mkdir -p gpurun_out
timeout 1500 python -m pytest tests/ -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1; echo "exit=$?" >> gpurun_out/gpu_tests.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 scripts/batch_diag.py > gpurun_out/batch_diag_2b.log 2>&1; echo "exit=$?" >> gpurun_out/batch_diag_2b.log
bash scripts/gpu_bench_multi.sh 2
timeout 900 python bench.py --no-kernels --no-energy > gpurun_out/bench_r50_n1.log 2>&1; echo "exit=$?" >> gpurun_out/bench_r50_n1.log
