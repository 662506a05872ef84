# round 2, call 9 (2 GPUs): multi-rank parity (all-gather path), NCCL collective log, multi-rank GPU tests, bench N=2
mkdir -p gpurun_out/r02
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=COLL timeout 600 $TR --master-port 29511 scripts/mgpu_check.py > gpurun_out/r02/g09_mgpu_check_n2.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g09_mgpu_check_n2.log
timeout 900 python -m pytest tests/test_gpu_multirank.py -q -m gpu > gpurun_out/r02/g09_multirank_tests.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g09_multirank_tests.log
timeout 1200 $TR --master-port 29512 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/r02/g09_bench_n2.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g09_bench_n2.log
timeout 900 $TR --master-port 29513 bench.py --impl reference --gpus 2 --steps 3 --warmup 3 > gpurun_out/r02/g09_bench_ref_n2.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g09_bench_ref_n2.log
