# round 2, call 47 (2 GPUs): final code -- multi-rank parity (incl. the broadcast lowering), GPU tests on 2 GPUs,
# bench N=1 and N=2, reference arm N=2
mkdir -p gpurun_out/r02
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=COLL timeout 600 $TR --nproc-per-node 2 --master-port 29551 scripts/mgpu_check.py > gpurun_out/r02/g47_mgpu_check_n2.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g47_mgpu_check_n2.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02/g47_gpu_tests_2gpu.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g47_gpu_tests_2gpu.log
timeout 900 python bench.py > gpurun_out/r02/g47_bench_n1.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g47_bench_n1.log
timeout 1200 $TR --nproc-per-node 2 --master-port 29552 bench.py --gpus 2 > gpurun_out/r02/g47_bench_n2.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g47_bench_n2.log
timeout 900 $TR --nproc-per-node 2 --master-port 29553 bench.py --impl reference --gpus 2 > gpurun_out/r02/g47_bench_ref_n2.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g47_bench_ref_n2.log
