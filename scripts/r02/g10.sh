# round 2, call 10 (4 GPUs): multi-rank parity at N=4, bench N=4 (+ N=2 on the same box) and the reference arm
mkdir -p gpurun_out/r02
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=COLL timeout 600 $TR --nproc-per-node 4 --master-port 29521 scripts/mgpu_check.py > gpurun_out/r02/g10_mgpu_check_n4.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g10_mgpu_check_n4.log
timeout 1200 $TR --nproc-per-node 4 --master-port 29522 bench.py --gpus 4 --steps 5 --warmup 3 > gpurun_out/r02/g10_bench_n4.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g10_bench_n4.log
timeout 600 $TR --nproc-per-node 4 --master-port 29523 bench.py --impl reference --gpus 4 --steps 3 --warmup 3 > gpurun_out/r02/g10_bench_ref_n4.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g10_bench_ref_n4.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-kernels --no-cpu > gpurun_out/r02/g10_bench_n1.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g10_bench_n1.log
