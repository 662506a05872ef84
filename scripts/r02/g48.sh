# round 2, call 48 (4 GPUs): final code on one 4-GPU box -- multi-rank parity at 4 ranks, bench N=1/2/4, reference arm N=4
mkdir -p gpurun_out/r02
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=COLL timeout 600 $TR --nproc-per-node 4 --master-port 29561 scripts/mgpu_check.py > gpurun_out/r02/g48_mgpu_check_n4.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g48_mgpu_check_n4.log
timeout 900 python bench.py > gpurun_out/r02/g48_bench_n1.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g48_bench_n1.log
timeout 1200 $TR --nproc-per-node 2 --master-port 29562 bench.py --gpus 2 > gpurun_out/r02/g48_bench_n2.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g48_bench_n2.log
timeout 1200 $TR --nproc-per-node 4 --master-port 29563 bench.py --gpus 4 > gpurun_out/r02/g48_bench_n4.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g48_bench_n4.log
timeout 900 $TR --nproc-per-node 4 --master-port 29564 bench.py --impl reference --gpus 4 > gpurun_out/r02/g48_bench_ref_n4.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g48_bench_ref_n4.log
