# round 2, call 25 (4 GPUs): final multi-GPU records -- parity at 2 and 4 ranks, bench N=1/2/4 on one box, reference arm
mkdir -p gpurun_out/r02
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 $TR --nproc-per-node 4 --master-port 29541 scripts/mgpu_check.py > gpurun_out/r02/g25_mgpu_check_n4.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g25_mgpu_check_n4.log
timeout 600 $TR --nproc-per-node 2 --master-port 29542 scripts/mgpu_check.py > gpurun_out/r02/g25_mgpu_check_n2.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g25_mgpu_check_n2.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02/g25_bench_n1.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g25_bench_n1.log
timeout 1200 $TR --nproc-per-node 2 --master-port 29543 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r02/g25_bench_n2.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g25_bench_n2.log
timeout 1200 $TR --nproc-per-node 4 --master-port 29544 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/r02/g25_bench_n4.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g25_bench_n4.log
timeout 900 $TR --nproc-per-node 4 --master-port 29545 bench.py --impl reference --gpus 4 --steps 5 --warmup 3 > gpurun_out/r02/g25_bench_ref_n4.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g25_bench_ref_n4.log
