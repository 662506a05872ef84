# round 2, call 57 (4 GPUs): peer-memory halo rows at 4 ranks -- parity, timeline, bench N=1/2/4 (+ N=4 NCCL path), ref arm
mkdir -p gpurun_out/r02
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 $TR --nproc-per-node 4 --master-port 29631 scripts/mgpu_check.py > gpurun_out/r02/g57_mgpu_check_n4.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g57_mgpu_check_n4.log
timeout 300 $TR --nproc-per-node 4 --master-port 29632 scripts/r02/halo_timeline.py > gpurun_out/r02/g57_timeline_n4.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g57_timeline_n4.log
timeout 900 python bench.py > gpurun_out/r02/g57_bench_n1.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g57_bench_n1.log
timeout 1200 $TR --nproc-per-node 2 --master-port 29633 bench.py --gpus 2 > gpurun_out/r02/g57_bench_n2.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g57_bench_n2.log
timeout 1200 $TR --nproc-per-node 4 --master-port 29634 bench.py --gpus 4 > gpurun_out/r02/g57_bench_n4.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g57_bench_n4.log
CQ_WAVE_P2P=0 timeout 1200 $TR --nproc-per-node 4 --master-port 29635 bench.py --gpus 4 --no-kernels --no-cpu --no-energy > gpurun_out/r02/g57_bench_n4_nccl.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g57_bench_n4_nccl.log
timeout 900 $TR --nproc-per-node 4 --master-port 29636 bench.py --impl reference --gpus 4 > gpurun_out/r02/g57_bench_ref_n4.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g57_bench_ref_n4.log
