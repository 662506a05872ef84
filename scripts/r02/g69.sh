# round 2, call 69 (4 GPUs): final code -- GPU tests on 4 GPUs, multi-rank parity at 4 and 2 ranks, bench N=1/2/4, reference arm N=4
mkdir -p gpurun_out/r02
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02/g69_gpu_tests_4gpu.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g69_gpu_tests_4gpu.log
timeout 600 $TR --nproc-per-node 4 --master-port 29651 scripts/mgpu_check.py > gpurun_out/r02/g69_mgpu_check_n4.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g69_mgpu_check_n4.log
timeout 600 $TR --nproc-per-node 2 --master-port 29652 scripts/mgpu_check.py > gpurun_out/r02/g69_mgpu_check_n2.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g69_mgpu_check_n2.log
timeout 900 python bench.py > gpurun_out/r02/g69_bench_n1.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g69_bench_n1.log
timeout 1200 $TR --nproc-per-node 2 --master-port 29653 bench.py --gpus 2 > gpurun_out/r02/g69_bench_n2.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g69_bench_n2.log
timeout 1200 $TR --nproc-per-node 4 --master-port 29654 bench.py --gpus 4 > gpurun_out/r02/g69_bench_n4.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g69_bench_n4.log
timeout 900 $TR --nproc-per-node 4 --master-port 29655 bench.py --impl reference --gpus 4 > gpurun_out/r02/g69_bench_ref_n4.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g69_bench_ref_n4.log
