N=4
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
timeout 400 $TR --master-port 29511 scripts/mgpu_check.py > gpurun_out/mgpu_check_$N.log 2>&1; echo "exit=$?" >> gpurun_out/mgpu_check_$N.log
timeout 900 $TR --master-port 29512 bench.py --gpus $N --steps 3 --warmup 3 --sgemm-variants 3xtf32 > gpurun_out/bench_$N.log 2>&1; echo "exit=$?" >> gpurun_out/bench_$N.log
timeout 300 $TR --master-port 29513 bench.py --impl reference --gpus $N --steps 3 --warmup 3 > gpurun_out/bench_ref_$N.log 2>&1; echo "exit=$?" >> gpurun_out/bench_ref_$N.log
timeout 900 python -m pytest tests/test_gpu_multirank.py -q -x > gpurun_out/gpu_multirank_4gpu.log 2>&1; echo "exit=$?" >> gpurun_out/gpu_multirank_4gpu.log
