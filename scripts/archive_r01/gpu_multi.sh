# usage: bash scripts/gpu_multi.sh N   (run on an N-GPU box)
N=${1:-2}
mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/topo_$N.txt 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
timeout 600 $TR --master-port 29511 scripts/mgpu_check.py > gpurun_out/mgpu_check_$N.log 2>&1; echo "exit=$?" >> gpurun_out/mgpu_check_$N.log
timeout 900 $TR --master-port 29512 bench.py --gpus $N --steps 3 --warmup 3 --sgemm-variants 3xtf32 > gpurun_out/bench_$N.log 2>&1; echo "exit=$?" >> gpurun_out/bench_$N.log
timeout 300 $TR --master-port 29513 bench.py --impl reference --gpus $N --steps 3 --warmup 3 > gpurun_out/bench_ref_$N.log 2>&1; echo "exit=$?" >> gpurun_out/bench_ref_$N.log
