# round 2, call 49 (2 GPUs): per-pass device timeline of the fused wave at N=2 (interior, edges, halo exchange);
# e2e pipeline depth sweep at N=1
mkdir -p gpurun_out/r02
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 $TR --nproc-per-node 2 --master-port 29571 scripts/r02/halo_timeline.py > gpurun_out/r02/g49_timeline_n2.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g49_timeline_n2.log
timeout 600 python scripts/r02/e2e_depth.py > gpurun_out/r02/g49_e2e_depth.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g49_e2e_depth.log
