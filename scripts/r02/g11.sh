# round 2, call 11: FP32-pipe microbenchmark of the wave cell mix (packed vs scalar variants)
mkdir -p gpurun_out/r02
cd scripts/r02/micro && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fpmix fpmix.cu && cd - && \
timeout 300 /tmp/fpmix > gpurun_out/r02/g11_fpmix.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g11_fpmix.log
# run_batch host timeline at N=1 (why e2e varies 59-125 ms per simulation between boxes)
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29531 scripts/batch_diag.py > gpurun_out/r02/g11_batch_diag.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g11_batch_diag.log
timeout 300 python scripts/pcie_duplex.py > gpurun_out/r02/g11_pcie.log 2>&1
nvidia-smi topo -m > gpurun_out/r02/g11_topo.txt 2>&1; lscpu > gpurun_out/r02/g11_lscpu.txt 2>&1; numactl -H >> gpurun_out/r02/g11_lscpu.txt 2>&1
