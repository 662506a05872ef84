# round 2, call 89 (2 GPUs): the 2-rank check with run_batch in both halo modes (NCCL default, peer forced),
# and the multi-rank GPU tests
mkdir -p gpurun_out/r02
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29591 \
  scripts/mgpu_check.py > gpurun_out/r02/g89_mgpu_check_n2.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g89_mgpu_check_n2.log
timeout 900 python -m pytest tests/test_gpu_multirank.py -m gpu -q > gpurun_out/r02/g89_multirank.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g89_multirank.log
grep -E "PASS|FAIL" gpurun_out/r02/g89_mgpu_check_n2.log | head -30; tail -n 2 gpurun_out/r02/g89_multirank.log
