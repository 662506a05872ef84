# round 2, call 8: V=8 / ring-resident level 0 variants of the KL=8 pass: parity + interleaved timing
mkdir -p gpurun_out/r02
PARITY_CFGS="8,59;8,56;8,62;4,59" timeout 1200 python scripts/r02/fused_ab.py > gpurun_out/r02/g08_fused_ab.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g08_fused_ab.log
