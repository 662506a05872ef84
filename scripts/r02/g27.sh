mkdir -p gpurun_out/r02
cd scripts/r02/micro && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/parts parts.cu && cd - && \
timeout 300 /tmp/parts > gpurun_out/r02/g27_parts.log 2>&1; echo "exit=$?" >> gpurun_out/r02/g27_parts.log
