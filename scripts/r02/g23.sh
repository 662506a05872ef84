# round 2, call 23: ncu --set full of the SAXPY, N-body kick and 3xTF32 SGEMM kernels (current code)
mkdir -p gpurun_out/r02
for k in saxpy nbody sgemm; do
  case $k in saxpy) R=regex:saxpy_kernel;; nbody) R=regex:nbody_kick_kernel;; sgemm) R=regex:sgemm_3xtf32;; esac
  timeout 300 python scripts/r02/prof_kernels.py $k > gpurun_out/r02/g23_$k.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none -k $R -s 1 -c 1 -o gpurun_out/r02/$k python scripts/r02/prof_kernels.py $k >> gpurun_out/r02/g23_$k.log 2>&1
  echo "exit=$?" >> gpurun_out/r02/g23_$k.log
done
