// 3xTF32 SGEMM on tcgen05 (placeholder until the tensor-core path lands).
#include "cq_common.cuh"

namespace cq {

int sgemm_3xtf32(cudaStream_t st, int sm_count, const float* a, int64_t lda, const float* b, int64_t ldb,
                 float* c, int64_t ldc, int64_t m, int64_t n, int64_t k) {
  (void)st; (void)sm_count; (void)a; (void)lda; (void)b; (void)ldb; (void)c; (void)ldc;
  (void)m; (void)n; (void)k;
  set_error("cq_sgemm: 3xTF32 variant not built yet");
  return CQ_ERR_UNSUPPORTED;
}

}  // namespace cq
