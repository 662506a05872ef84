// SGEMM for the slice-mapped matmul task: C[m,n] = A[m,k] . B[k,n], fp32.
//
// The reference cannot express matmul (reductions are a non-goal,
// SPEC.md:181); its planner still fixes the data distribution (slice(1) on A,
// slice(0) on B, one_to_one on C row slabs, model.py:209-231).  Two
// implementations:
//   * CQ_SGEMM_FFMA   -- SIMT fp32, 128x128x8 tiles, 8x8 outputs per thread,
//                        register double buffering.  Correctness anchor.
//   * CQ_SGEMM_3XTF32 -- tcgen05.mma kind::tf32 with the hi/lo split
//                        (a_hi*b_hi + a_hi*b_lo + a_lo*b_hi), see cq_tf32.cu.
#include "cq_common.cuh"

namespace cq {

constexpr int SG_BM = 128, SG_BN = 128, SG_BK = 8, SG_THREADS = 256;

template <bool kVec>
__global__ void __launch_bounds__(SG_THREADS) sgemm_ffma_kernel(const float* __restrict__ A, int64_t lda,
                                                                const float* __restrict__ B, int64_t ldb,
                                                                float* __restrict__ C, int64_t ldc, int64_t m,
                                                                int64_t n, int64_t k) {
  __shared__ __align__(16) float As[2][SG_BK][SG_BM];
  __shared__ __align__(16) float Bs[2][SG_BK][SG_BN];
  const int tid = threadIdx.x;
  const int64_t row0 = (int64_t)blockIdx.y * SG_BM, col0 = (int64_t)blockIdx.x * SG_BN;
  // global->smem assignment
  const int a_r = tid >> 1, a_k = (tid & 1) * 4;   // A: 128 rows x 8 k, 4 per thread
  const int b_k = tid >> 5, b_c = (tid & 31) * 4;  // B: 8 k x 128 cols, 4 per thread
  // compute assignment: 4+4 rows, 4+4 cols per thread
  const int ty = tid >> 4, tx = tid & 15;

  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;

  float ra[4], rb[4];
  auto load_tiles = [&](int64_t kk) {
    int64_t gr = row0 + a_r;
    if (kVec) {
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (gr < m && kk + a_k < k) v = *reinterpret_cast<const float4*>(A + gr * lda + kk + a_k);
      ra[0] = v.x; ra[1] = v.y; ra[2] = v.z; ra[3] = v.w;
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) ra[q] = (gr < m && kk + a_k + q < k) ? A[gr * lda + kk + a_k + q] : 0.f;
    }
    int64_t gk = kk + b_k, gc = col0 + b_c;
    if (kVec) {
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (gk < k && gc < n) v = *reinterpret_cast<const float4*>(B + gk * ldb + gc);
      rb[0] = v.x; rb[1] = v.y; rb[2] = v.z; rb[3] = v.w;
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) rb[q] = (gk < k && gc + q < n) ? B[gk * ldb + gc + q] : 0.f;
    }
  };
  auto store_tiles = [&](int buf) {
#pragma unroll
    for (int q = 0; q < 4; ++q) As[buf][a_k + q][a_r] = ra[q];
    *reinterpret_cast<float4*>(&Bs[buf][b_k][b_c]) = make_float4(rb[0], rb[1], rb[2], rb[3]);
  };

  load_tiles(0);
  store_tiles(0);
  __syncthreads();
  int buf = 0;
  for (int64_t kk = 0; kk < k; kk += SG_BK) {
    const bool more = kk + SG_BK < k;
    if (more) load_tiles(kk + SG_BK);
#pragma unroll
    for (int q = 0; q < SG_BK; ++q) {
      float4 a0 = *reinterpret_cast<const float4*>(&As[buf][q][ty * 4]);
      float4 a1 = *reinterpret_cast<const float4*>(&As[buf][q][64 + ty * 4]);
      float4 b0 = *reinterpret_cast<const float4*>(&Bs[buf][q][tx * 4]);
      float4 b1 = *reinterpret_cast<const float4*>(&Bs[buf][q][64 + tx * 4]);
      float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    if (more) {
      store_tiles(buf ^ 1);
      __syncthreads();
      buf ^= 1;
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    int64_t r = row0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + i - 4);
    if (r >= m) continue;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      int64_t c = col0 + h * 64 + tx * 4;
      if (kVec && c + 3 < n) {
        *reinterpret_cast<float4*>(C + r * ldc + c) =
            make_float4(acc[i][h * 4], acc[i][h * 4 + 1], acc[i][h * 4 + 2], acc[i][h * 4 + 3]);
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (c + j < n) C[r * ldc + c + j] = acc[i][h * 4 + j];
      }
    }
  }
}

int sgemm_3xtf32(int device, int stream, cudaStream_t st, int sm_count, const float* a, int64_t lda,
                 const float* b, int64_t ldb, float* c, int64_t ldc, int64_t m, int64_t n, int64_t k);

}  // namespace cq

using namespace cq;

extern "C" int cq_sgemm(int device, int stream, int variant, const float* a, int64_t lda, const float* b,
                        int64_t ldb, float* c, int64_t ldc, int64_t m, int64_t n, int64_t k) {
  CQ_TRY(ensure_device(device));
  cudaStream_t st = stream_of(device, stream);
  CQ_REQUIRE(st != nullptr, "bad stream %d", stream);
  CQ_CHECK_CUDA(cudaSetDevice(device));
  if (m <= 0 || n <= 0) return CQ_OK;
  if (variant == CQ_SGEMM_3XTF32) {
    return sgemm_3xtf32(device, stream, st, device_state(device)->sm_count, a, lda, b, ldb, c, ldc, m, n, k);
  }
  CQ_REQUIRE(variant == CQ_SGEMM_FFMA, "cq_sgemm: unknown variant %d", variant);
  dim3 grid((unsigned)((n + SG_BN - 1) / SG_BN), (unsigned)((m + SG_BM - 1) / SG_BM));
  bool vec = ((lda | ldb | ldc) % 4 == 0) && (((uintptr_t)a | (uintptr_t)b | (uintptr_t)c) % 16 == 0) &&
             (k % 4 == 0) && (n % 4 == 0);
  if (vec)
    sgemm_ffma_kernel<true><<<grid, SG_THREADS, 0, st>>>(a, lda, b, ldb, c, ldc, m, n, k);
  else
    sgemm_ffma_kernel<false><<<grid, SG_THREADS, 0, st>>>(a, lda, b, ldb, c, ldc, m, n, k);
  CQ_CHECK_LAUNCH();
  return CQ_OK;
}
