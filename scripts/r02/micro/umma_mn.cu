// One tcgen05.mma kind::tf32 (M=128, N=64, K=8) with A K-major and B either
// K-major (control) or MN-major under several descriptor encodings, against
// a CPU product: which encoding reads B straight from a [k, n] tile.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o umma_mn umma_mn.cu
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// byte offset of element (row r, col c) of a 128-byte-row SW128 block: 16-byte chunk index ^ (row % 8)
__device__ __forceinline__ int sw128(int r, int c) { return r * 128 + ((((c * 4) >> 4) ^ (r & 7)) << 4) + ((c * 4) & 15); }

__global__ void kern(const float* A, const float* B, float* C, int mode, uint32_t lbo, uint32_t sbo, int bmajor) {
  // A: 128 x 8 (K-major, rows of 32 floats = 128 B, 8-row groups 1 KB apart)
  // B: K-major control: 64 rows (n) x 8 k; MN-major: 8 k-rows x 64 n in two 32-column chunks
  __shared__ __align__(1024) uint8_t sa[128 * 128];
  __shared__ __align__(1024) uint8_t sb[4 * 1024 * 4];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int t = threadIdx.x;
  for (int i = t; i < (int)sizeof(sa) / 4; i += blockDim.x) reinterpret_cast<float*>(sa)[i] = 0.f;
  for (int i = t; i < (int)sizeof(sb) / 4; i += blockDim.x) reinterpret_cast<float*>(sb)[i] = 0.f;
  __syncthreads();
  for (int i = t; i < 128 * 8; i += blockDim.x) {
    int r = i / 8, c = i % 8;
    *reinterpret_cast<float*>(sa + (r / 8) * 1024 + sw128(r % 8, c)) = A[r * 8 + c];
  }
  for (int i = t; i < 8 * 64; i += blockDim.x) {
    int kr = i / 64, n = i % 64;
    float v = B[kr * 64 + n];
    if (!bmajor) {   // K-major: row n, col kr
      *reinterpret_cast<float*>(sb + (n / 8) * 1024 + sw128(n % 8, kr)) = v;
    } else {          // MN-major: chunk n/32 at (n/32) * chunk_stride, row kr, col n%32
      // SWIZZLE_128B_BASE32B atoms: 4 k-rows x 128 B, 32-byte chunks XORed with (row & 3);
      // atom (n/32, kr/4) at (n/32) * lbo + (kr/4) * sbo
      const int r = kr & 3, c = n % 32;
      const int off = (n / 32) * (int)lbo + (kr / 4) * (int)sbo + r * 128 + ((((c * 4) >> 5) ^ r) << 5) + ((c * 4) & 31);
      *reinterpret_cast<float*>(sb + off) = v;
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (t == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
  if (t < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(su32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tbase;
  if (t == 0) {
    uint64_t da = ((uint64_t)(su32(sa) & 0x3FFFF) >> 4) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) |
                  (2ull << 61);
    uint64_t db;
    if (!bmajor)
      db = ((uint64_t)(su32(sb) & 0x3FFFF) >> 4) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) |
           (2ull << 61);
    else
      db = ((uint64_t)(su32(sb) & 0x3FFFF) >> 4) | ((uint64_t)(lbo >> 4) << 16) | ((uint64_t)(sbo >> 4) << 32) |
           (1ull << 46) | ((uint64_t)mode << 61);
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (bmajor ? (1u << 16) : 0u) | ((64u >> 3) << 17) |
                           ((128u >> 4) << 24);
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
                 ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(0u));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
  }
  // wait for the MMA
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W_%=;\n}\n" ::"r"(su32(&bar))
               : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int w = t / 32, lane = t % 32;
  for (int h = 0; h < 4; ++h) {
    uint32_t r[16];
    const uint32_t addr = tmem + ((uint32_t)(w * 32) << 16) + (uint32_t)(h * 16);
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int q = 0; q < 16; ++q) C[(w * 32 + lane) * 64 + h * 16 + q] = __uint_as_float(r[q]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (t < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem));
}

int main() {
  const int M = 128, N = 64, K = 8;
  float hA[M * K], hB[K * N], hC[M * N], ref[M * N];
  for (int i = 0; i < M * K; ++i) hA[i] = (float)((i * 7 % 13) - 6);
  for (int i = 0; i < K * N; ++i) hB[i] = (float)((i * 5 % 11) - 5);
  for (int r = 0; r < M; ++r)
    for (int n = 0; n < N; ++n) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += (double)hA[r * K + k] * hB[k * N + n];
      ref[r * N + n] = (float)s;
    }
  float *dA, *dB, *dC;
  cudaMalloc(&dA, sizeof(hA));
  cudaMalloc(&dB, sizeof(hB));
  cudaMalloc(&dC, sizeof(hC));
  cudaMemcpy(dA, hA, sizeof(hA), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, sizeof(hB), cudaMemcpyHostToDevice);
  struct V { const char* name; int bmajor, chunk; uint32_t lbo, sbo; } vs[] = {  // chunk = layout type
      {"K-major control", 0, 0, 0, 0},
      {"MN B32 atoms, n fastest LBO=512 SBO=1024", 1, 1, 512, 1024},
      {"MN B32 atoms, k fastest LBO=1024 SBO=512", 1, 1, 1024, 512},
      {"MN B32 atoms, n fastest LBO=512 SBO=1024 t2", 1, 2, 512, 1024},
      {"MN B32 atoms, LBO=2048 SBO=512", 1, 1, 2048, 512},
      {"MN B32 atoms, LBO=512 SBO=2048", 1, 1, 512, 2048},
  };
  for (auto& v : vs) {
    cudaMemset(dC, 0xff, sizeof(hC));
    kern<<<1, 128>>>(dA, dB, dC, v.chunk, v.lbo, v.sbo, v.bmajor);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(hC, dC, sizeof(hC), cudaMemcpyDeviceToHost);
    double err = 0;
    int zeros = 0;
    for (int i = 0; i < M * N; ++i) {
      err = fmax(err, fabs((double)hC[i] - ref[i]));
      zeros += hC[i] == 0.f;
    }
    printf("%-40s %s max err %.3g zeros %d  C[0..3] %g %g %g %g ref %g %g %g %g\n", v.name, cudaGetErrorString(e), err, zeros,
           hC[0], hC[1], hC[2], hC[3], ref[0], ref[1], ref[2], ref[3]);
  }
  return 0;
}
