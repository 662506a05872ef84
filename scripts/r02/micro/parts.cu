// Microbenchmark: which part of the fused wave pass's row loop costs what.
// The 8-level register-window math (FMA form) per input row, plus, by
// variant bit: 1 = the two ring reads (LDS) per row, 2 = the cp.async
// refill + commit + wait per row (from a small L2-resident buffer),
// 4 = the two streaming stores per row with the |x| max, 8 = unroll the
// ring by 6 rows (else 3).  Prints cycles per warp level-row per SMSP.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o parts parts.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
typedef unsigned long long f32x2;
__device__ __forceinline__ f32x2 pack2(float lo, float hi) { f32x2 r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi)); return r; }
__device__ __forceinline__ void unpack2(f32x2 v, float& lo, float& hi) { asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v)); }
__device__ __forceinline__ f32x2 add2(f32x2 a, f32x2 b) { f32x2 r; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ f32x2 mul2(f32x2 a, f32x2 b) { f32x2 r; asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ f32x2 fma2(f32x2 a, f32x2 b, f32x2 c) { f32x2 r; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }

__device__ __forceinline__ float4 cell(float4 m, float4 n, float4 s, float4 p, float wv, float ev, float c) {
  float a0, a1, b0, b1;
  unpack2(add2(pack2(n.x, n.y), pack2(s.x, s.y)), a0, a1);
  unpack2(add2(pack2(n.z, n.w), pack2(s.z, s.w)), b0, b1);
  a0 = __fadd_rn(__fadd_rn(a0, wv), m.y);
  a1 = __fadd_rn(__fadd_rn(a1, m.x), m.z);
  b0 = __fadd_rn(__fadd_rn(b0, m.y), m.w);
  b1 = __fadd_rn(__fadd_rn(b1, m.z), ev);
  const f32x2 uA = pack2(m.x, m.y), uB = pack2(m.z, m.w);
  const f32x2 m4 = pack2(-4.f, -4.f), two = pack2(2.f, 2.f);
  const f32x2 lapA = fma2(uA, m4, pack2(a0, a1)), lapB = fma2(uB, m4, pack2(b0, b1));
  const f32x2 tA = fma2(uA, two, pack2(-p.x, -p.y)), tB = fma2(uB, two, pack2(-p.z, -p.w));
  float l0, l1, l2, l3, t0, t1, t2, t3;
  const f32x2 cc = pack2(c, c);
  unpack2(mul2(cc, lapA), l0, l1);
  unpack2(mul2(cc, lapB), l2, l3);
  unpack2(tA, t0, t1);
  unpack2(tB, t2, t3);
  float4 o;
  o.x = __fadd_rn(t0, l0); o.y = __fadd_rn(t1, l1); o.z = __fadd_rn(t2, l2); o.w = __fadd_rn(t3, l3);
  return o;
}

__device__ __forceinline__ void cp16(void* smem, const void* g) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(g) : "memory");
}

template <int VAR, int SMODE = 0>
__global__ void __launch_bounds__(32, 12) bench(const float4* __restrict__ src, float4* __restrict__ dst, int iters,
                                                float c, float* amax_out) {
  constexpr int D = (VAR & 8) ? 6 : 3;
  __shared__ float4 ring[D][2][32];
  __shared__ __align__(128) float4 stage[2][2][32];   // SMODE 4: rows staged for a TMA bulk store
  __shared__ __align__(128) float4 stage5[2][D][2][32];  // SMODE 5: a turn of rows, double-buffered
  const int lane = threadIdx.x;
  float4 L[8][3];
  float4 P[3];
#pragma unroll
  for (int j = 0; j < 8; ++j)
#pragma unroll
    for (int k = 0; k < 3; ++k) L[j][k] = make_float4(lane * 1e-3f + j, k * 1e-3f, 0.5f, 0.25f);
#pragma unroll
  for (int k = 0; k < 3; ++k) P[k] = make_float4(0.1f, 0.2f, 0.3f, k * 0.01f);
#pragma unroll
  for (int k = 0; k < D; ++k) { ring[k][0][lane] = L[0][k % 3]; ring[k][1][lane] = P[k % 3]; }
  const float4* s = src + (blockIdx.x % 64) * 4096 + lane;   // 64 x 64 KB: L2-resident source rows
  float4* o = dst + (size_t)blockIdx.x * 1024 + lane;   // each warp its own 16 rows x 2 x 512 B
  float amax = 0.f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int sd = 0; sd < D; ++sd) {
      const int sl = sd % 3, so = (sd + 1) % 3, sm = (sd + 2) % 3;
      if (VAR & 2) asm volatile("cp.async.wait_group %0;" ::"n"(D - 1) : "memory");
      if (VAR & 1) {
        L[0][sl] = ring[sd][0][lane];
        P[sl] = ring[sd][1][lane];
      } else {
        L[0][sl] = make_float4(L[0][so].y, L[0][so].x, L[0][sm].w, L[0][sm].z);
      }
      if (VAR & 2) {
        const int r = (it * D + sd) & 63;
        cp16(&ring[sd][0][lane], s + r * 32);
        cp16(&ring[sd][1][lane], s + r * 32 + 2048);
        asm volatile("cp.async.commit_group;" ::: "memory");
      }
#pragma unroll
      for (int j = 1; j <= 8; ++j) {
        const float4 mid = L[j - 1][sm];
        const float wv = __shfl_up_sync(0xffffffffu, mid.w, 1);
        const float ev = __shfl_down_sync(0xffffffffu, mid.x, 1);
        const float4 pp = j == 1 ? P[sm] : L[j - 2][so];
        const float4 r = cell(mid, L[j - 1][so], L[j - 1][sl], pp, wv, ev, c);
        if (j < 8) L[j][sl] = r;
        if ((VAR & 4) && j >= 7) {
          const int row = (it * D + sd) & 15;
          float4* a = o + row * 32 + (j == 8 ? 512 : 0);
          if (SMODE == 0 || SMODE == 2) __stcs(a, r);
          if (SMODE == 1 || SMODE == 3) *a = r;
          if (SMODE == 6 && j == 8) __stcs(a, r);                       // one store per row
          if (SMODE == 7) stage[sd & 1][j == 8][lane] = r;              // shared-memory stores only
          if (SMODE == 8) {                                              // two 8-byte stores
            __stcs(reinterpret_cast<float2*>(a), make_float2(r.x, r.y));
            __stcs(reinterpret_cast<float2*>(a) + 1, make_float2(r.z, r.w));
          }
          if (SMODE == 4) {
            // stage the lane's 16 B, then one lane bulk-stores the 512-B row
            const int buf = sd & 1, k = j == 8;
            if (k == 0) asm volatile("cp.async.bulk.wait_group.read 2;" ::: "memory");
            stage[buf][k][lane] = r;
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
              const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(&stage[buf][k][0]));
              asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 512;" ::"l"(a - lane), "r"(sa)
                           : "memory");
              asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
          }
          if (SMODE == 5) stage5[it & 1][sd][j == 8][lane] = r;
          if (SMODE == 0 || SMODE == 1 || SMODE == 4 || SMODE == 5 || SMODE >= 6)
            amax = fmaxf(amax, fmaxf(fmaxf(fabsf(r.x), fabsf(r.y)), fmaxf(fabsf(r.z), fabsf(r.w))));
        }
      }
    }
    if ((VAR & 4) && SMODE == 5) {
      // the turn's 2 x D rows leave in bulk copies issued by one lane; the
      // other half of the staging buffer must have been read out before it
      // is rewritten next turn
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
#pragma unroll
        for (int sd = 0; sd < D; ++sd)
#pragma unroll
          for (int k = 0; k < 2; ++k) {
            const int row = (it * D + sd) & 15;
            const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(&stage5[it & 1][sd][k][0]));
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 512;" ::"l"(o - lane + row * 32 + k * 512),
                         "r"(sa) : "memory");
          }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
      __syncwarp();
    }
  }
  float acc = amax;
#pragma unroll
  for (int j = 0; j < 8; ++j) acc += L[j][0].x + L[j][1].y + L[j][2].z;
  amax_out[blockIdx.x * 32 + lane] = acc;
}

template <int VAR, int SMODE = 0>
void run(const float4* s, float4* d, float* a, int sms, int wps, int iters) {
  const int blocks = sms * wps;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  bench<VAR, SMODE><<<blocks, 32>>>(s, d, 4, 0.25f, a);
  cudaEventRecord(e0);
  bench<VAR, SMODE><<<blocks, 32>>>(s, d, iters, 0.25f, a);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  constexpr int D = (VAR & 8) ? 6 : 3;
  const double lvl = (double)blocks * iters * D * 8;
  int mhz = 0;
  cudaDeviceGetAttribute(&mhz, cudaDevAttrClockRate, 0);
  printf("variant %2d store mode %d (lds %d cp.async %d stores %d unroll %d) warps/SM %2d: %.3f ms, %.1f cycles per "
         "level-row per SMSP\n", VAR, SMODE, VAR & 1, (VAR >> 1) & 1, (VAR >> 2) & 1, D, wps, ms,
         ms * 1e-3 * (mhz * 1e3) * (sms * 4) / lvl);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float4 *s, *d;
  float* a;
  cudaMalloc(&s, 64 << 20);
  cudaMalloc(&d, (size_t)sms * 64 * 1024 * 16);
  cudaMalloc(&a, sms * 64 * 32 * sizeof(float));
  const int iters = 400;
  for (int rep = 0; rep < 2; ++rep) {
    run<13, 0>(s, d, a, sms, 12, iters);
    run<13, 6>(s, d, a, sms, 12, iters);
    run<13, 7>(s, d, a, sms, 12, iters);
    run<13, 8>(s, d, a, sms, 12, iters);
    run<9, 0>(s, d, a, sms, 12, iters);
    run<3>(s, d, a, sms, 12, iters * 2);
    run<7, 0>(s, d, a, sms, 12, iters * 2);
    run<7, 1>(s, d, a, sms, 12, iters * 2);
    run<7, 2>(s, d, a, sms, 12, iters * 2);
    run<7, 3>(s, d, a, sms, 12, iters * 2);
    run<7, 4>(s, d, a, sms, 12, iters * 2);
    run<7, 5>(s, d, a, sms, 12, iters * 2);
    run<15, 0>(s, d, a, sms, 12, iters);
    run<15, 5>(s, d, a, sms, 12, iters);
    run<8>(s, d, a, sms, 12, iters);
    run<9>(s, d, a, sms, 12, iters);
    run<11>(s, d, a, sms, 12, iters);
    run<13>(s, d, a, sms, 12, iters);
  }
  return 0;
}
