// Microbenchmark: throughput of the wave cell update's FP32 instruction mix
// on one SM sub-partition configuration (registers only, no memory), for
// variants of how the 7 operations per cell are packed (FP32x2 vs scalar).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fpmix fpmix.cu
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long f32x2;
__device__ __forceinline__ f32x2 pack2(float lo, float hi) { f32x2 r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi)); return r; }
__device__ __forceinline__ void unpack2(f32x2 v, float& lo, float& hi) { asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v)); }
__device__ __forceinline__ f32x2 add2(f32x2 a, f32x2 b) { f32x2 r; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ f32x2 mul2(f32x2 a, f32x2 b) { f32x2 r; asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ f32x2 fma2(f32x2 a, f32x2 b, f32x2 c) { f32x2 r; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }

template <int VAR>
__device__ __forceinline__ float4 cell(float4 m, float4 n, float4 s, float4 p, float wv, float ev, float c) {
  float a0, a1, b0, b1;
  if (VAR == 2) {  // n + s scalar
    a0 = __fadd_rn(n.x, s.x); a1 = __fadd_rn(n.y, s.y); b0 = __fadd_rn(n.z, s.z); b1 = __fadd_rn(n.w, s.w);
  } else {
    unpack2(add2(pack2(n.x, n.y), pack2(s.x, s.y)), a0, a1);
    unpack2(add2(pack2(n.z, n.w), pack2(s.z, s.w)), b0, b1);
  }
  a0 = __fadd_rn(__fadd_rn(a0, wv), m.y);
  a1 = __fadd_rn(__fadd_rn(a1, m.x), m.z);
  b0 = __fadd_rn(__fadd_rn(b0, m.y), m.w);
  b1 = __fadd_rn(__fadd_rn(b1, m.z), ev);
  const f32x2 uA = pack2(m.x, m.y), uB = pack2(m.z, m.w);
  const f32x2 m4 = pack2(-4.f, -4.f), two = pack2(2.f, 2.f);
  const f32x2 lapA = fma2(uA, m4, pack2(a0, a1)), lapB = fma2(uB, m4, pack2(b0, b1));
  const f32x2 tA = fma2(uA, two, pack2(-p.x, -p.y)), tB = fma2(uB, two, pack2(-p.z, -p.w));
  float l0, l1, l2, l3, t0, t1, t2, t3;
  if (VAR == 1) {  // c * lap scalar
    float q0, q1, q2, q3;
    unpack2(lapA, q0, q1); unpack2(lapB, q2, q3);
    l0 = __fmul_rn(c, q0); l1 = __fmul_rn(c, q1); l2 = __fmul_rn(c, q2); l3 = __fmul_rn(c, q3);
  } else {
    const f32x2 cc = pack2(c, c);
    unpack2(mul2(cc, lapA), l0, l1);
    unpack2(mul2(cc, lapB), l2, l3);
  }
  unpack2(tA, t0, t1);
  unpack2(tB, t2, t3);
  float4 o;
  o.x = __fadd_rn(t0, l0); o.y = __fadd_rn(t1, l1); o.z = __fadd_rn(t2, l2); o.w = __fadd_rn(t3, l3);
  return o;
}

// 8 levels of a 3-row window per warp, as the fused pass (no memory traffic)
template <int VAR>
__global__ void __launch_bounds__(32, 12) bench(float* out, int iters, float c) {
  const int lane = threadIdx.x;
  float4 L[8][3];
  float4 P[3];
#pragma unroll
  for (int j = 0; j < 8; ++j)
#pragma unroll
    for (int k = 0; k < 3; ++k) L[j][k] = make_float4(lane * 1e-3f + j, k * 1e-3f, 0.5f, 0.25f);
#pragma unroll
  for (int k = 0; k < 3; ++k) P[k] = make_float4(0.1f, 0.2f, 0.3f, k * 0.01f);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int sd = 0; sd < 3; ++sd) {
      const int s = sd, so = (sd + 1) % 3, sm = (sd + 2) % 3;
      L[0][s] = make_float4(L[0][so].y, L[0][so].x, L[0][sm].w, L[0][sm].z);  // new input row (cheap)
#pragma unroll
      for (int j = 1; j < 8; ++j) {
        const float4 mid = L[j - 1][sm];
        const float wv = __shfl_up_sync(0xffffffffu, mid.w, 1);
        const float ev = __shfl_down_sync(0xffffffffu, mid.x, 1);
        const float4 pp = j == 1 ? P[sm] : L[j - 2][so];
        L[j][s] = cell<VAR>(mid, L[j - 1][so], L[j - 1][s], pp, wv, ev, c);
      }
    }
  }
  float acc = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) acc += L[j][0].x + L[j][1].y + L[j][2].z;
  out[blockIdx.x * 32 + lane] = acc;
}

template <int VAR>
float run(float* d, int blocks, int iters) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  bench<VAR><<<blocks, 32>>>(d, 10, 0.25f);
  cudaEventRecord(a);
  bench<VAR><<<blocks, 32>>>(d, iters, 0.25f);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* d;
  cudaMalloc(&d, 1 << 24);
  const int iters = 2000;
  for (int wps : {4, 8, 12}) {
    const int blocks = sms * wps;
    for (int rep = 0; rep < 2; ++rep) {
      const double lvlrows = (double)blocks * iters * 3 * 7;  // warp level-rows
      float t0 = run<0>(d, blocks, iters), t1 = run<1>(d, blocks, iters), t2 = run<2>(d, blocks, iters);
      auto rate = [&](float ms) { return lvlrows / (ms * 1e-3) / (sms * 4) / 1.9e9; };  // level-rows per SMSP per cycle @1.9GHz
      printf("warps/SM %2d: base %.3f ms (%.1f cyc/level-row/SMSP)  scalar-mul %.3f ms (%.1f)  scalar-ns %.3f ms (%.1f)\n",
             wps, t0, 1 / rate(t0), t1, 1 / rate(t1), t2, 1 / rate(t2));
    }
  }
  return 0;
}
