// libcq compute kernels for sm_100a.
//
// These replace the reference's per-cell Python evaluation
// (pkg/src/clusterq/simulator.py:151-158 -> kernel.py:291-331 eval_kernel,
// model.py:442-453 ReadView.read).  Arithmetic is performed with one
// rounding per DSL operator in the DSL's left-to-right tree order (no FMA
// contraction: explicit __*_rn intrinsics), so float64 results are
// bit-identical to the reference and float32 results are bit-identical to a
// binary32 restatement of the same tree.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "cq_common.cuh"

namespace cq {

// ------------------------------------------------------------ arithmetic
template <typename T> struct Ar;
template <> struct Ar<double> {
  static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
  static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
  static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
  static __device__ __forceinline__ double div(double a, double b, bool&) { return __ddiv_rn(a, b); }
  static __device__ __forceinline__ double neg(double a) { return -a; }
  static __device__ __forceinline__ double from_id(int64_t i) { return (double)i; }
  static __device__ __forceinline__ double from_bits(int64_t b) { return __longlong_as_double(b); }
};
template <> struct Ar<float> {
  static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
  static __device__ __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }
  static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
  static __device__ __forceinline__ float div(float a, float b, bool&) { return __fdiv_rn(a, b); }
  static __device__ __forceinline__ float neg(float a) { return -a; }
  static __device__ __forceinline__ float from_id(int64_t i) { return __ll2float_rn(i); }
  // constants arrive as binary64 bit patterns; round once to binary32
  static __device__ __forceinline__ float from_bits(int64_t b) { return __double2float_rn(__longlong_as_double(b)); }
};
// wrapping two's-complement int64, truncating division (kernel.py:275-288, 315-321)
template <> struct Ar<long long> {
  typedef unsigned long long U;
  static __device__ __forceinline__ long long add(long long a, long long b) { return (long long)((U)a + (U)b); }
  static __device__ __forceinline__ long long sub(long long a, long long b) { return (long long)((U)a - (U)b); }
  static __device__ __forceinline__ long long mul(long long a, long long b) { return (long long)((U)a * (U)b); }
  static __device__ __forceinline__ long long div(long long a, long long b, bool& fail) {
    if (b == 0) { fail = true; return 0; }
    U ua = a < 0 ? (U)0 - (U)a : (U)a;
    U ub = b < 0 ? (U)0 - (U)b : (U)b;
    U q = ua / ub;
    return (long long)(((a < 0) != (b < 0)) ? (U)0 - q : q);
  }
  static __device__ __forceinline__ long long neg(long long a) { return (long long)((U)0 - (U)a); }
  static __device__ __forceinline__ long long from_id(int64_t i) { return (long long)i; }
  static __device__ __forceinline__ long long from_bits(int64_t b) { return (long long)b; }
};

__device__ __forceinline__ int64_t view_off(const cq_view_t& v, int64_t p0, int64_t p1, int64_t p2) {
  return (p0 - v.alloc.lo[0]) * v.stride[0] + (p1 - v.alloc.lo[1]) * v.stride[1] +
         (p2 - v.alloc.lo[2]) * v.stride[2];
}

__device__ __forceinline__ int64_t clamp64(int64_t v, int64_t lo, int64_t hi_excl) {
  return v < lo ? lo : (v >= hi_excl ? hi_excl - 1 : v);
}

static inline int64_t box_volume(const cq_box_t& b) {
  int64_t v = 1;
  for (int k = 0; k < CQ_MAX_DIMS; ++k) v *= (b.hi[k] - b.lo[k]);
  return v;
}

static inline int grid_for(int64_t work, int threads, int sm_count, int per_sm) {
  int64_t g = (work + threads - 1) / threads;
  int64_t cap = (int64_t)sm_count * per_sm;
  if (g > cap) g = cap;
  return (int)(g < 1 ? 1 : g);
}

// First-error record: key = (row-major cell index << 4) | code, atomicMin.
__device__ void report_error(unsigned long long* flag, int code, int64_t lin, int64_t p0, int64_t p1,
                             int64_t p2) {
  unsigned long long key = ((unsigned long long)lin << 4) | (unsigned long long)code;
  unsigned long long old = atomicMin(flag, key);
  if (old > key) {
    long long* pt = (long long*)(flag + 1);
    pt[0] = p0;
    pt[1] = p1;
    pt[2] = p2;
  }
}

// ------------------------------------------------------- peer pass ordering
// One thread spins until every given slot (a local word a neighbour's
// p2p_signal_kernel writes) reaches *count; gives up after timeout_ns and
// records CQ_ERR_P2P in the sticky error flag rather than hang the stream.
__global__ void p2p_wait_kernel(const unsigned long long* slot0, const unsigned long long* slot1,
                                const unsigned long long* count, long long timeout_ns,
                                unsigned long long* flag) {
  const unsigned long long want = *count;
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (const unsigned long long* sl : {slot0, slot1}) {
    if (sl == nullptr) continue;
    while (true) {
      unsigned long long v;
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(sl) : "memory");
      if (v >= want) break;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if ((long long)(t - t0) > timeout_ns) {
        report_error(flag, CQ_ERR_P2P, 0, (int64_t)want, (int64_t)v, 0);
        return;
      }
      __nanosleep(64);
    }
  }
}

__global__ void p2p_signal_kernel(unsigned long long* count, unsigned long long* peer0,
                                  unsigned long long* peer1) {
  const unsigned long long v = *count + 1;
  *count = v;
  __threadfence_system();  // the pass's stores and copies before the signal
  if (peer0) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(peer0), "l"(v) : "memory");
  if (peer1) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(peer1), "l"(v) : "memory");
}

// ------------------------------------------------------------------- fill
template <typename T>
__global__ void fill_kernel(cq_view_t dst, cq_box_t box, cq_box_t extent, int mode, T value) {
  int64_t n1 = box.hi[1] - box.lo[1], n2 = box.hi[2] - box.lo[2];
  int64_t total = (box.hi[0] - box.lo[0]) * n1 * n2;
  int64_t e1 = extent.hi[1] - extent.lo[1], e2 = extent.hi[2] - extent.lo[2];
  T* out = (T*)dst.ptr;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t i2 = t % n2, r = t / n2;
    int64_t i1 = r % n1, i0 = r / n1;
    int64_t p0 = box.lo[0] + i0, p1 = box.lo[1] + i1, p2 = box.lo[2] + i2;
    T v;
    if (mode == 1) v = Ar<T>::from_id((p0 * e1 + p1) * e2 + p2);
    else v = value;
    out[view_off(dst, p0, p1, p2)] = v;
  }
}

// ------------------------------------------------------------------ SAXPY
// 16-byte vector loads/stores, grid-stride; one rounding per operator.
template <typename T>
__global__ void __launch_bounds__(256) saxpy_kernel(T alpha, const T* __restrict__ x,
                                                    const T* __restrict__ y, T* __restrict__ z,
                                                    int64_t n) {
  constexpr int V = 16 / sizeof(T);
  typedef typename std::conditional<sizeof(T) == 4, float4, double2>::type Vec;
  int64_t nv = n / V;
  const Vec* xv = reinterpret_cast<const Vec*>(x);
  const Vec* yv = reinterpret_cast<const Vec*>(y);
  Vec* zv = reinterpret_cast<Vec*>(z);
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  // two independent vectors in flight per thread
  for (; t + stride < nv; t += 2 * stride) {
    Vec a0 = __ldcs(xv + t), b0 = __ldcs(yv + t);
    Vec a1 = __ldcs(xv + t + stride), b1 = __ldcs(yv + t + stride);
    T* pa0 = reinterpret_cast<T*>(&a0);
    T* pb0 = reinterpret_cast<T*>(&b0);
    T* pa1 = reinterpret_cast<T*>(&a1);
    T* pb1 = reinterpret_cast<T*>(&b1);
#pragma unroll
    for (int k = 0; k < V; ++k) {
      pa0[k] = Ar<T>::add(Ar<T>::mul(alpha, pa0[k]), pb0[k]);
      pa1[k] = Ar<T>::add(Ar<T>::mul(alpha, pa1[k]), pb1[k]);
    }
    __stcs(zv + t, a0);
    __stcs(zv + t + stride, a1);
  }
  for (; t < nv; t += stride) {
    Vec a0 = __ldcs(xv + t), b0 = __ldcs(yv + t);
    T* pa0 = reinterpret_cast<T*>(&a0);
    T* pb0 = reinterpret_cast<T*>(&b0);
#pragma unroll
    for (int k = 0; k < V; ++k) pa0[k] = Ar<T>::add(Ar<T>::mul(alpha, pa0[k]), pb0[k]);
    __stcs(zv + t, a0);
  }
  int64_t tail = nv * V + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (tail < n) z[tail] = Ar<T>::add(Ar<T>::mul(alpha, x[tail]), y[tail]);
}

__global__ void saxpy_i64_kernel(long long alpha, const long long* x, const long long* y, long long* z,
                                 int64_t n) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    z[t] = Ar<long long>::add(Ar<long long>::mul(alpha, x[t]), y[t]);
}

// ---------------------------------------------------------------- wave 5pt
// out = ((k2*u) - upr) + (c*((((uN + uS) + uW) + uE) - (k4*u)))   [DSL tree]
template <typename T>
__device__ __forceinline__ T wave_cell(T u, T upr, T n, T s, T w, T e, T c, T k2, T k4) {
  typedef Ar<T> A;
  T lap = A::sub(A::add(A::add(A::add(n, s), w), e), A::mul(k4, u));
  return A::add(A::sub(A::mul(k2, u), upr), A::mul(c, lap));
}

// Vectorised row-marching kernel.  A thread owns V consecutive columns and
// walks RB rows downwards keeping rows r-1, r, r+1 of u in registers, so u is
// read from DRAM once per cell (12 B/cell/step for f32: u, upr, out).  West/
// east neighbours come from adjacent lanes by shuffle; warp-edge lanes fetch
// one extra scalar (an L1 hit).  Requirements (host-checked): the box spans
// whole rows [0, W) of the innermost axis, W % V == 0, views 16-B aligned
// with row pitch % V == 0.
template <typename T, int RB>
__global__ void __launch_bounds__(256) wave5_rows_kernel(cq_view_t u, cq_view_t upr, cq_view_t out,
                                                         int64_t row_lo, int64_t row_hi, int64_t H,
                                                         int64_t W, T c, T k2, T k4) {
  constexpr int V = 16 / sizeof(T);
  typedef typename std::conditional<sizeof(T) == 4, float4, double2>::type Vec;
  const int lane = threadIdx.x & 31;
  const int64_t col = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * V;
  const int64_t r0 = row_lo + (int64_t)blockIdx.y * RB;
  if (r0 >= row_hi) return;
  const int64_t r1 = min(r0 + (int64_t)RB, row_hi);
  const bool active = col < W;
  const int64_t cc = active ? col : 0;
  const T* ub = (const T*)u.ptr;
  const T* pb = (const T*)upr.ptr;
  T* ob = (T*)out.ptr;
  const int64_t us = u.stride[1], ps = upr.stride[1], os = out.stride[1];
  // rows live on axis 1, columns on axis 2 (leading axis 0 is [0,1))
  auto urow = [&](int64_t r) -> const T* {
    r = clamp64(r, 0, H);
    return ub + (r - u.alloc.lo[1]) * us + (cc - u.alloc.lo[2]);
  };
  Vec vm = *reinterpret_cast<const Vec*>(urow(r0 - 1));
  Vec vc = *reinterpret_cast<const Vec*>(urow(r0));
  const bool west_edge = (lane == 0);
  const bool east_edge = (lane == 31) || (col + V >= W);
  for (int64_t r = r0; r < r1; ++r) {
    Vec vn = *reinterpret_cast<const Vec*>(urow(r + 1));
    const T* prow = pb + (r - upr.alloc.lo[1]) * ps + (cc - upr.alloc.lo[2]);
    Vec vp = *reinterpret_cast<const Vec*>(prow);
    const T* cur = reinterpret_cast<const T*>(&vc);
    const T* up_ = reinterpret_cast<const T*>(&vm);
    const T* dn = reinterpret_cast<const T*>(&vn);
    const T* pr = reinterpret_cast<const T*>(&vp);
    // west neighbour of element 0, east neighbour of element V-1
    T wnb = __shfl_up_sync(0xffffffffu, cur[V - 1], 1);
    T enb = __shfl_down_sync(0xffffffffu, cur[0], 1);
    const T* crow = urow(r);
    if (west_edge) wnb = (cc == 0) ? cur[0] : crow[-1];
    if (east_edge) enb = (cc + V >= W) ? cur[V - 1] : crow[V];
    Vec vo;
    T* o = reinterpret_cast<T*>(&vo);
#pragma unroll
    for (int k = 0; k < V; ++k) {
      T w = (k == 0) ? wnb : cur[k - 1];
      T e = (k == V - 1) ? enb : cur[k + 1];
      o[k] = wave_cell<T>(cur[k], pr[k], up_[k], dn[k], w, e, c, k2, k4);
    }
    if (active) *reinterpret_cast<Vec*>(ob + (r - out.alloc.lo[1]) * os + (cc - out.alloc.lo[2])) = vo;
    vm = vc;
    vc = vn;
  }
}

// Generic per-cell fallback for any box / alignment.
template <typename T>
__global__ void wave5_cell_kernel(cq_view_t u, cq_view_t upr, cq_view_t out, cq_box_t box,
                                  int64_t H, int64_t W, T c, T k2, T k4) {
  int64_t n1 = box.hi[1] - box.lo[1], n2 = box.hi[2] - box.lo[2];
  int64_t total = (box.hi[0] - box.lo[0]) * n1 * n2;
  const T* ub = (const T*)u.ptr;
  const T* pb = (const T*)upr.ptr;
  T* ob = (T*)out.ptr;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t j = box.lo[2] + t % n2, r = t / n2;
    int64_t i = box.lo[1] + r % n1, p0 = box.lo[0] + r / n1;
    int64_t im = clamp64(i - 1, 0, H), ip = clamp64(i + 1, 0, H);
    int64_t jm = clamp64(j - 1, 0, W), jp = clamp64(j + 1, 0, W);
    T uc = ub[view_off(u, p0, i, j)];
    T v = wave_cell<T>(uc, pb[view_off(upr, p0, i, j)], ub[view_off(u, p0, im, j)],
                       ub[view_off(u, p0, ip, j)], ub[view_off(u, p0, i, jm)],
                       ub[view_off(u, p0, i, jp)], c, k2, k4);
    ob[view_off(out, p0, i, j)] = v;
  }
}

// ------------------------------------------------------- expression kernel
template <typename T>
__device__ __forceinline__ T load_as(const cq_view_t& v, int kind, int64_t off) {
  if (kind == CQ_F64) return (T)((const double*)v.ptr)[off];
  if (kind == CQ_F32) return (T)((const float*)v.ptr)[off];
  return (T)((const long long*)v.ptr)[off];
}

template <typename T>
__global__ void __launch_bounds__(128) expr_kernel(const __grid_constant__ cq_expr_t X,
                                                   unsigned long long* flag) {
  int64_t n1 = X.box.hi[1] - X.box.lo[1], n2 = X.box.hi[2] - X.box.lo[2];
  int64_t total = (X.box.hi[0] - X.box.lo[0]) * n1 * n2;
  const int kdims = X.dims;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t p[3];
    p[2] = X.box.lo[2] + t % n2;
    int64_t r = t / n2;
    p[1] = X.box.lo[1] + r % n1;
    p[0] = X.box.lo[0] + r / n1;
    T results[CQ_EXPR_MAX_OUT];
    bool failed = false;
    for (int o = 0; o < X.n_out; ++o) {
      T stack[32];
      int sp = 0;
      for (int pc = X.out_code_begin[o]; pc < X.out_code_end[o]; ++pc) {
        int op = X.code_op[pc], arg = X.code_arg[pc];
        switch (op) {
          case 0: stack[sp++] = Ar<T>::from_bits(X.consts[arg]); break;
          case 1: stack[sp++] = Ar<T>::from_id(p[arg]); break;
          case 2: {
            int vi = X.slot_view[arg];
            const cq_view_t& v = X.views[vi];
            int bd = X.view_dims[vi];
            int64_t q[3] = {0, 0, 0};
            for (int j = 0; j < bd; ++j) {
              int64_t x = p[3 - kdims + j] + X.slot_off[arg][j];
              int ax = 3 - bd + j;
              q[ax] = clamp64(x, X.view_extent[vi].lo[ax], X.view_extent[vi].hi[ax]);
            }
            int nchk = X.view_n_check[vi];
            if (nchk > 0) {
              bool inside = false;
              for (int b = 0; b < nchk && !inside; ++b) {
                const cq_box_t& cb = X.view_check[vi][b];
                inside = q[0] >= cb.lo[0] && q[0] < cb.hi[0] && q[1] >= cb.lo[1] && q[1] < cb.hi[1] &&
                         q[2] >= cb.lo[2] && q[2] < cb.hi[2];
              }
              if (!inside) {
                report_error(flag, CQ_ERR_MAPPER, t, p[0], p[1], p[2]);
                failed = true;
                stack[sp++] = (T)0;
                break;
              }
            }
            stack[sp++] = load_as<T>(v, X.kind, view_off(v, q[0], q[1], q[2]));
            break;
          }
          case 3: stack[sp - 1] = Ar<T>::neg(stack[sp - 1]); break;
          default: {
            T b = stack[--sp];
            T a = stack[sp - 1];
            T res;
            if (op == 4) res = Ar<T>::add(a, b);
            else if (op == 5) res = Ar<T>::sub(a, b);
            else if (op == 6) res = Ar<T>::mul(a, b);
            else {
              bool dz = false;
              res = Ar<T>::div(a, b, dz);
              if (dz) {
                report_error(flag, CQ_ERR_EVAL, t, p[0], p[1], p[2]);
                failed = true;
              }
            }
            stack[sp - 1] = res;
          }
        }
      }
      results[o] = stack[0];
    }
    if (failed) continue;
    for (int o = 0; o < X.n_out; ++o) {
      const cq_view_t& v = X.out[o];
      int64_t off = view_off(v, p[0], p[1], p[2]);
      if (X.kind == CQ_F64) ((double*)v.ptr)[off] = (double)results[o];
      else if (X.kind == CQ_F32) ((float*)v.ptr)[off] = (float)results[o];
      else ((long long*)v.ptr)[off] = (long long)results[o];
    }
  }
}

// ------------------------------------------------------------------ N-body
// Block = 8 warps x 32 lanes; a lane owns NB_IPT i-bodies, so a block covers
// 32*NB_IPT i-bodies and its 8 warps split the j range into 8 fixed slices
// of [0, n) (independent of the i partition, so results are bit-identical
// for any GPU count).  Each warp stages 32 j-bodies per tile in shared
// memory and every lane reads them back by broadcast (LDS.128); partial
// accelerations are summed over the warps in fixed order.
constexpr int NB_WARPS = 8;

// r2 >= eps2 > 0, so the flush-to-zero approximate reciprocal square root
// needs no denormal guard: one MUFU.RSQ per interaction.
__device__ __forceinline__ float rsqrt_ftz(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Blackwell packed FP32 (FADD2/FMUL2/FFMA2): each instruction applies the
// same IEEE round-to-nearest operation to two independent lanes, so a lane
// pair of i-bodies costs half the issue slots with per-body results identical
// to the scalar formulation.
typedef unsigned long long f32x2;

__device__ __forceinline__ f32x2 pack2(float lo, float hi) {
  f32x2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void unpack2(f32x2 v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ f32x2 add2(f32x2 a, f32x2 b) {
  f32x2 r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f32x2 sub2(f32x2 a, f32x2 b) {
  f32x2 r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f32x2 mul2(f32x2 a, f32x2 b) {
  f32x2 r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f32x2 fma2(f32x2 a, f32x2 b, f32x2 c) {
  f32x2 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}

// one j-body (duplicated into both lanes) against a pair of i-bodies:
//   d = p_j - p_i; r2 = d.d + eps2; s = m_j * (inv*inv*inv), inv = rsqrt(r2)
//   a += d * s          (20 flop / interaction by the GPU Gems convention)
__device__ __forceinline__ void nb_interact2(f32x2 pix, f32x2 piy, f32x2 piz, f32x2 jx, f32x2 jy, f32x2 jz,
                                             f32x2 jm, f32x2 eps2, f32x2& ax, f32x2& ay, f32x2& az) {
  f32x2 dx = sub2(jx, pix), dy = sub2(jy, piy), dz = sub2(jz, piz);
  f32x2 r2 = fma2(dx, dx, fma2(dy, dy, fma2(dz, dz, eps2)));
  float rl, rh;
  unpack2(r2, rl, rh);
  f32x2 inv = pack2(rsqrt_ftz(rl), rsqrt_ftz(rh));
  f32x2 s = mul2(jm, mul2(mul2(inv, inv), inv));
  ax = fma2(dx, s, ax);
  ay = fma2(dy, s, ay);
  az = fma2(dz, s, az);
}

// NP = i-body pairs per lane (independent FFMA2 chains); a block covers
// 64*NP i-bodies.
// The j range [0, n) is cut into NB_JCOLS * NB_WARPS fixed slices: j column
// c = col0 + blockIdx.y owns NB_WARPS consecutive slices, one per warp.
// Each block writes its per-body partial (sum over its warps, fixed order)
// to part_out[c]; nbody_kick_finalize sums the columns in fixed order and
// applies the kick.  The slicing depends only on n, never on the i range,
// so a body's acceleration is bit-identical for any GPU count, and the extra
// grid dimension keeps every SM busy when each GPU owns few i-bodies.
constexpr int NB_JCOLS = 8;

template <int NP>
__global__ void __launch_bounds__(NB_WARPS * 32) nbody_kick_kernel(const float4* __restrict__ pos,
                                                                   int64_t n, float* __restrict__ part_out,
                                                                   int64_t i_lo, int64_t i_hi, float eps2,
                                                                   int col0) {
  constexpr int NB_IBLOCK = 64 * NP;
  // j tile, each body duplicated for the packed lanes: (x,x,y,y), (z,z,m,m)
  __shared__ __align__(16) float4 tile[NB_WARPS][32][2];
  __shared__ float part[NB_WARPS][3][NB_IBLOCK];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t ibase = i_lo + (int64_t)blockIdx.x * NB_IBLOCK;
  f32x2 px[NP], py[NP], pz[NP], ax[NP], ay[NP], az[NP];
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    int64_t i0 = ibase + lane + 32 * (2 * p), i1 = i0 + 32;
    float4 a = pos[i0 < i_hi ? i0 : i_hi - 1];
    float4 b = pos[i1 < i_hi ? i1 : i_hi - 1];
    px[p] = pack2(a.x, b.x);
    py[p] = pack2(a.y, b.y);
    pz[p] = pack2(a.z, b.z);
    ax[p] = ay[p] = az[p] = 0ull;
  }
  const f32x2 e2 = pack2(eps2, eps2);
  const int col = col0 + blockIdx.y;  // j column of this block
  const int64_t slice = (int64_t)col * NB_WARPS + warp;
  constexpr int64_t kSlices = (int64_t)NB_JCOLS * NB_WARPS;
  const int64_t jb = (n * slice) / kSlices, je = (n * (slice + 1)) / kSlices;
  float4 next = (jb + lane < je) ? pos[jb + lane] : make_float4(0.f, 0.f, 0.f, 0.f);
  for (int64_t j0 = jb; j0 < je; j0 += 32) {
    tile[warp][lane][0] = make_float4(next.x, next.x, next.y, next.y);
    tile[warp][lane][1] = make_float4(next.z, next.z, next.w, next.w);
    __syncwarp();
    int64_t jn = j0 + 32 + lane;
    next = (jn < je) ? pos[jn] : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 8
    for (int k = 0; k < 32; ++k) {
      const ulonglong2 xy = *reinterpret_cast<const ulonglong2*>(&tile[warp][k][0]);
      const ulonglong2 zm = *reinterpret_cast<const ulonglong2*>(&tile[warp][k][1]);
#pragma unroll
      for (int p = 0; p < NP; ++p)
        nb_interact2(px[p], py[p], pz[p], xy.x, xy.y, zm.x, zm.y, e2, ax[p], ay[p], az[p]);
    }
    __syncwarp();
  }
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    float lo, hi;
    unpack2(ax[p], lo, hi);
    part[warp][0][lane + 64 * p] = lo;
    part[warp][0][lane + 64 * p + 32] = hi;
    unpack2(ay[p], lo, hi);
    part[warp][1][lane + 64 * p] = lo;
    part[warp][1][lane + 64 * p + 32] = hi;
    unpack2(az[p], lo, hi);
    part[warp][2][lane + 64 * p] = lo;
    part[warp][2][lane + 64 * p + 32] = hi;
  }
  __syncthreads();
  const int64_t count = i_hi - i_lo;
  for (int t = threadIdx.x; t < NB_IBLOCK; t += blockDim.x) {
    int64_t i = ibase + t;
    if (i < i_hi) {
      float sx = 0.f, sy = 0.f, sz = 0.f;
#pragma unroll
      for (int w = 0; w < NB_WARPS; ++w) {
        sx += part[w][0][t];
        sy += part[w][1][t];
        sz += part[w][2][t];
      }
      float* o = part_out + ((int64_t)col * count + (i - i_lo)) * 3;
      o[0] = sx;
      o[1] = sy;
      o[2] = sz;
    }
  }
}

// v_i += dt * sum over the NB_JCOLS column partials, in column order.
__global__ void nbody_kick_finalize(const float* __restrict__ part, const float4* vel_in, float4* vel,
                                    int64_t count, float dt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    float sx = 0.f, sy = 0.f, sz = 0.f;
#pragma unroll
    for (int c = 0; c < NB_JCOLS; ++c) {
      const float* p = part + ((int64_t)c * count + i) * 3;
      sx += p[0];
      sy += p[1];
      sz += p[2];
    }
    float4 v = vel_in[i];
    v.x = fmaf(dt, sx, v.x);
    v.y = fmaf(dt, sy, v.y);
    v.z = fmaf(dt, sz, v.z);
    vel[i] = v;
  }
}

__global__ void nbody_drift_kernel(const float4* p_in, const float4* __restrict__ v, float4* p,
                                   int64_t count, float dt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    float4 a = p_in[i], b = v[i];
    a.x = fmaf(dt, b.x, a.x);
    a.y = fmaf(dt, b.y, a.y);
    a.z = fmaf(dt, b.z, a.z);
    p[i] = a;
  }
}

// ---------------------------------------------- wave 5pt, KL steps per pass
// Temporal blocking of the wave ping-pong: from X(t) (u) and X(t-1) (upr)
// one pass computes X(t+1) .. X(t+KL) on chip and writes only X(t+KL)
// (out_last) and X(t+KL-1) (out_prev): 16 B/cell per KL steps instead of
// 12 B/cell per step.  Every intermediate cell is the same DSL tree with the
// same operands as the one-step kernel (wave_cell order, one rounding per
// operator; packed FP32x2 lanes are per-lane IEEE RN), so the result is
// bit-identical to KL launches of wave5_rows_kernel.
//
// A warp owns a strip of 32*V loaded columns (lane = V columns) and emits
// the middle 32*V - 2*KL: level j is exact on columns [j, 32V-j) of the
// strip (west/east neighbours by shuffle; the strip edge loses one column per
// level).  It marches a piece of rows [r0, r1), loading rows [r0-KL, r1+KL) of the
// inputs, keeping a 3-row window per level in registers (slot = row mod 3)
// and a D-row prefetch ring (loop unrolled by lcm so every slot index is
// static).  Global borders clamp exactly like the DSL's ReadView (the border
// cell reads itself).  Rows outside [in_lo, in_hi) are not read; the caller
// keeps [out_lo, out_hi) inside the trapezoid they determine.
template <typename T, int V> struct FVec;
template <> struct FVec<float, 2> { typedef float2 T; };
template <> struct FVec<float, 4> { typedef float4 T; };
template <> struct FVec<double, 2> { typedef double2 T; };

__device__ __forceinline__ double first_of(double2 v) { return v.x; }
__device__ __forceinline__ double last_of(double2 v) { return v.y; }
__device__ __forceinline__ float first_of(float2 v) { return v.x; }
__device__ __forceinline__ float last_of(float2 v) { return v.y; }
__device__ __forceinline__ float first_of(float4 v) { return v.x; }
__device__ __forceinline__ float last_of(float4 v) { return v.w; }

// ptxas contracts mul.rn.f32x2 feeding add/sub.rn.f32x2 into FFMA2 (even
// with .rn and --fmad=false), which would skip a rounding of the DSL tree.
// So no packed product ever feeds a packed add: the body's k2 = 2 and k4 = 4
// products are formed as exact sums (u+u == fl(2u), 2u+2u == fl(4u), also
// for subnormals and overflow), and c*lap is two scalar __fmul_rn (float2
// path) or a packed mul whose halves feed scalar adds, which ptxas leaves
// alone (float4 path; the SASS of the fused kernels has no scalar FFMA).
// (Forming the product as fma(c, x, -0) to keep the final add packed does
// not work: ptxas drops the -0 addend and contracts again.)
__device__ __forceinline__ f32x2 wave_pair(f32x2 u, f32x2 n, f32x2 s, f32x2 w, f32x2 e, f32x2 p, float c) {
  const f32x2 u2 = add2(u, u), u4 = add2(u2, u2);
  const f32x2 lap = sub2(add2(add2(add2(n, s), w), e), u4);
  float l0, l1;
  unpack2(lap, l0, l1);
  return add2(sub2(u2, p), pack2(__fmul_rn(c, l0), __fmul_rn(c, l1)));
}

__device__ __forceinline__ float2 wave_vec(float2 m, float2 n, float2 s, float2 p, float wv, float ev, float c) {
  const f32x2 o = wave_pair(pack2(m.x, m.y), pack2(n.x, n.y), pack2(s.x, s.y), pack2(wv, m.x), pack2(m.y, ev),
                            pack2(p.x, p.y), c);
  float2 r;
  unpack2(o, r.x, r.y);
  return r;
}

// float64 (the reference's own element kind): scalar DADD/DMUL, which ptxas
// does not contract
__device__ __forceinline__ double2 wave_vec(double2 m, double2 n, double2 s, double2 p, double wv, double ev,
                                            double c) {
  double2 o;
  o.x = wave_cell<double>(m.x, p.x, n.x, s.x, wv, m.y, c, 2.0, 4.0);
  o.y = wave_cell<double>(m.y, p.y, n.y, s.y, m.x, ev, c, 2.0, 4.0);
  return o;
}

__device__ __forceinline__ float4 wave_vec(float4 m, float4 n, float4 s, float4 p, float wv, float ev, float c) {
  // n + s on the aligned halves of the float4s (packed, no register moves);
  // + w and + e as scalar adds on the lanes' own registers (the neighbour
  // pairs (w, x), (y, z), (w, e) straddle the register pairs); the rest packed
  const f32x2 nsA = add2(pack2(n.x, n.y), pack2(s.x, s.y));
  const f32x2 nsB = add2(pack2(n.z, n.w), pack2(s.z, s.w));
  float a0, a1, b0, b1;
  unpack2(nsA, a0, a1);
  unpack2(nsB, b0, b1);
  a0 = __fadd_rn(__fadd_rn(a0, wv), m.y);
  a1 = __fadd_rn(__fadd_rn(a1, m.x), m.z);
  b0 = __fadd_rn(__fadd_rn(b0, m.y), m.w);
  b1 = __fadd_rn(__fadd_rn(b1, m.z), ev);
  const f32x2 uA = pack2(m.x, m.y), uB = pack2(m.z, m.w);
  const f32x2 u2A = add2(uA, uA), u2B = add2(uB, uB);
  const f32x2 lapA = sub2(pack2(a0, a1), add2(u2A, u2A));
  const f32x2 lapB = sub2(pack2(b0, b1), add2(u2B, u2B));
  const f32x2 tA = sub2(u2A, pack2(p.x, p.y)), tB = sub2(u2B, pack2(p.z, p.w));
  // c*lap packed, added as scalars (not contracted: see wave_vec_fast)
  const f32x2 cc = pack2(c, c);
  float l0, l1, l2, l3;
  unpack2(mul2(cc, lapA), l0, l1);
  unpack2(mul2(cc, lapB), l2, l3);
  float t0, t1, t2, t3;
  unpack2(tA, t0, t1);
  unpack2(tB, t2, t3);
  float4 o;
  o.x = __fadd_rn(t0, l0);
  o.y = __fadd_rn(t1, l1);
  o.z = __fadd_rn(t2, l2);
  o.w = __fadd_rn(t3, l3);
  return o;
}

// Fast form of the same tree for fields known to be bounded: while 4u and
// 2u do not overflow (|u| < 2^125), fl(4u) and fl(2u) are exact, so
//   fl(sum - fl(4u)) == fma(-4, u, sum)        (one rounding of the same sum)
//   fl(fl(2u) - p)   == fma(2, u, -p)          (likewise)
// with the same signed zero on exact cancellation, since an FMA's zero sum
// follows the rules of addition.  (The sign-symmetric -fma(-2, u, p) is
// equal only for non-zero results: it turns t = +0 into -0, and +0 + (-0)
// differs from -0 - (+0) when c*lap is -0.)
// -- bit-identical, 7 instead of 9 FP-pipe operations per cell.  The bound
// comes from the previous pass (wave5_fused_kernel's amax_out); the first
// pass of a chain, fields that grow past the limit and the border path use
// the exact form.  (A per-warp guard inside the loop measured slower: 18.3 vs
// 20.8 TB/s; the decision here is one load per block.)
__device__ __forceinline__ float4 wave_vec_fast(float4 m, float4 n, float4 s, float4 p, float wv, float ev,
                                                float c) {
  const f32x2 nsA = add2(pack2(n.x, n.y), pack2(s.x, s.y));
  const f32x2 nsB = add2(pack2(n.z, n.w), pack2(s.z, s.w));
  float a0, a1, b0, b1;
  unpack2(nsA, a0, a1);
  unpack2(nsB, b0, b1);
  a0 = __fadd_rn(__fadd_rn(a0, wv), m.y);
  a1 = __fadd_rn(__fadd_rn(a1, m.x), m.z);
  b0 = __fadd_rn(__fadd_rn(b0, m.y), m.w);
  b1 = __fadd_rn(__fadd_rn(b1, m.z), ev);
  const f32x2 uA = pack2(m.x, m.y), uB = pack2(m.z, m.w);
  const f32x2 m4 = pack2(-4.f, -4.f), two = pack2(2.f, 2.f);
  const f32x2 lapA = fma2(uA, m4, pack2(a0, a1)), lapB = fma2(uB, m4, pack2(b0, b1));
  // t = fma(2, u, -p): the same addends as fl(2u) + (-p), so also the same
  // signed zero when 2u == p (the form -fma(-2, u, p) gives -0 there)
  const f32x2 tA = fma2(uA, two, pack2(-p.x, -p.y)), tB = fma2(uB, two, pack2(-p.z, -p.w));
  // c*lap as fma(c, lap, +0), then a packed add: an FFMA2 result is not a
  // product ptxas can contract into the add.  fl(c*lap + 0) == fl(c*lap)
  // except for an exact -0 product (+0 instead), i.e. lap == -0 when c > 0,
  // which needs u == +0; then t = fl(2u - p) is never -0, and t + (-0) ==
  // t + (+0).  So for c > 0 (the host enables this form only then) the bits
  // are those of the DSL's t + c*lap.
  const f32x2 cc = pack2(c, c), zero = pack2(0.f, 0.f);
  const f32x2 oA = add2(tA, fma2(cc, lapA, zero)), oB = add2(tB, fma2(cc, lapB, zero));
  float4 o;
  unpack2(oA, o.x, o.y);
  unpack2(oB, o.z, o.w);
  return o;
}
template <typename Vec>
__device__ __forceinline__ Vec wave_vec_fast(Vec m, Vec n, Vec s, Vec p, decltype(m.x) wv, decltype(m.x) ev,
                                            decltype(m.x) c) {
  return wave_vec(m, n, s, p, wv, ev, c);  // other widths / float64: exact form
}

__device__ __forceinline__ float abs_max(float4 v) { return fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))); }
__device__ __forceinline__ float abs_max(float2 v) { return fmaxf(fabsf(v.x), fabsf(v.y)); }
__device__ __forceinline__ float abs_max(double2 v) { return (float)fmax(fabs(v.x), fabs(v.y)); }
// running max |x| of stored vectors: two 3-input FMNMX per float4
__device__ __forceinline__ float amax_with(float m, float4 v) {
  m = fmaxf(fmaxf(m, fabsf(v.x)), fabsf(v.y));
  return fmaxf(fmaxf(m, fabsf(v.z)), fabsf(v.w));
}
__device__ __forceinline__ float amax_with(float m, float2 v) { return fmaxf(fmaxf(m, fabsf(v.x)), fabsf(v.y)); }
__device__ __forceinline__ float amax_with(float m, double2 v) { return fmaxf(m, abs_max(v)); }


__device__ __forceinline__ void cp_async_row(void* smem, const void* gmem, bool valid, int bytes) {
  const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  const int src_size = valid ? bytes : 0;  // 0: zero-fill, source not read
  if (bytes == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(gmem), "r"(src_size) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst), "l"(gmem), "r"(src_size) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Input rows stream through a per-warp shared-memory ring D rows deep
// (cp.async, one commit group per row, each lane fetches and later reads
// back only its own V columns), so D rows of both inputs are in flight per
// warp without holding them in registers.
// Warps per SM (one-warp blocks): the register-heavy KL = 8, V = 4 variant
// runs 12 -- with 32-bit row counters and running prefetch pointers it fits
// the 168 registers that 3 warps per SM sub-partition allow (64-bit row
// arithmetic needed ~200 and capped it at 8; 16 warps at 128 registers
// spill 72 bytes a thread and measured 11% slower, profiles/r01/w16_ab.log);
// the other KL = 8 shapes 8, KL = 4 runs 16.  (Keeping the rows two iterations old of every
// level in shared memory freed ~32 registers but measured slower: 16.7 vs
// 20.8 TB/s, the extra LDS/STS per level cost more than the occupancy
// gained.)
template <int KL, int V>
struct FusedShape {
  static constexpr int kWarpsPerSm = KL == 8 ? (V == 4 ? 12 : 8) : 16;
};

// Work split.  The pass's work is the output rows [out_lo, out_hi) of every
// column strip, cut into pieces of `per_warp` rows; by default (map 2)
// piece q is strip q % strips, row range q / strips, and it is the
// one-warp block q -- so consecutive blocks, resident together, march
// neighbouring strips over the same rows and the strips' shared halo
// columns come out of L2 once (ncu: 2.31 GB DRAM reads per 16384^2 pass;
// strip-major ranges read 2.73 GB and ran 26% slower, profiles/r02).
// One-warp blocks keep every per-piece quantity (rows, phases, store
// windows) block-uniform, so ptxas proves the warp converged at each
// shuffle: with a warp index from threadIdx the hot loop carried two
// divergence checks and reconvergence barriers per row, the 12-warp block
// also spilled, and the pass ran 15% slower (profiles/r02/fused_layout_ab.log;
// CQ_FUSED_WPB / CQ_FUSED_MAP select those layouts for A/B runs).  A range
// of the strip-major maps (0, 1) that crosses a strip end is two pieces.
// Each piece marches its rows plus 2*KL halo rows in three phases of whole
// ring turns: full border checks where a level meets row 0 / H-1 or a
// prefetch leaves [in_lo, in_hi) (first / last turns of border pieces),
// column checks only for strips touching column 0 / W-1, and the unchecked
// body (FMA form when the previous pass bounded |X|, else the exact form).
// march modes (bit flags): row-border checks, column-border checks, FMA form
enum { kRows = 1, kCols = 2, kFast = 4, kEdgeAll = kRows | kCols };

// Up to two peer allocations (CUDA IPC pointers) that also receive some of
// the pass's output rows: the neighbouring ranks' halo rows for their next
// pass, written over NVLink while the pass runs (executor._PeerHalo).
struct FusedMirrors {
  cq_mirror_t m[2];
  int n;
  cq_peer_sync_t sync;
  int sync_on, n_edge;  // blocks with an edge piece (the last one signals)
};

// an edge block waits for the neighbours' previous pass (their rows for this
// one are in place, and they no longer read the rows this one sends them)
__device__ __forceinline__ void edge_wait(const FusedMirrors& mir, unsigned long long* flag) {
  const unsigned long long want = *(volatile unsigned long long*)mir.sync.count;
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const unsigned long long* sl = (const unsigned long long*)mir.sync.slot[k];
    if (sl == nullptr) continue;
    while (true) {
      unsigned long long v;
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(sl) : "memory");
      if (v >= want) break;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if ((long long)(t - t0) > mir.sync.timeout_ns) {
        report_error(flag, CQ_ERR_P2P, 0, (int64_t)want, (int64_t)v, 0);
        return;
      }
      __nanosleep(32);
    }
  }
}

// the last edge block of the pass: count += 1, published to the neighbours
__device__ __forceinline__ void edge_done(const FusedMirrors& mir) {
  __threadfence_system();
  if (atomicAdd((unsigned int*)mir.sync.done, 1u) == (unsigned int)mir.n_edge - 1) {
    *(volatile unsigned int*)mir.sync.done = 0;
    const unsigned long long v = *(volatile unsigned long long*)mir.sync.count + 1;
    *(volatile unsigned long long*)mir.sync.count = v;
    __threadfence_system();
#pragma unroll
    for (int k = 0; k < 2; ++k)
      if (mir.sync.peer_slot[k] != nullptr)
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(mir.sync.peer_slot[k]), "l"(v) : "memory");
  }
}

// PEER: the multi-rank variant (peer stores, in-pass ordering, per-piece
// bound); without it the kernel compiles exactly as the single-GPU pass.
template <typename T, int KL, int V, int D, int WPB, bool PEER>
__global__ void __launch_bounds__(32 * WPB, FusedShape<KL, V>::kWarpsPerSm / WPB)
    wave5_fused_kernel(cq_view_t u, cq_view_t upr, cq_view_t out_last, cq_view_t out_prev, int64_t in_lo,
                       int64_t in_hi, int64_t out_lo, int64_t out_hi, int64_t H, int64_t W, T c,
                       int64_t per_warp, int map, const float* __restrict__ amax_in,
                       float* __restrict__ amax_out, float limit, int64_t fast_lo, int64_t fast_hi,
                       const __grid_constant__ FusedMirrors mir, unsigned long long* err_flag) {
  typedef typename FVec<T, V>::T Vec;
  bool mirrored = false;  // this block stored rows to a peer
  static_assert(KL >= 2 && KL % V == 0, "strip offsets must stay vector aligned");
  static_assert(D % 3 == 0, "prefetch ring must be a multiple of the window");
  constexpr int SW = 32 * V - 2 * KL;
  extern __shared__ __align__(16) uint8_t fused_smem[];
  const int lane = threadIdx.x & 31, warp = WPB == 1 ? 0 : threadIdx.x >> 5;
  Vec* ring = reinterpret_cast<Vec*>(fused_smem) + (size_t)warp * D * 2 * 32;  // [D][2][32] per warp
  const int64_t rows = out_hi - out_lo;
  const int64_t strips = (W + SW - 1) / SW, total = strips * rows;
  const int64_t q = map == 1 ? (int64_t)warp * gridDim.x + blockIdx.x : (int64_t)blockIdx.x * WPB + warp;
  int64_t p, pend;
  if (map == 2) {
    // strip-minor: range q is strip q % strips, piece q / strips
    const int64_t st = q % strips, a0 = q / strips * per_warp;
    p = st * rows + a0;
    pend = a0 < rows ? st * rows + min(rows, a0 + per_warp) : p;
  } else {
    p = q * per_warp;
    pend = min(p + per_warp, total);
  }
  // |inputs| bound from the previous pass (amax_in, null: unknown); NaN
  // compares false and keeps the exact form
  const bool fast = p < pend && amax_in != nullptr && *amax_in < limit;
  float amax = 0.f;  // max |stored value| of this warp (amax_out)
  const int64_t us = u.stride[1], ps = upr.stride[1];
  const int64_t ls = out_last.stride[1], pstr = out_prev.stride[1];

  while (p < pend) {  // warp-uniform
    const int64_t strip = p / rows;
    const int64_t a = p - strip * rows, b = min(rows, a + (pend - p));
    p += b - a;
    const int64_t r0 = out_lo + a, r1 = out_lo + b;
    const int64_t c0 = strip * SW - KL;  // first loaded column of the strip
    const int64_t col = c0 + lane * V;
    const bool colok = col >= 0 && col < W;
    const bool keep = lane >= KL / V && lane < 32 - KL / V && col < W;
    const int64_t rb = r0 - KL, re = r1 + KL;  // input rows this piece streams
    const T* ub = (const T*)u.ptr + (colok ? col : 0) - u.alloc.lo[2] + (rb - u.alloc.lo[1]) * us;
    const T* pb = (const T*)upr.ptr + (colok ? col : 0) - upr.alloc.lo[2] + (rb - upr.alloc.lo[1]) * ps;
    T* sl = (T*)out_last.ptr + (col - out_last.alloc.lo[2]) + (r0 - out_last.alloc.lo[1]) * ls;
    T* sp = (T*)out_prev.ptr + (col - out_prev.alloc.lo[2]) + (r0 - out_prev.alloc.lo[1]) * pstr;
    // rows are counted from rb in 32-bit (t = ri - rb); the store windows in
    // t: out_prev (level KL-1, row rb + t - KL + 1 in [r0, r1)) and out_last
    // (level KL, row rb + t - KL >= r0; always < r1)
    const int nrow = (int)(re - rb);
    const int prev_lo = 2 * KL - 1, prev_hi = (int)(r1 - rb) + KL - 1, last_lo = 2 * KL;
    // phases (whole ring turns): iterations t < t1 see row 0 (t <= KL - rb)
    // or prefetch below in_lo; t >= t2 see row H-1 (t >= H - rb) or
    // prefetch at / above in_hi (only when re > in_hi)
    const int nfull = nrow / D * D;
    int64_t top = in_lo - rb - D, bot = H - rb;
    if (KL - rb + 1 > top) top = KL - rb + 1;
    if (top < 0) top = 0;
    if (nrow < bot) bot = nrow;
    if (re > in_hi && in_hi - rb - D < bot) bot = in_hi - rb - D;
    if (bot < 0) bot = 0;
    const int t1 = (int)(top >= nfull ? nfull : (top + D - 1) / D * D);
    int t2 = (int)(bot >= nfull ? nfull : bot / D * D);
    if (t2 < t1) t2 = t1;
    const bool col_edge = !(c0 > 0 && c0 + 32 * V < W);
    // the bound covers rows [fast_lo, fast_hi) only (e.g. not a neighbour's halo rows)
    bool fast_piece = PEER ? fast && rb >= fast_lo && re <= fast_hi : fast;
    // does this piece write rows a peer also receives (block-uniform)
    bool mirror_piece = false;
    for (int k = 0; PEER && k < mir.n; ++k) mirror_piece |= r0 < mir.m[k].row_hi && r1 > mir.m[k].row_lo;
    mirrored |= mirror_piece;
    if (PEER) {
      if (mirror_piece && mir.sync_on) {
        if (lane == 0) edge_wait(mir, err_flag);  // before any input row is fetched
        __syncwarp();
        // the bound now includes the neighbours' rows this piece reads
        fast_piece = amax_in != nullptr && *(volatile const float*)amax_in < limit && rb >= fast_lo &&
                     re <= fast_hi;
      }
    }

    // running source pointers of the next row to prefetch (row rb + t + D)
    const T* uf = ub + (int64_t)D * us;
    const T* pf = pb + (int64_t)D * ps;
    // fetch input row rb + k into ring slot `slot` from (uk, pk)
    auto fetch = [&](auto mode, int slot, int k, const T* uk, const T* pk) {
      constexpr int M = decltype(mode)::value;
      bool ok = true;
      if (M & kRows) {
        const int64_t r = rb + k;
        ok = colok && r >= in_lo && r < in_hi;
      } else if (M & kCols) {
        ok = colok;
      }
      if (!ok) uk = ub, pk = pb;  // any mapped address; zero-filled, not read
      cp_async_row(ring + (slot * 2 + 0) * 32 + lane, uk, ok, sizeof(Vec));
      cp_async_row(ring + (slot * 2 + 1) * 32 + lane, pk, ok, sizeof(Vec));
    };
    Vec L[KL][3];  // level j (0 = X(t)) rows, slot = t % 3
    Vec P[3];      // X(t-1) rows, same slots
#pragma unroll
    for (int q = 0; q < D; ++q) {
      if (q < nrow) fetch(std::integral_constant<int, kEdgeAll>{}, q, q, ub + (int64_t)q * us, pb + (int64_t)q * ps);
      cp_async_commit();
    }
    // one input row: land it, prefetch row t + D, advance levels 1..LM.
    // (Skipping level j before iteration 2j, its first row of the
    // trapezoid, in a prologue saved 3.75% of the level-rows but cost the
    // main loop 29 register moves per turn: not kept.)
    auto row = [&](auto mode, auto lm, const int t, const int sd) {
      constexpr int M = decltype(mode)::value;
      constexpr int LM = decltype(lm)::value;
      const int s = sd % 3, so = (sd + 1) % 3, sm = (sd + 2) % 3;  // rows t, t-2, t-1
      cp_async_wait<D - 1>();  // row t (the oldest group) has landed
      L[0][s] = ring[(sd * 2 + 0) * 32 + lane];
      P[s] = ring[(sd * 2 + 1) * 32 + lane];
      if (t + D < nrow) fetch(mode, sd, t + D, uf, pf);
      cp_async_commit();
      uf += us;
      pf += ps;
#pragma unroll
      for (int j = 1; j <= LM; ++j) {
        const Vec mid = L[j - 1][sm];
        Vec nn = L[j - 1][so], ss = L[j - 1][s];
        T wv = __shfl_up_sync(0xffffffffu, last_of(mid), 1);
        T ev = __shfl_down_sync(0xffffffffu, first_of(mid), 1);
        if (M & kRows) {
          const int64_t rho = rb + t - j;
          if (rho == 0) nn = mid;
          if (rho == H - 1) ss = mid;
        }
        if (M & kCols) {
          if (col == 0) wv = first_of(mid);
          if (col + V == W) ev = last_of(mid);
        }
        const Vec pp = (j == 1) ? P[sm] : L[j >= 2 ? j - 2 : 0][so];
        const Vec o = (M & kFast) ? wave_vec_fast(mid, nn, ss, pp, wv, ev, c) : wave_vec(mid, nn, ss, pp, wv, ev, c);
        if (j < KL) L[j][s] = o;
        if (j == KL - 1 && t >= prev_lo && t < prev_hi) {
          if (keep) {
            __stcs(reinterpret_cast<Vec*>(sp), o);
            amax = amax_with(amax, o);
          }
          sp += pstr;
        }
        if (j == KL && t >= last_lo) {
          if (keep) {
            __stcs(reinterpret_cast<Vec*>(sl), o);
            amax = amax_with(amax, o);
          }
          sl += ls;
        }
      }
    };
    // whole ring turns without a bounds test (the warp stays converged, so
    // the shuffles need no collective fallback), then the remainder
    using AllLevels = std::integral_constant<int, KL>;
    auto turns = [&](auto mode, int& t, const int end) {
#pragma unroll 1
      for (; t < end; t += D) {
#pragma unroll
        for (int sd = 0; sd < D; ++sd) row(mode, AllLevels{}, t + sd, sd);
      }
    };
    int t = 0;
    turns(std::integral_constant<int, kEdgeAll>{}, t, t1);
    if (col_edge) {
      if (fast_piece) turns(std::integral_constant<int, kCols | kFast>{}, t, t2);
      else turns(std::integral_constant<int, kCols>{}, t, t2);
    } else {
      if (fast_piece) turns(std::integral_constant<int, kFast>{}, t, t2);
      else turns(std::integral_constant<int, 0>{}, t, t2);
    }
    turns(std::integral_constant<int, kEdgeAll>{}, t, nfull);
#pragma unroll
    for (int sd = 0; sd < D; ++sd)
      if (nfull + sd < nrow) row(std::integral_constant<int, kEdgeAll>{}, AllLevels{}, nfull + sd, sd);
    cp_async_wait<0>();
    if (PEER && mirror_piece && keep) {
      // the piece's rows a peer also receives, re-read from what this lane
      // just stored (same thread: program order) and written over NVLink
      for (int k = 0; k < mir.n; ++k) {
        const cq_mirror_t& m = mir.m[k];
        for (int64_t r = max(r0, m.row_lo); r < min(r1, m.row_hi); ++r) {
          const T* ll = (const T*)out_last.ptr + (col - out_last.alloc.lo[2]) + (r - out_last.alloc.lo[1]) * ls;
          const T* lp = (const T*)out_prev.ptr + (col - out_prev.alloc.lo[2]) + (r - out_prev.alloc.lo[1]) * pstr;
          *reinterpret_cast<Vec*>((T*)m.last + (r - m.row0) * m.stride + (col - m.col0)) = *reinterpret_cast<const Vec*>(ll);
          *reinterpret_cast<Vec*>((T*)m.prev + (r - m.row0) * m.stride + (col - m.col0)) = *reinterpret_cast<const Vec*>(lp);
        }
      }
    }
  }
  if (amax_out != nullptr) {
    // values are >= 0, so their int bit patterns order like the floats
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    if (lane == 0) atomicMax(reinterpret_cast<int*>(amax_out), __float_as_int(amax));
    // the rows a neighbour receives also raise its bound for the next pass
    // (before the completion signal it waits for)
    if (PEER && mirrored && lane == 0)
      for (int k = 0; k < 2; ++k)
        if (mir.sync_on && mir.sync.peer_amax[k] != nullptr)
          atomicMax_system(reinterpret_cast<int*>(mir.sync.peer_amax[k]), __float_as_int(amax));
  }
  if (PEER && mirrored) {
    // the peer rows (and bounds) before the pass's completion signal
    if (mir.sync_on) {
      if (lane == 0) edge_done(mir);
    } else {
      __threadfence_system();
    }
  }
}

// Launch geometry of one fused pass over output rows [out_lo, out_lo + rows)
// of a W-column grid: rows per warp range, the grid, and the cells the
// launched warps compute per level (strip width x marched rows, halo
// columns / rows and dead lanes included) -- the denominator of the pass's
// recompute share (bench.py's roofline).
//
// Rows per piece: 224 for the KL = 8 pass and 24 for the HBM-bound KL = 4
// pass (interleaved sweeps, profiles/r02/fused_rows_sweep.log: longer
// pieces cut the halo recompute but every one-wave layout -- 1366 rows,
// all pieces in flight at once -- ran 10-25% slower), fewer when a launch
// would not fill the warp slots (short slabs, halo-row edge launches).
// CQ_FUSED_ROWS=<rows> forces the length.
struct FusedGeometry {
  int64_t per_warp, blocks, warps, computed_cells;
  int smem, threads, map;
};

static int fused_map() {
  const char* e = getenv("CQ_FUSED_MAP");  // read per launch (A/B sweeps)
  return e ? atoi(e) : 2;
}

template <typename T, int KL, int V, int D, int WPB>
static int fused_geometry(int64_t rows, int64_t W, FusedGeometry* g) {
  constexpr int sw = 32 * V - 2 * KL;
  auto kern = wave5_fused_kernel<T, KL, V, D, WPB, false>;
  auto kern_peer = wave5_fused_kernel<T, KL, V, D, WPB, true>;
  const int smem = WPB * D * 2 * 32 * V * (int)sizeof(T);
  CQ_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CQ_CHECK_CUDA(cudaFuncSetAttribute(kern_peer, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  // resident blocks per SM of this instantiation (same on every B200)
  static const int per_sm = [&] {
    int nb = 0;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, 32 * WPB, smem) == cudaSuccess ? nb : 0;
  }();
  int dev = 0, sms = 0;
  CQ_CHECK_CUDA(cudaGetDevice(&dev));
  CQ_CHECK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int64_t strips = (W + sw - 1) / sw, total = strips * rows;
  const int64_t slots = std::max<int64_t>(1, (int64_t)per_sm * sms) * WPB;
  g->map = fused_map();
  const char* env = getenv("CQ_FUSED_ROWS");  // read per launch (sweeps set it between launches)
  const int64_t forced = env ? (int64_t)atoll(env) : 0;
  int64_t per;
  if (forced > 0) {
    per = forced;
  } else {
    // short pieces (profiles/r02 sweeps), shorter still when a launch would
    // not fill the warp slots
    const int64_t cap = KL == 8 ? 224 : 24, floor_rows = KL == 8 ? 16 : 8;
    per = std::min(cap, std::max(floor_rows, (total + slots - 1) / slots));
  }
  per = std::max<int64_t>(1, per);
  g->per_warp = per;
  const int64_t pieces = (rows + per - 1) / per;
  g->warps = g->map == 2 ? strips * pieces : (total + per - 1) / per;
  g->blocks = (g->warps + WPB - 1) / WPB;
  // every piece marches its rows + 2 KL halo rows over 32 V columns
  int64_t marched = 0;
  if (g->map == 2) {
    marched = strips * (rows + 2 * KL * pieces);
  } else {
    for (int64_t q = 0; q < g->warps; ++q) {
      for (int64_t p = q * per, e = std::min(p + per, total); p < e;) {
        const int64_t a = p % rows, b = std::min(rows, a + (e - p));
        marched += b - a + 2 * KL;
        p += b - a;
      }
    }
  }
  g->computed_cells = marched * 32 * V;
  g->smem = smem;
  g->threads = 32 * WPB;
  return CQ_OK;
}

template <typename T, int KL, int V, int D, int WPB>
static int launch_fused(cudaStream_t st, const cq_view_t& u, const cq_view_t& upr, const cq_view_t& ol,
                        const cq_view_t& op, int64_t in_lo, int64_t in_hi, int64_t out_lo, int64_t out_hi,
                        int64_t H, int64_t W, T c, const float* amax_in, float* amax_out, float limit,
                        int64_t fast_lo, int64_t fast_hi, FusedMirrors mir, unsigned long long* err_flag) {
  FusedGeometry g;
  CQ_TRY((fused_geometry<T, KL, V, D, WPB>(out_hi - out_lo, W, &g)));
  if (mir.sync_on) {
    // blocks (strip-minor pieces) whose rows meet a mirror range
    CQ_REQUIRE(g.map == 2, "cq_wave5_fused_ex: peer sync needs the strip-minor layout");
    const int64_t rows = out_hi - out_lo, pieces = (rows + g.per_warp - 1) / g.per_warp;
    const int64_t strips = g.warps / pieces;
    int64_t edge_pieces = 0;
    for (int64_t q = 0; q < pieces; ++q) {
      const int64_t a = out_lo + q * g.per_warp, b = std::min(out_hi, a + g.per_warp);
      bool e = false;
      for (int k = 0; k < mir.n; ++k) e |= a < mir.m[k].row_hi && b > mir.m[k].row_lo;
      edge_pieces += e;
    }
    mir.n_edge = (int)(strips * edge_pieces);
    if (mir.n_edge == 0) mir.sync_on = 0;
  }
  if (mir.n > 0)
    wave5_fused_kernel<T, KL, V, D, WPB, true><<<(unsigned)g.blocks, g.threads, g.smem, st>>>(
        u, upr, ol, op, in_lo, in_hi, out_lo, out_hi, H, W, c, g.per_warp, g.map, amax_in, amax_out, limit, fast_lo,
        fast_hi, mir, err_flag);
  else
    wave5_fused_kernel<T, KL, V, D, WPB, false><<<(unsigned)g.blocks, g.threads, g.smem, st>>>(
        u, upr, ol, op, in_lo, in_hi, out_lo, out_hi, H, W, c, g.per_warp, g.map, amax_in, amax_out, limit, fast_lo,
        fast_hi, mir, err_flag);
  return CQ_OK;
}

// One fused pass: its launch parameters, or (geometry != null) only the
// geometry it would launch with.
struct FusedLaunch {
  cudaStream_t st;
  const cq_view_t *u, *upr, *out_last, *out_prev;
  int64_t in_lo, in_hi, out_lo, out_hi, H, W;
  double c, k2, k4;
  const float* amax_in;
  float* amax_out;
  float limit;
  FusedGeometry* geometry;
  int64_t fast_lo, fast_hi;
  FusedMirrors mir;
  unsigned long long* err_flag;
};

template <typename T, int KL, int V, int D, int WPB = 1>
static int fused_run(const FusedLaunch& L) {
  if (L.geometry) return fused_geometry<T, KL, V, D, WPB>(L.out_hi - L.out_lo, L.W, L.geometry);
  return launch_fused<T, KL, V, D, WPB>(L.st, *L.u, *L.upr, *L.out_last, *L.out_prev, L.in_lo, L.in_hi, L.out_lo,
                                        L.out_hi, L.H, L.W, (T)L.c, L.amax_in, L.amax_out, L.limit, L.fast_lo,
                                        L.fast_hi, L.mir, L.err_flag);
}

// warps per block: CQ_FUSED_WPB (A/B sweeps; 1 = one-warp blocks)
static int fused_wpb() {
  const char* e = getenv("CQ_FUSED_WPB");
  return e ? atoi(e) : 1;
}

// tuning: CQ_WAVE_FUSED_CFG="V,D" (lane width, cp.async ring depth);
// default 4,6 (KL = 4: two 8-warp blocks / SM; KL = 8: one 12-warp block /
// SM, its 8 levels of register windows need ~153 registers)
static int fused_dispatch(int kind, int levels, const FusedLaunch& L) {
  if (kind == CQ_F64) {
    // two doubles per lane (16-byte rows): 56 (KL = 4) or 48 (KL = 8) valid
    // columns per warp strip
    return levels == 4 ? fused_run<double, 4, 2, 6>(L) : fused_run<double, 8, 2, 6>(L);
  }
  int v = 0, d = 0;   // read per launch (A/B sweeps switch it between launches)
  if (const char* e = getenv("CQ_WAVE_FUSED_CFG")) sscanf(e, "%d,%d", &v, &d);
  const int cfg_env = v ? v * 100 + d : 0;
  const int cfg = cfg_env ? cfg_env : 4 * 100 + 6;
  switch (cfg * 10 + levels) {
#define CQ_FUSED_CASE(VV, DD, KL) \
  case (VV * 100 + DD) * 10 + KL: \
    return fused_run<float, KL, VV, DD>(L);
    case (4 * 100 + 6) * 10 + 4:
      return fused_wpb() == 8 ? fused_run<float, 4, 4, 6, 8>(L) : fused_run<float, 4, 4, 6>(L);
    case (4 * 100 + 6) * 10 + 8:
      return fused_wpb() == 12 ? fused_run<float, 8, 4, 6, 12>(L) : fused_run<float, 8, 4, 6>(L);
    CQ_FUSED_CASE(4, 9, 4) CQ_FUSED_CASE(4, 9, 8)
    CQ_FUSED_CASE(4, 12, 4) CQ_FUSED_CASE(4, 12, 8)
    CQ_FUSED_CASE(2, 12, 4) CQ_FUSED_CASE(2, 12, 8)
#undef CQ_FUSED_CASE
    default:
      set_error("cq_wave5_fused: CQ_WAVE_FUSED_CFG=%d not compiled", cfg);
      return CQ_ERR_ARG;
  }
}

}  // namespace cq

using namespace cq;

#define CQ_GET_STREAM(dev, s)                                               \
  CQ_TRY(ensure_device(dev));                                               \
  cudaStream_t st = stream_of(dev, s);                                      \
  CQ_REQUIRE(st != nullptr, "bad stream %d", s);                            \
  CQ_CHECK_CUDA(cudaSetDevice(dev));                                        \
  DeviceState* ds = device_state(dev);                                      \
  (void)ds;

extern "C" {

int cq_fill(int device, int stream, int kind, const cq_view_t* dst, const cq_box_t* box,
            const cq_box_t* extent, int mode, double value, int64_t ivalue) {
  CQ_GET_STREAM(device, stream);
  int64_t vol = box_volume(*box);
  if (vol <= 0) return CQ_OK;
  int grid = grid_for(vol, 256, ds->sm_count, 8);
  if (kind == CQ_F64) {
    fill_kernel<double><<<grid, 256, 0, st>>>(*dst, *box, *extent, mode, mode == 0 ? 0.0 : value);
  } else if (kind == CQ_F32) {
    fill_kernel<float><<<grid, 256, 0, st>>>(*dst, *box, *extent, mode,
                                             mode == 0 ? 0.f : (float)value);
  } else {
    fill_kernel<long long><<<grid, 256, 0, st>>>(*dst, *box, *extent, mode, mode == 0 ? 0LL : (long long)ivalue);
  }
  CQ_CHECK_LAUNCH();
  return CQ_OK;
}

int cq_saxpy(int device, int stream, int kind, double alpha, int64_t ialpha, const void* x,
             const void* y, void* z, int64_t n) {
  CQ_GET_STREAM(device, stream);
  if (n <= 0) return CQ_OK;
  if (kind == CQ_I64) {
    saxpy_i64_kernel<<<grid_for(n, 256, ds->sm_count, 8), 256, 0, st>>>(
        (long long)ialpha, (const long long*)x, (const long long*)y, (long long*)z, n);
    CQ_CHECK_LAUNCH();
    return CQ_OK;
  }
  bool aligned = (((uintptr_t)x | (uintptr_t)y | (uintptr_t)z) & 15) == 0;
  CQ_REQUIRE(aligned, "cq_saxpy: operands must be 16-byte aligned");
  int per = (kind == CQ_F32) ? 4 : 2;
  int64_t vec = n / per;
  // persistent-style grid: 148 SMs x 8 blocks x 256 threads, 2 vectors per trip
  int grid = grid_for((vec + 1) / 2, 256, ds->sm_count, 8);
  if (kind == CQ_F32)
    saxpy_kernel<float><<<grid, 256, 0, st>>>((float)alpha, (const float*)x, (const float*)y, (float*)z, n);
  else
    saxpy_kernel<double><<<grid, 256, 0, st>>>(alpha, (const double*)x, (const double*)y, (double*)z, n);
  CQ_CHECK_LAUNCH();
  return CQ_OK;
}

int cq_wave5(int device, int stream, int kind, const cq_view_t* u, const cq_view_t* upr,
             const cq_view_t* out, const cq_box_t* box, const cq_box_t* extent, double c,
             double k2, double k4) {
  CQ_GET_STREAM(device, stream);
  CQ_REQUIRE(kind == CQ_F32 || kind == CQ_F64, "cq_wave5: float kinds only");
  int64_t vol = box_volume(*box);
  if (vol <= 0) return CQ_OK;
  const int64_t H = extent->hi[1], W = extent->hi[2];
  const int eb = kind == CQ_F32 ? 4 : 8;
  const int V = 16 / eb;
  bool rows_ok = box->hi[0] - box->lo[0] == 1 && box->lo[2] == 0 && box->hi[2] == W && W % V == 0;
  for (const cq_view_t* v : {u, upr, out}) {
    rows_ok = rows_ok && ((uintptr_t)v->ptr % 16 == 0) && v->stride[1] % V == 0 && v->alloc.lo[2] == 0 &&
              v->stride[2] == 1;
  }
  if (rows_ok) {
    constexpr int RB = 32;
    int64_t rows = box->hi[1] - box->lo[1];
    dim3 grid((unsigned)((W / V + 255) / 256), (unsigned)((rows + RB - 1) / RB));
    if (kind == CQ_F32)
      wave5_rows_kernel<float, RB><<<grid, 256, 0, st>>>(*u, *upr, *out, box->lo[1], box->hi[1], H, W,
                                                         (float)c, (float)k2, (float)k4);
    else
      wave5_rows_kernel<double, RB><<<grid, 256, 0, st>>>(*u, *upr, *out, box->lo[1], box->hi[1], H, W,
                                                          c, k2, k4);
  } else {
    int grid = grid_for(vol, 256, ds->sm_count, 8);
    if (kind == CQ_F32)
      wave5_cell_kernel<float><<<grid, 256, 0, st>>>(*u, *upr, *out, *box, H, W, (float)c, (float)k2,
                                                     (float)k4);
    else
      wave5_cell_kernel<double><<<grid, 256, 0, st>>>(*u, *upr, *out, *box, H, W, c, k2, k4);
  }
  CQ_CHECK_LAUNCH();
  return CQ_OK;
}

int cq_wave5_fused(int device, int stream, int kind, int levels, const cq_view_t* u, const cq_view_t* upr,
                   const cq_view_t* out_last, const cq_view_t* out_prev, int64_t in_lo, int64_t in_hi,
                   int64_t out_lo, int64_t out_hi, const cq_box_t* extent, double c, double k2, double k4) {
  return cq_wave5_fused_bounded(device, stream, kind, levels, u, upr, out_last, out_prev, in_lo, in_hi, out_lo,
                                out_hi, extent, c, k2, k4, nullptr, nullptr);
}

int cq_wave5_fused_bounded(int device, int stream, int kind, int levels, const cq_view_t* u, const cq_view_t* upr,
                           const cq_view_t* out_last, const cq_view_t* out_prev, int64_t in_lo, int64_t in_hi,
                           int64_t out_lo, int64_t out_hi, const cq_box_t* extent, double c, double k2, double k4,
                           const float* amax_in, float* amax_out) {
  return cq_wave5_fused_ex(device, stream, kind, levels, u, upr, out_last, out_prev, in_lo, in_hi, out_lo, out_hi,
                           extent, c, k2, k4, amax_in, amax_out, in_lo, in_hi, nullptr, 0, nullptr);
}

int cq_wave5_fused_ex(int device, int stream, int kind, int levels, const cq_view_t* u, const cq_view_t* upr,
                      const cq_view_t* out_last, const cq_view_t* out_prev, int64_t in_lo, int64_t in_hi,
                      int64_t out_lo, int64_t out_hi, const cq_box_t* extent, double c, double k2, double k4,
                      const float* amax_in, float* amax_out, int64_t fast_lo, int64_t fast_hi,
                      const cq_mirror_t* mirrors, int n_mirrors, const cq_peer_sync_t* sync) {
  CQ_GET_STREAM(device, stream);
  if (out_hi <= out_lo) return CQ_OK;
  const int64_t H = extent->hi[1], W = extent->hi[2];
  CQ_REQUIRE(levels == 4 || levels == 8, "cq_wave5_fused: levels must be 4 or 8 (got %d)", levels);
  CQ_REQUIRE(kind == CQ_F32 || kind == CQ_F64, "cq_wave5_fused: float kinds only");
  CQ_REQUIRE(W % 4 == 0, "cq_wave5_fused: row length must be a multiple of 4");
  CQ_REQUIRE(k2 == 2.0 && k4 == 4.0, "cq_wave5_fused: the body's constants must be k2 = 2, k4 = 4");
  for (const cq_view_t* v : {u, upr, out_last, out_prev}) {
    CQ_REQUIRE(((uintptr_t)v->ptr % 16 == 0) && v->stride[1] % 4 == 0 && v->alloc.lo[2] == 0 &&
                   v->alloc.hi[2] == W && v->stride[2] == 1,
               "cq_wave5_fused: views must hold whole 16-byte aligned rows");
  }
  CQ_REQUIRE(out_last->ptr != u->ptr && out_last->ptr != upr->ptr && out_prev->ptr != u->ptr &&
                 out_prev->ptr != upr->ptr && out_last->ptr != out_prev->ptr,
             "cq_wave5_fused: outputs must not alias the inputs");
  // the trapezoid: level L is exact on rows [in_lo + L, in_hi - L), except at the true borders
  const int64_t lo_ok = in_lo == 0 ? 0 : in_lo + levels, hi_ok = in_hi == H ? H : in_hi - levels;
  CQ_REQUIRE(out_lo >= lo_ok && out_hi <= hi_ok && in_lo >= 0 && in_hi <= H,
             "cq_wave5_fused: rows [%lld, %lld) are not determined by input rows [%lld, %lld)",
             (long long)out_lo, (long long)out_hi, (long long)in_lo, (long long)in_hi);
  // the fast form is exact while every value of the pass stays below 2^125
  // (then 2u and 4u do not overflow); one step grows max|X| by at most
  // g = 3 + 8|c| (|2u| + |p| + |c| |n+s+w+e-4u|), so inputs below
  // 2^124 / g^levels are safe (CQ_WAVE_FAST=0 disables the fast form)
  static const bool fast_ok = [] {
    const char* e = getenv("CQ_WAVE_FAST");
    return !(e && e[0] == '0');
  }();
  // (and c > 0: the form's c*lap + 0 product, see wave_vec_fast)
  const float limit = fast_ok && c > 0.0
                          ? (float)(std::ldexp(1.0, 124) / std::pow(3.0 + 8.0 * std::fabs(c) + 1e-3, levels))
                          : 0.f;
  CQ_REQUIRE(n_mirrors >= 0 && n_mirrors <= 2 && (n_mirrors == 0 || mirrors != nullptr),
             "cq_wave5_fused_ex: 0..2 mirrors");
  FusedMirrors mir{};
  for (int k = 0; k < n_mirrors; ++k) mir.m[k] = mirrors[k];
  mir.n = n_mirrors;
  if (sync != nullptr) {
    CQ_REQUIRE(sync->count != nullptr && sync->done != nullptr && n_mirrors > 0,
               "cq_wave5_fused_ex: peer sync needs counters and mirrors");
    mir.sync = *sync;
    mir.sync_on = 1;
  }
  FusedLaunch L{st, u, upr, out_last, out_prev, in_lo, in_hi, out_lo, out_hi, H, W, c, k2, k4, amax_in, amax_out,
                limit, nullptr, fast_lo, fast_hi, mir, (unsigned long long*)ds->error_flag};
  CQ_TRY(fused_dispatch(kind, levels, L));
  CQ_CHECK_LAUNCH();
  return CQ_OK;
}

int cq_wave5_fused_geometry(int device, int kind, int levels, int64_t rows, int64_t W, int64_t out[4]) {
  CQ_TRY(ensure_device(device));
  CQ_CHECK_CUDA(cudaSetDevice(device));
  CQ_REQUIRE(levels == 4 || levels == 8, "cq_wave5_fused_geometry: levels must be 4 or 8 (got %d)", levels);
  CQ_REQUIRE(kind == CQ_F32 || kind == CQ_F64, "cq_wave5_fused_geometry: float kinds only");
  CQ_REQUIRE(rows > 0 && W > 0, "cq_wave5_fused_geometry: empty launch");
  FusedGeometry g;
  FusedLaunch L{};
  L.out_lo = 0;
  L.out_hi = rows;
  L.W = W;
  L.geometry = &g;
  CQ_TRY(fused_dispatch(kind, levels, L));
  out[0] = g.per_warp;
  out[1] = g.blocks;
  out[2] = g.warps;
  out[3] = g.computed_cells;
  return CQ_OK;
}

int cq_p2p_wait(int device, int stream, const uint64_t* slot0, const uint64_t* slot1, const uint64_t* count,
                int64_t timeout_ns) {
  CQ_GET_STREAM(device, stream);
  CQ_REQUIRE(count != nullptr, "cq_p2p_wait: null counter");
  p2p_wait_kernel<<<1, 1, 0, st>>>((const unsigned long long*)slot0, (const unsigned long long*)slot1,
                                   (const unsigned long long*)count, (long long)timeout_ns,
                                   (unsigned long long*)ds->error_flag);
  CQ_CHECK_LAUNCH();
  return CQ_OK;
}

int cq_p2p_signal(int device, int stream, uint64_t* count, uint64_t* peer0, uint64_t* peer1) {
  CQ_GET_STREAM(device, stream);
  CQ_REQUIRE(count != nullptr, "cq_p2p_signal: null counter");
  p2p_signal_kernel<<<1, 1, 0, st>>>((unsigned long long*)count, (unsigned long long*)peer0,
                                     (unsigned long long*)peer1);
  CQ_CHECK_LAUNCH();
  return CQ_OK;
}

int cq_expr_eval(int device, int stream, const cq_expr_t* expr) {
  CQ_GET_STREAM(device, stream);
  int64_t vol = box_volume(expr->box);
  if (vol <= 0) return CQ_OK;
  CQ_REQUIRE(expr->n_out >= 1 && expr->n_out <= CQ_EXPR_MAX_OUT, "cq_expr_eval: bad n_out");
  unsigned long long* flag = (unsigned long long*)ds->error_flag;
  int grid = grid_for(vol, 128, ds->sm_count, 16);
  if (expr->kind == CQ_F64) expr_kernel<double><<<grid, 128, 0, st>>>(*expr, flag);
  else if (expr->kind == CQ_F32) expr_kernel<float><<<grid, 128, 0, st>>>(*expr, flag);
  else expr_kernel<long long><<<grid, 128, 0, st>>>(*expr, flag);
  CQ_CHECK_LAUNCH();
  return CQ_OK;
}

int cq_error_flag(int device, int* code, int64_t point[CQ_MAX_DIMS], int clear) {
  CQ_TRY(ensure_device(device));
  DeviceState* ds = device_state(device);
  CQ_CHECK_CUDA(cudaSetDevice(device));
  unsigned long long buf[4];
  CQ_CHECK_CUDA(cudaMemcpy(buf, ds->error_flag, sizeof(buf), cudaMemcpyDeviceToHost));
  // "no error" is the all-ones key written at device setup and on clear
  if (buf[0] == ~0ull) {
    *code = 0;
  } else {
    *code = (int)(buf[0] & 15ull);
    memcpy(point, &buf[1], 3 * sizeof(int64_t));
  }
  if (clear) {
    unsigned long long reset[4] = {~0ull, 0, 0, 0};
    CQ_CHECK_CUDA(cudaMemcpy(ds->error_flag, reset, sizeof(reset), cudaMemcpyHostToDevice));
  }
  return CQ_OK;
}

int cq_error_flag_async(int device, int stream, void* host32) {
  CQ_GET_STREAM(device, stream);
  CQ_REQUIRE(host32 != nullptr, "cq_error_flag_async: null host buffer");
  CQ_CHECK_CUDA(cudaMemcpyAsync(host32, ds->error_flag, 4 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
  return CQ_OK;
}

static int nbody_partial(cudaStream_t st, const float* pos, int64_t n, float* part, int64_t i_lo, int64_t i_hi,
                         float eps2, int col_lo, int col_hi) {
  static int forced = [] {
    const char* e = getenv("CQ_NBODY_NP");
    return e ? atoi(e) : 0;
  }();
  const int64_t bodies = i_hi - i_lo;
  // NB_JCOLS block columns give >= 8x more blocks than i-tiles, so the
  // widest variant (4 pairs per lane, best steady-state rate) fills the GPU
  // even at 32768 bodies per GPU; CQ_NBODY_NP overrides for experiments.
  const int use = forced ? forced : 4;
  switch (use) {
#define NB_LAUNCH(P)                                                                                        \
  case P:                                                                                                 \
    nbody_kick_kernel<P><<<dim3((unsigned)((bodies + 64 * P - 1) / (64 * P)), col_hi - col_lo), NB_WARPS * 32, 0, \
                           st>>>((const float4*)pos, n, part, i_lo, i_hi, eps2, col_lo);                \
    break;
    NB_LAUNCH(1)
    NB_LAUNCH(2)
    NB_LAUNCH(3)
    default:
    NB_LAUNCH(4)
#undef NB_LAUNCH
  }
  CQ_CHECK_LAUNCH();
  return CQ_OK;
}

int cq_nbody_kick(int device, int stream, const float* pos, int64_t n, const float* vel_in,
                  float* vel, int64_t i_lo, int64_t i_hi, float eps2, float dt) {
  CQ_GET_STREAM(device, stream);
  if (i_hi <= i_lo) return CQ_OK;
  const int64_t bodies = i_hi - i_lo;
  float* part = nullptr;
  CQ_TRY(scratch(device, stream, 1, (size_t)NB_JCOLS * bodies * 3 * sizeof(float), (void**)&part));
  CQ_TRY(nbody_partial(st, pos, n, part, i_lo, i_hi, eps2, 0, NB_JCOLS));
  nbody_kick_finalize<<<grid_for(bodies, 256, ds->sm_count, 8), 256, 0, st>>>(
      part, (const float4*)vel_in, (float4*)vel, bodies, dt);
  CQ_CHECK_LAUNCH();
  return CQ_OK;
}

int cq_nbody_jcols(int* cols) {
  *cols = NB_JCOLS;
  return CQ_OK;
}

int cq_nbody_kick_partial(int device, int stream, const float* pos, int64_t n, float* part, int64_t i_lo,
                          int64_t i_hi, float eps2, int col_lo, int col_hi) {
  CQ_GET_STREAM(device, stream);
  CQ_REQUIRE(0 <= col_lo && col_lo <= col_hi && col_hi <= NB_JCOLS, "cq_nbody_kick_partial: columns [%d, %d) "
             "outside [0, %d)", col_lo, col_hi, NB_JCOLS);
  if (i_hi <= i_lo || col_hi == col_lo) return CQ_OK;
  return nbody_partial(st, pos, n, part, i_lo, i_hi, eps2, col_lo, col_hi);
}

int cq_nbody_kick_finalize(int device, int stream, const float* part, const float* vel_in, float* vel,
                           int64_t count, float dt) {
  CQ_GET_STREAM(device, stream);
  if (count <= 0) return CQ_OK;
  nbody_kick_finalize<<<grid_for(count, 256, ds->sm_count, 8), 256, 0, st>>>(
      part, (const float4*)vel_in, (float4*)vel, count, dt);
  CQ_CHECK_LAUNCH();
  return CQ_OK;
}

int cq_nbody_drift(int device, int stream, const float* p_in, const float* v, float* p,
                   int64_t count, float dt) {
  CQ_GET_STREAM(device, stream);
  if (count <= 0) return CQ_OK;
  nbody_drift_kernel<<<grid_for(count, 256, ds->sm_count, 8), 256, 0, st>>>(
      (const float4*)p_in, (const float4*)v, (float4*)p, count, dt);
  CQ_CHECK_LAUNCH();
  return CQ_OK;
}

}  // extern "C"
