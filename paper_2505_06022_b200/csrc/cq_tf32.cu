// 3xTF32 SGEMM on the 5th-generation tensor cores (tcgen05 + TMEM + TMA).
//
// C[m,n] = A[m,k] . B[k,n] in fp32 accuracy from TF32 products:
//   a = a_hi + a_lo with a_hi = a with the low 13 mantissa bits cleared
//   (exactly representable in TF32) and a_lo = a - a_hi (exact in fp32);
//   C ~= a_hi*b_hi + a_hi*b_lo + a_lo*b_hi   (a_lo*b_lo ~ 2^-22 |ab| dropped)
// accumulated in fp32 in TMEM.  This is the matmul of BASELINE config 3
// (slice-mapped): the normalised error |C - C64| / sum|a||b|
// stays ~1e-8, where plain 1xTF32 (~5e-6 at K = 16384) fails the 1e-6 bar.
//
// Structure (one CTA per 128 x BN output tile, 1 CTA / SM):
//   split pass : A -> A_lo ([m,k], K-major; A is its own hi operand); B ->
//                B_lo ([k,n]; B its own hi, read MN-major by the CTA-pair
//                kernel) or Bt_hi, Bt_lo ([n,k], transposed to K-major);
//   warp 0     : TMA producer, 4 tiles (A_hi, A_lo, B_hi, B_lo) per 32-wide k
//                block into a STAGES-deep ring, 128-byte swizzle;
//   warp 1     : TMEM allocator + single-thread tcgen05.mma issuer,
//                3 MMAs (M=128, N=BN, K=8) per 8-wide k step, commits free the
//                smem stage; every `group_kb` k blocks the accumulator buffer
//                (one of two in TMEM) is handed to the epilogue;
//   warps 2..  : 4*BN/64 epilogue warps (32 rows x 64 columns each) drain
//                each finished group with tcgen05.ld into fp32 registers
//                (round-to-nearest adds), then store C once.
#include <cuda.h>
#include <cstdlib>
#include <cudaTypedefs.h>

#include "cq_common.cuh"

namespace cq {
namespace tf32 {

constexpr int BM = 128;
// BK (fp32 per k block) is a template parameter: 32 -> 128-byte swizzle
// atoms (one row = one k block), 16 -> 64-byte atoms (half-size stages,
// twice as many in flight).

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ void prefetch_map(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}

// K-major operand tile, 128-byte swizzle: rows of 128 B, 8-row groups 1024 B
// apart (SBO), LBO unused for swizzled K-major; descriptor version 1 (sm_100).
template <int BK>
__device__ __forceinline__ uint64_t smem_desc(const void* tile) {
  uint64_t addr = smem_u32(tile);
  uint64_t d = 0;
  d |= (addr & 0x3FFFFull) >> 4;          // start address      [0,14)
  d |= (uint64_t)1 << 16;                  // LBO (ignored)      [16,30)
  d |= (uint64_t)((8 * BK * 4) >> 4) << 32; // SBO: 8-row group  [32,46)
  d |= (uint64_t)1 << 46;                  // version            [46,48)
  d |= (uint64_t)(BK == 32 ? 2 : 4) << 61; // SWIZZLE_128B / 64B [61,64)
  return d;
}

// MN-major operand tile straight from a row-major [k, n] matrix: 32-column
// chunks (128 B per k row) one TMA box each, BK rows deep, in the 128-byte
// swizzle with 32-byte atoms (the only MN-major smem layout kind::tf32 takes:
// 4 k rows x 128 B, 32-byte chunks XORed with k % 4).  LBO = the distance
// between n chunks (one box, BK * 128 B), SBO = between 4-row k groups
// (512 B); layout type 1 = SWIZZLE_128B_BASE32B.  The encoding was pinned
// on one MMA against a CPU product (scripts/r02/micro/umma_mn.cu,
// profiles/r02/tf32_mn_major_descriptor_micro.log).
template <int BK>
__device__ __forceinline__ uint64_t smem_desc_mn(const void* tile) {
  uint64_t addr = smem_u32(tile);
  uint64_t d = 0;
  d |= (addr & 0x3FFFFull) >> 4;            // start address      [0,14)
  d |= (uint64_t)((BK * 128) >> 4) << 16;   // LBO: n chunk       [16,30)
  d |= (uint64_t)(512 >> 4) << 32;          // SBO: 4-row k group [32,46)
  d |= (uint64_t)1 << 46;                   // version            [46,48)
  d |= (uint64_t)1 << 61;                   // SWIZZLE_128B_BASE32B
  return d;
}

// kind::tf32 instruction descriptor: F32 accumulate, TF32 A/B, A K-major,
// B K-major or (b_mn) MN-major.
__host__ __device__ constexpr uint32_t instr_desc(int m, int n, bool b_mn = false) {
  return (1u << 4)                    // c_format = F32
         | (2u << 7)                  // a_format = TF32
         | (2u << 10)                 // b_format = TF32
         | (b_mn ? (1u << 16) : 0u)   // b_major = MN
         | ((uint32_t)(n >> 3) << 17)  // N >> 3
         | ((uint32_t)(m >> 4) << 24); // M >> 4
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// TMA load of one box into the same smem offset of every CTA in `mask`,
// completing bytes on each destination CTA's mbarrier at the same offset.
__device__ __forceinline__ void tma_load_2d_mc(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                               uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "h"(mask)
      : "memory");
}

// MMA completion -> arrive on the mbarrier at this offset in every CTA of `mask`
__device__ __forceinline__ void mma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// The tensor core's fp32 accumulation truncates; a single TMEM accumulator
// over K = 16384 (6144 MMAs) builds a bias of ~6e-6 (normalised).  So K is
// processed in groups of `group_kb` 32-wide k blocks: each group accumulates
// in one of two TMEM buffers while the epilogue warps drain the other into
// round-to-nearest fp32 registers (FADD).  Error ~1e-7 at K = 16384.
template <int BN>
struct Epi {
  static constexpr int kWarps = 4 * (BN / 64);   // 32 rows x 64 columns each
  static constexpr int kThreads = 64 + 32 * kWarps;
  static constexpr uint32_t kTmemCols = 2 * BN;  // double-buffered accumulator
};

template <int BN, int STAGES, int BK>
struct Smem {
  float a_hi[STAGES][BM * BK];
  float a_lo[STAGES][BM * BK];
  float b_hi[STAGES][BN * BK];
  float b_lo[STAGES][BN * BK];
  uint64_t full[STAGES];
  uint64_t empty[STAGES];
  uint64_t tfull[2];
  uint64_t tempty[2];
  uint32_t tmem_base;
};

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

// MC = CTAs per cluster along M sharing one B tile: each loads BN/MC rows of
// B (hi and lo) and multicasts them to all MC CTAs, so per-CTA TMA traffic
// per k block drops from 32*(BM+BN)*8 to 32*(BM+BN/MC)*8 bytes.
template <int BN, int STAGES, int MC, int BK>
__global__ void __launch_bounds__(Epi<BN>::kThreads, 1)
    sgemm_3xtf32_kernel(const __grid_constant__ CUtensorMap map_ahi, const __grid_constant__ CUtensorMap map_alo,
                        const __grid_constant__ CUtensorMap map_bhi, const __grid_constant__ CUtensorMap map_blo,
                        float* __restrict__ C, int64_t ldc, int m, int n, int k, int group_kb) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte alignment for the 128-byte swizzle atoms
  Smem<BN, STAGES, BK>& S = *reinterpret_cast<Smem<BN, STAGES, BK>*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile_n = blockIdx.x, tile_m = blockIdx.y;
  const int num_kb = (k + BK - 1) / BK;
  const int num_groups = (num_kb + group_kb - 1) / group_kb;
  constexpr uint32_t kStageBytes = (2 * BM * BK + 2 * BN * BK) * sizeof(float);

  if (warp == 0 && lane == 0) {
    prefetch_map(&map_ahi);
    prefetch_map(&map_alo);
    prefetch_map(&map_bhi);
    prefetch_map(&map_blo);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&S.full[s], 1);
      mbar_init(&S.empty[s], MC);  // the stage is free once every consumer CTA is done
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&S.tfull[b], 1);
      mbar_init(&S.tempty[b], Epi<BN>::kWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&S.tmem_base)),
                 "r"(Epi<BN>::kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (MC > 1) cluster_sync();  // peers' barriers are initialised before any multicast
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = S.tmem_base;
  const uint32_t crank = MC > 1 ? cluster_rank() : 0;
  constexpr uint16_t kMask = (uint16_t)((1u << MC) - 1);
  constexpr int kBRows = BN / MC;

  if (warp == 0) {
    if (lane == 0) {
      for (int kb = 0; kb < num_kb; ++kb) {
        const int s = kb % STAGES;
        const uint32_t phase = (kb / STAGES) & 1;
        mbar_wait(&S.empty[s], phase ^ 1);
        mbar_expect_tx(&S.full[s], kStageBytes);
        const int kc = kb * BK;
        tma_load_2d(S.a_hi[s], &map_ahi, &S.full[s], kc, tile_m * BM);
        tma_load_2d(S.a_lo[s], &map_alo, &S.full[s], kc, tile_m * BM);
        if (MC == 1) {
          tma_load_2d(S.b_hi[s], &map_bhi, &S.full[s], kc, tile_n * BN);
          tma_load_2d(S.b_lo[s], &map_blo, &S.full[s], kc, tile_n * BN);
        } else {
          const int row = tile_n * BN + (int)crank * kBRows;
          tma_load_2d_mc(S.b_hi[s] + crank * kBRows * BK, &map_bhi, &S.full[s], kc, row, kMask);
          tma_load_2d_mc(S.b_lo[s] + crank * kBRows * BK, &map_blo, &S.full[s], kc, row, kMask);
        }
      }
      if (MC > 1) {
        // producer tail: every consumer arrive on this CTA's stage barriers
        // has landed before the CTA may exit
        for (int kb = num_kb; kb < num_kb + STAGES; ++kb) {
          mbar_wait(&S.empty[kb % STAGES], ((kb / STAGES) & 1) ^ 1);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = instr_desc(BM, BN);
      int kb = 0;
      for (int g = 0; g < num_groups; ++g) {
        const int buf = g & 1;
        mbar_wait(&S.tempty[buf], ((g >> 1) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t acc_addr = tmem + (uint32_t)(buf * BN);
        const int kb_end = min(kb + group_kb, num_kb);
        for (int first = kb; kb < kb_end; ++kb) {
          const int s = kb % STAGES;
          const uint32_t phase = (kb / STAGES) & 1;
          mbar_wait(&S.full[s], phase);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint64_t dah = smem_desc<BK>(S.a_hi[s]), dal = smem_desc<BK>(S.a_lo[s]);
          const uint64_t dbh = smem_desc<BK>(S.b_hi[s]), dbl = smem_desc<BK>(S.b_lo[s]);
#pragma unroll
          for (int kk = 0; kk < BK / 8; ++kk) {
            // advance 8 fp32 = 32 bytes inside the swizzle atom: +2 in addr>>4
            const uint64_t o = (uint64_t)(kk * 2);
            mma_tf32(acc_addr, dah + o, dbh + o, idesc, (kb != first || kk != 0) ? 1u : 0u);
            mma_tf32(acc_addr, dah + o, dbl + o, idesc, 1);
            mma_tf32(acc_addr, dal + o, dbh + o, idesc, 1);
          }
          if (MC == 1) mma_commit(&S.empty[s]);
          else mma_commit_mc(&S.empty[s], kMask);
        }
        mma_commit(&S.tfull[buf]);
      }
    }
  } else {
    // epilogue warp e: TMEM lanes 32*(warp%4).. (tile rows), columns 64*seg..
    const int e = warp - 2;
    const int lane_group = warp & 3;
    const int seg = e >> 2;
    float acc[64];
#pragma unroll
    for (int q = 0; q < 64; ++q) acc[q] = 0.f;
    for (int g = 0; g < num_groups; ++g) {
      const int buf = g & 1;
      mbar_wait(&S.tfull[buf], (g >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t base = tmem + ((uint32_t)(lane_group * 32) << 16) + (uint32_t)(buf * BN + seg * 64);
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        uint32_t r[16];
        tmem_ld16(base + (uint32_t)(h * 16), r);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int q = 0; q < 16; ++q) acc[h * 16 + q] += __uint_as_float(r[q]);
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.tempty[buf]);
    }
    const int row = tile_m * BM + lane_group * 32 + lane;
    const int col = tile_n * BN + seg * 64;
    if (row < m) {
      float* dst = C + (int64_t)row * ldc + col;
      if (col + 64 <= n && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
#pragma unroll
        for (int q = 0; q < 16; ++q)
          reinterpret_cast<float4*>(dst)[q] = make_float4(acc[4 * q], acc[4 * q + 1], acc[4 * q + 2], acc[4 * q + 3]);
      } else {
#pragma unroll
        for (int q = 0; q < 64; ++q)
          if (col + q < n) dst[q] = acc[q];
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (MC > 1) cluster_sync();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(Epi<BN>::kTmemCols));
  }
}

// ------------------------------------------------------------ 2-SM variant
// A CTA pair (cluster of 2) computes a 256 x BN tile with
// tcgen05.mma.cta_group::2 (M = 256): CTA r keeps A rows [128r, 128r+128)
// and B rows (n) [r*BN/2, (r+1)*BN/2) of the tile in its own shared memory
// (same offsets in both CTAs), the leader (r = 0) issues every MMA, and each
// CTA's TMEM receives its own 128 rows x BN columns.  Against the 1-SM kernel
// this halves the B bytes each SM stages and feeds to the tensor core per
// MMA, so per-SM shared-memory traffic drops from 5 to 3.3 KB per 8-wide k
// step of one product -- less energy per flop under the power cap.
// Tiles are rasterised in groups of `group_m` pairs down M, so a wave of
// clusters reads a compact block of A rows and B columns (L2 reuse) rather
// than all of B.
template <int BN, int STAGES, int BK>
struct Smem2 {
  float a_hi[STAGES][BM * BK];
  float a_lo[STAGES][BM * BK];
  float b_hi[STAGES][BN / 2 * BK];
  float b_lo[STAGES][BN / 2 * BK];
  uint64_t full[STAGES];
  uint64_t empty[STAGES];
  uint64_t tfull[2];
  uint64_t tempty[2];
  uint32_t tmem_base;
};

// TMA load of this CTA's half; completion bytes go to the leader's barrier
// (the peer bit of the shared::cluster address cleared).
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, uint32_t leader_bar, int c0,
                                                 int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(leader_bar), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ void mma_tf32_pair(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                              uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

// completion of the pair's MMAs -> arrive on the barrier at this offset in both CTAs
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

__device__ __forceinline__ void mbar_arrive_leader(uint64_t* bar) {
  asm volatile(
      "{\n"
      ".reg .b32 ra;\n"
      "mapa.shared::cluster.u32 ra, %0, 0;\n"
      "mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];\n"
      "}\n" ::"r"(smem_u32(bar))
      : "memory");
}

// MNB: B hi / lo are read MN-major straight from [k, n] (BN / 64 boxes of 32
// columns per CTA) instead of from the transposed [n, k] copies.
template <int BN, int STAGES, int BK, bool MNB>
__global__ void __launch_bounds__(Epi<BN>::kThreads, 1)
    sgemm_3xtf32_2sm_kernel(const __grid_constant__ CUtensorMap map_ahi, const __grid_constant__ CUtensorMap map_alo,
                            const __grid_constant__ CUtensorMap map_bhi, const __grid_constant__ CUtensorMap map_blo,
                            float* __restrict__ C, int64_t ldc, int m, int n, int k, int group_kb, int pairs_m,
                            int tiles_n, int group_m) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  Smem2<BN, STAGES, BK>& S = *reinterpret_cast<Smem2<BN, STAGES, BK>*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = cluster_rank();
  // grouped rasterisation of (m pair, n tile) over the linear cluster index
  const int pair = blockIdx.x >> 1;
  const int per_group = group_m * tiles_n;
  const int first = (pair / per_group) * group_m;
  const int gsize = min(pairs_m - first, group_m);
  const int pm = first + (pair % per_group) % gsize;
  const int tn = (pair % per_group) / gsize;
  const int row0 = (pm * 2 + (int)crank) * BM;
  const int col0 = tn * BN;
  const int num_kb = (k + BK - 1) / BK;
  const int num_groups = (num_kb + group_kb - 1) / group_kb;
  constexpr uint32_t kStageBytes = (2 * BM * BK + 2 * (BN / 2) * BK) * sizeof(float);

  if (warp == 0 && lane == 0) {
    prefetch_map(&map_ahi);
    prefetch_map(&map_alo);
    prefetch_map(&map_bhi);
    prefetch_map(&map_blo);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&S.full[s], 1);   // the leader's expect_tx arrival; both CTAs' bytes
      mbar_init(&S.empty[s], 1);  // the leader's multicast MMA commit
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&S.tfull[b], 1);
      mbar_init(&S.tempty[b], 2 * Epi<BN>::kWarps);  // both CTAs' epilogue warps (leader's copy)
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&S.tmem_base)),
                 "r"(Epi<BN>::kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = S.tmem_base;

  if (warp == 0) {
    if (lane == 0) {
      for (int kb = 0; kb < num_kb; ++kb) {
        const int s = kb % STAGES;
        const uint32_t phase = (kb / STAGES) & 1;
        mbar_wait(&S.empty[s], phase ^ 1);
        if (crank == 0) mbar_expect_tx(&S.full[s], 2 * kStageBytes);
        const uint32_t bar = smem_u32(&S.full[s]) & 0xFEFFFFFFu;
        const int kc = kb * BK;
        tma_load_2d_pair(S.a_hi[s], &map_ahi, bar, kc, row0);
        tma_load_2d_pair(S.a_lo[s], &map_alo, bar, kc, row0);
        if constexpr (MNB) {
#pragma unroll
          for (int j = 0; j < BN / 64; ++j) {
            const int cn = col0 + (int)crank * (BN / 2) + 32 * j;
            tma_load_2d_pair(S.b_hi[s] + j * 32 * BK, &map_bhi, bar, cn, kc);
            tma_load_2d_pair(S.b_lo[s] + j * 32 * BK, &map_blo, bar, cn, kc);
          }
        } else {
          tma_load_2d_pair(S.b_hi[s], &map_bhi, bar, kc, col0 + (int)crank * (BN / 2));
          tma_load_2d_pair(S.b_lo[s], &map_blo, bar, kc, col0 + (int)crank * (BN / 2));
        }
      }
      // every multicast commit on this CTA's stage barriers has landed
      for (int kb = num_kb; kb < num_kb + STAGES; ++kb) mbar_wait(&S.empty[kb % STAGES], ((kb / STAGES) & 1) ^ 1);
    }
  } else if (warp == 1) {
    if (lane == 0 && crank == 0) {
      constexpr uint32_t idesc = instr_desc(2 * BM, BN, MNB);
      int kb = 0;
      for (int g = 0; g < num_groups; ++g) {
        const int buf = g & 1;
        mbar_wait(&S.tempty[buf], ((g >> 1) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t acc_addr = tmem + (uint32_t)(buf * BN);
        const int kb_end = min(kb + group_kb, num_kb);
        for (int first_kb = kb; kb < kb_end; ++kb) {
          const int s = kb % STAGES;
          mbar_wait(&S.full[s], (kb / STAGES) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint64_t dah = smem_desc<BK>(S.a_hi[s]), dal = smem_desc<BK>(S.a_lo[s]);
          const uint64_t dbh = MNB ? smem_desc_mn<BK>(S.b_hi[s]) : smem_desc<BK>(S.b_hi[s]);
          const uint64_t dbl = MNB ? smem_desc_mn<BK>(S.b_lo[s]) : smem_desc<BK>(S.b_lo[s]);
#pragma unroll
          for (int kk = 0; kk < BK / 8; ++kk) {
            const uint64_t o = (uint64_t)(kk * 2);             // 8 k = 32 B along a K-major row
            const uint64_t ob = MNB ? (uint64_t)(kk * 64) : o;  // 8 k rows = 1 KB of MN-major rows
            mma_tf32_pair(acc_addr, dah + o, dbh + ob, idesc, (kb != first_kb || kk != 0) ? 1u : 0u);
            mma_tf32_pair(acc_addr, dah + o, dbl + ob, idesc, 1);
            mma_tf32_pair(acc_addr, dal + o, dbh + ob, idesc, 1);
          }
          mma_commit_pair(&S.empty[s]);
        }
        mma_commit_pair(&S.tfull[buf]);
      }
    }
  } else {
    const int e = warp - 2;
    const int lane_group = warp & 3;
    const int seg = e >> 2;
    float acc[64];
#pragma unroll
    for (int q = 0; q < 64; ++q) acc[q] = 0.f;
    for (int g = 0; g < num_groups; ++g) {
      const int buf = g & 1;
      mbar_wait(&S.tfull[buf], (g >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t base = tmem + ((uint32_t)(lane_group * 32) << 16) + (uint32_t)(buf * BN + seg * 64);
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        uint32_t r[16];
        tmem_ld16(base + (uint32_t)(h * 16), r);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int q = 0; q < 16; ++q) acc[h * 16 + q] += __uint_as_float(r[q]);
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive_leader(&S.tempty[buf]);
    }
    const int row = row0 + lane_group * 32 + lane;
    const int col = col0 + seg * 64;
    if (row < m && col < n) {
      float* dst = C + (int64_t)row * ldc + col;
      if (col + 64 <= n && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
#pragma unroll
        for (int q = 0; q < 16; ++q)
          reinterpret_cast<float4*>(dst)[q] = make_float4(acc[4 * q], acc[4 * q + 1], acc[4 * q + 2], acc[4 * q + 3]);
      } else {
#pragma unroll
        for (int q = 0; q < 64; ++q)
          if (col + q < n) dst[q] = acc[q];
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  cluster_sync();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(Epi<BN>::kTmemCols));
  }
}

// ---------------------------------------------------------------- split pass
__device__ __forceinline__ float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

// A [m,k] (lda) -> hi, lo [m,k] dense (k contiguous)
__global__ void split_rows_kernel(const float* __restrict__ a, int64_t lda, float* __restrict__ hi,
                                  float* __restrict__ lo, int64_t m, int64_t k) {
  int64_t total = m * k;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = t / k, c = t % k;
    float x = a[r * lda + c];
    float h = tf32_hi(x);
    hi[t] = h;
    lo[t] = x - h;
  }
}

// A [m,k] dense -> lo only: the tensor core reads fp32 operands as TF32 by
// dropping the low 13 mantissa bits, so A itself is its hi part (checked
// bit for bit against the masked copy: tests/test_gpu_parity.py)
__global__ void split_lo_kernel(const float* __restrict__ a, float* __restrict__ lo, int64_t total) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const float x = a[t];
    lo[t] = x - tf32_hi(x);
  }
}

// B [k,n] (ldb) -> lo [k,n] dense, for the MN-major path (B is its own hi)
__global__ void split_lo_rows_kernel(const float* __restrict__ b, int64_t ldb, float* __restrict__ lo, int64_t k,
                                     int64_t n) {
  const int64_t total = k * n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const float x = b[(t / n) * ldb + t % n];
    lo[t] = x - tf32_hi(x);
  }
}

// B [k,n] (ldb) -> hi, lo transposed [n,k] dense, via 32x32 shared tiles
__global__ void split_transpose_kernel(const float* __restrict__ b, int64_t ldb, float* __restrict__ hi,
                                       float* __restrict__ lo, int64_t k, int64_t n) {
  __shared__ float tile[32][33];
  int64_t k0 = (int64_t)blockIdx.y * 32, n0 = (int64_t)blockIdx.x * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    int64_t kk = k0 + i, nn = n0 + threadIdx.x;
    tile[i][threadIdx.x] = (kk < k && nn < n) ? b[kk * ldb + nn] : 0.f;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    int64_t nn = n0 + i, kk = k0 + threadIdx.x;
    if (nn < n && kk < k) {
      float x = tile[threadIdx.x][i];
      float h = tf32_hi(x);
      hi[nn * k + kk] = h;
      lo[nn * k + kk] = x - h;
    }
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 2-D row-major fp32 [rows, cols] (cols contiguous, row pitch ld), box = [bk
// cols, box_rows]; swizzle 128 B (bk 32) / 64 B (bk 16), or 128 B with
// 32-byte atoms for the MN-major B boxes (atom32).
static int make_map(CUtensorMap* map, const float* base, int64_t rows, int64_t cols, int box_rows, int bk,
                    int64_t ld = 0, bool atom32 = false) {
  auto encode = get_encode();
  if (!encode) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return CQ_ERR_CUDA;
  }
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld ? ld : cols) * sizeof(float)};
  cuuint32_t box[2] = {(cuuint32_t)bk, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE,
                      atom32 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B
                             : (bk == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B),
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d)", (int)r);
    return CQ_ERR_CUDA;
  }
  return CQ_OK;
}

template <int BN, int STAGES, int MC, int BK>
static int launch(cudaStream_t st, const float* ahi, const float* alo, const float* bhi, const float* blo, float* c,
                  int64_t ldc, int64_t m, int64_t n, int64_t k) {
  CUtensorMap ma, mal, mb, mbl;
  CQ_TRY(make_map(&ma, ahi, m, k, BM, BK));
  CQ_TRY(make_map(&mal, alo, m, k, BM, BK));
  CQ_TRY(make_map(&mb, bhi, n, k, BN / MC, BK));
  CQ_TRY(make_map(&mbl, blo, n, k, BN / MC, BK));
  size_t smem = sizeof(Smem<BN, STAGES, BK>) + 1024;
  auto kern = sgemm_3xtf32_kernel<BN, STAGES, MC, BK>;
  CQ_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  unsigned tiles_m = (unsigned)((m + BM - 1) / BM);
  tiles_m = (tiles_m + MC - 1) / MC * MC;  // whole clusters; extra tiles load zeros, store nothing
  dim3 grid((unsigned)((n + BN - 1) / BN), tiles_m);
  int group_kb = 128 / BK;  // K = 128 per TMEM accumulation group
  if (const char* g = getenv("CQ_TF32_GROUP_KB")) group_kb = atoi(g) > 0 ? atoi(g) : group_kb;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(Epi<BN>::kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 1;
  attr[0].val.clusterDim.y = MC;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CQ_CHECK_CUDA(cudaLaunchKernelEx(&cfg, kern, ma, mal, mb, mbl, c, ldc, (int)m, (int)n, (int)k, group_kb));
  return CQ_OK;
}

// MNB: bhi is B itself ([k, n], row pitch ldb) and blo its dense [k, n] lo
// part; otherwise both are the transposed [n, k] copies.
template <int BN, int STAGES, int BK, bool MNB>
static int launch_2sm(cudaStream_t st, const float* ahi, const float* alo, const float* bhi, int64_t ldb,
                      const float* blo, float* c, int64_t ldc, int64_t m, int64_t n, int64_t k) {
  CUtensorMap ma, mal, mb, mbl;
  CQ_TRY(make_map(&ma, ahi, m, k, BM, BK));
  CQ_TRY(make_map(&mal, alo, m, k, BM, BK));
  if constexpr (MNB) {
    static_assert(BK == 32, "MN-major B boxes are 32 columns x BK rows");
    CQ_TRY(make_map(&mb, bhi, k, n, BK, 32, ldb, true));
    CQ_TRY(make_map(&mbl, blo, k, n, BK, 32, n, true));
  } else {
    CQ_TRY(make_map(&mb, bhi, n, k, BN / 2, BK));
    CQ_TRY(make_map(&mbl, blo, n, k, BN / 2, BK));
  }
  size_t smem = sizeof(Smem2<BN, STAGES, BK>) + 1024;
  auto kern = sgemm_3xtf32_2sm_kernel<BN, STAGES, BK, MNB>;
  CQ_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int pairs_m = (int)((m + 2 * BM - 1) / (2 * BM));
  const int tiles_n = (int)((n + BN - 1) / BN);
  int group_kb = 128 / BK;
  if (const char* g = getenv("CQ_TF32_GROUP_KB")) group_kb = atoi(g) > 0 ? atoi(g) : group_kb;
  int group_m = 8;
  if (const char* g = getenv("CQ_TF32_GROUP_M")) group_m = atoi(g) > 0 ? atoi(g) : group_m;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(2 * pairs_m * tiles_n));
  cfg.blockDim = dim3(Epi<BN>::kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CQ_CHECK_CUDA(cudaLaunchKernelEx(&cfg, kern, ma, mal, mb, mbl, c, ldc, (int)m, (int)n, (int)k, group_kb, pairs_m,
                                   tiles_n, group_m));
  return CQ_OK;
}

}  // namespace tf32

int sgemm_3xtf32(int device, int stream, cudaStream_t st, int sm_count, const float* a, int64_t lda,
                 const float* b, int64_t ldb, float* c, int64_t ldc, int64_t m, int64_t n, int64_t k) {
  (void)sm_count;
  CQ_REQUIRE(k % 4 == 0, "3xTF32 sgemm needs k %% 4 == 0 (16-byte TMA row pitch)");
  CQ_REQUIRE(m < (1ll << 31) && n < (1ll << 31) && k < (1ll << 31), "3xTF32 sgemm: dims exceed int32");
  const char* bn = getenv("CQ_TF32_BN");
  const char* mc = getenv("CQ_TF32_MC");
  const char* bkv = getenv("CQ_TF32_BK");
  bool wide = n >= 256 && !(bn && atoi(bn) == 128);
  bool multicast = !(mc && atoi(mc) == 1);
  bool bk16 = bkv && atoi(bkv) == 16;
  const char* pair = getenv("CQ_TF32_2SM");
  bool two_sm = wide && !(pair && atoi(pair) == 0);
  // The CTA-pair kernel reads B MN-major straight from [k, n] when its rows
  // are 16-byte aligned (TMA pitch): B itself is the hi operand and the
  // split pass writes only its lo part, untransposed.
  const char* mnbv = getenv("CQ_TF32_MNB");
  const bool mnb = two_sm && !(mnbv && mnbv[0] == '0') && ldb % 4 == 0 && n % 4 == 0 &&
                   (reinterpret_cast<uintptr_t>(b) & 15) == 0;
  // scratch for the split operands, reused across calls: A_lo [m,k] (A is its
  // own hi part when dense -- the MMA truncates to TF32 -- else A_hi as
  // well), then B_lo [k,n] (MN-major path) or Bt_hi, Bt_lo [n,k]
  const char* rawv = getenv("CQ_TF32_RAW_HI");
  const bool raw_hi = lda == k && !(rawv && rawv[0] == '0');
  float* scratch = nullptr;
  size_t bytes = (size_t)((raw_hi ? 1 : 2) * m + (mnb ? 1 : 2) * n) * (size_t)k * sizeof(float);
  CQ_TRY(cq::scratch(device, stream, 0, bytes, (void**)&scratch));
  const float* ahi = raw_hi ? a : scratch;
  float* alo = raw_hi ? scratch : scratch + m * k;
  float* bhi = alo + m * k;
  float* blo = bhi + n * k;
  if (raw_hi)
    tf32::split_lo_kernel<<<sm_count * 8, 256, 0, st>>>(a, alo, m * k);
  else
    tf32::split_rows_kernel<<<sm_count * 8, 256, 0, st>>>(a, lda, scratch, alo, m, k);
  CQ_CHECK_LAUNCH();
  if (mnb) {
    float* blo_kn = alo + m * k;
    if (ldb == n)
      tf32::split_lo_kernel<<<sm_count * 8, 256, 0, st>>>(b, blo_kn, k * n);
    else
      tf32::split_lo_rows_kernel<<<sm_count * 8, 256, 0, st>>>(b, ldb, blo_kn, k, n);
    CQ_CHECK_LAUNCH();
    return tf32::launch_2sm<256, 3, 32, true>(st, ahi, alo, b, ldb, blo_kn, c, ldc, m, n, k);
  }
  dim3 tg((unsigned)((n + 31) / 32), (unsigned)((k + 31) / 32));
  tf32::split_transpose_kernel<<<tg, dim3(32, 8), 0, st>>>(b, ldb, bhi, blo, k, n);
  CQ_CHECK_LAUNCH();
  int status;
  if (two_sm)
    status = tf32::launch_2sm<256, 3, 32, false>(st, ahi, alo, bhi, k, blo, c, ldc, m, n, k);
  else if (wide && bk16)
    status = multicast ? tf32::launch<256, 4, 2, 16>(st, ahi, alo, bhi, blo, c, ldc, m, n, k)
                       : tf32::launch<256, 4, 1, 16>(st, ahi, alo, bhi, blo, c, ldc, m, n, k);
  else if (wide)
    status = multicast ? tf32::launch<256, 2, 2, 32>(st, ahi, alo, bhi, blo, c, ldc, m, n, k)
                       : tf32::launch<256, 2, 1, 32>(st, ahi, alo, bhi, blo, c, ldc, m, n, k);
  else
    status = multicast ? tf32::launch<128, 3, 2, 32>(st, ahi, alo, bhi, blo, c, ldc, m, n, k)
                       : tf32::launch<128, 3, 1, 32>(st, ahi, alo, bhi, blo, c, ldc, m, n, k);
  return status;
}

}  // namespace cq
