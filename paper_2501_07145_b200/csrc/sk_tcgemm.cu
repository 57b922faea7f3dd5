// FP32-accurate GEMM on the 5th-generation tensor cores (tcgen05, sm_100a):
// 3xTF32 split products accumulated in TMEM.
//
//   C[n][m] = sum_k A[m][k] * B[n][k]     (A: Mtot x K, B: Ntot x K, row-major fp32;
//                                          C row-major with row stride ldc)
//
// Inputs arrive pre-split as hi = rna_tf32(x) and lo = rna_tf32(x - hi) (the
// pack kernels of sk_gemm.cu; an unrounded lo would be truncated by the tensor
// core), and every k-step issues three MMAs,
//   D += A_hi B_hi + A_hi B_lo + A_lo B_hi,
// which keeps ~22 mantissa bits of each product (measured c4 parity:
// tests/test_gpu_parity.py). It is the cell-value stage of the GEMM-fed path
// (the increment inner products <dx_i, dy_j> of BASELINE c4).
//
// Accuracy: the tensor core's FP32 accumulation error grows with the number
// of MMAs chained into one accumulator (measured, tools/diag_c4_precision.py:
// 48 chained MMAs -> 4.5x the FP32 SGEMM error; 12 -> SGEMM level). So the
// hi*hi products (16 MMAs for K = 128) and the ~2^-11 smaller corrections
// hi*lo + lo*hi go to two TMEM accumulators (columns 0-255 and 256-511) that
// the epilogue adds in FP32.
//
// 2-SM mode (SK_TC_PAIR, default): CTA pairs (clusters of 2) run
// tcgen05.mma.cta_group::2 with M = 256: each CTA stages its own 128 A rows
// and 128 of the tile's 256 B rows (its TMA completes on the leader's `full`
// barrier), the leader's single thread issues the MMAs for both, commits
// multicast to both CTAs' `empty` / `tmem_full` barriers, and each CTA drains
// its own 128 accumulator rows from its own TMEM (the peer's epilogue arrives
// remotely on the leader's `tmem_empty`). Per CTA this halves the B bytes
// staged per flop (3 stages of 64 KB instead of 2 of 96 KB).
//
// Structure (one CTA per SM, persistent over 128 x 256 output tiles):
//  * warp 8, one thread: TMA producer. Per stage it loads a 32-wide K slice of
//    A_hi, A_lo (128 rows) and B_hi, B_lo (256 rows) into 128B-swizzled
//    K-major shared-memory tiles and signals `full[s]` (expect-tx bytes);
//  * warp 9, one thread: MMA issuer. Per stage 4 k-steps x 3 MMAs
//    (M=128, N=256, K=8, kind::tf32); tcgen05.commit frees the stage
//    (`empty[s]`) and, after the last stage of a tile, publishes the
//    accumulators (`tmem_full`);
//  * warps 0-7: epilogue. Warp w reads TMEM lanes 32(w%4).. (= rows m of the
//    tile), columns 128(w/4)..+127 of both accumulators, 16 at a time, sums
//    them into registers, releases TMEM (`tmem_empty`, so the next tile's
//    MMAs start) and then stores: one coalesced 128-byte store per column
//    (C is written n-major, m contiguous).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <mutex>

#include "sk_common.cuh"

namespace sk {
namespace tc {

constexpr int BM = 128;          // tile rows (A side, TMEM lanes)
constexpr int BN = 256;          // tile columns (B side, TMEM columns)
#ifndef SK_TC_KC
#define SK_TC_KC 32
#endif
constexpr int KC = SK_TC_KC;     // K floats per stage (one swizzle atom row: 128 or 64 bytes)
constexpr int STAGES = 2 * 32 / KC;
constexpr int SWZ_BYTES = KC * 4;  // swizzle atom width
// PAIR: 2-SM MMA (tcgen05 cta_group::2). A cluster of two CTAs computes a
// 256 x 256 tile: each CTA stages its own 128 rows of A and 128 of the 256 B
// rows, the leader CTA issues M = 256 MMAs that read both CTAs' shared memory
// and write each CTA's 128 accumulator rows into its own TMEM. Per CTA that
// halves the B bytes staged and read from shared memory per flop.
#ifndef SK_TC_PAIR
#define SK_TC_PAIR 1
#endif
constexpr bool PAIR = SK_TC_PAIR != 0;
constexpr int NCTA = PAIR ? 2 : 1;
constexpr int B_ROWS = BN / NCTA;          // B rows staged per CTA
constexpr int A_BYTES = BM * KC * 4;       // 16 KB per part
constexpr int B_BYTES = B_ROWS * KC * 4;   // 32 KB (16 KB in PAIR mode) per part
constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
constexpr int NSTAGES = PAIR ? 3 * 32 / KC : STAGES;  // 192 KB of stages
constexpr int NTHREADS = 320;  // 8 epilogue warps, producer, MMA issuer
constexpr uint32_t TMEM_COLS = 512;

struct TcParams {
  int64_t Mtot, Ntot, ldc;  // per batch entry
  int kchunks;
  int64_t tiles_m, tiles_n, batch;
  float *C;
  int64_t c_bstride;  // floats between batch entries of C
};

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
#ifdef SK_TC_DEBUG
  for (long long it = 0;; ++it) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (ok) return;
    if (it == (1ll << 24)) {
      printf("tc hang: block %d thread %d bar %x parity %u\n", blockIdx.x, threadIdx.x,
             smem_u32(bar), parity);
      __trap();
    }
  }
#endif
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, uint64_t *bar, int c0,
                                            int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
// shared::cluster address of the same object in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
// TMA into this CTA's shared memory, completing bytes on the leader CTA's barrier
__device__ __forceinline__ void tma_load_3d_pair(void *dst, const CUtensorMap *map,
                                                 uint32_t bar_cluster, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(bar_cluster), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t bar_cluster) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster)
               : "memory");
}
// shared-memory matrix descriptor: K-major, 128B (or 64B) swizzle, 8-row
// groups 8 * SWZ_BYTES apart
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);          // start address
  d |= (uint64_t)1 << 16;                           // leading byte offset (unused for swizzled K-major)
  d |= (uint64_t)((8 * SWZ_BYTES) >> 4) << 32;      // stride byte offset: 8 rows x atom width
  d |= (uint64_t)1 << 46;                           // descriptor version (sm_100)
  d |= (uint64_t)(SWZ_BYTES == 128 ? 2 : 4) << 61;  // layout: SWIZZLE_128B / SWIZZLE_64B
  return d;
}
// instruction descriptor: D f32, A/B tf32, both K-major, M = 128 (256 in PAIR
// mode: both CTAs' rows), N = 256
constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) |
                           ((uint32_t)((BM * NCTA) >> 4) << 24);

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t acc) {
  if constexpr (PAIR)
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(IDESC), "r"(acc));
  else
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(IDESC), "r"(acc));
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
// MMA completion -> barrier (PAIR: the barrier at the same offset in both CTAs)
__device__ __forceinline__ void mma_commit(uint64_t *bar) {
  if constexpr (PAIR)
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
        " [%0], %1;" ::"r"(smem_u32(bar)),
        "h"((uint16_t)3)
        : "memory");
  else
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}

__global__ void __launch_bounds__(NTHREADS, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap mAhi, const __grid_constant__ CUtensorMap mAlo,
                   const __grid_constant__ CUtensorMap mBhi, const __grid_constant__ CUtensorMap mBlo,
                   const TcParams P) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte aligned stage buffers (swizzle atoms), then barriers
  uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t *full = (uint64_t *)(smem + NSTAGES * STAGE_BYTES);
  uint64_t *empty = full + NSTAGES;
  uint64_t *tfull = empty + NSTAGES;
  uint64_t *tempty = tfull + 2;
  uint32_t *tmem_slot = (uint32_t *)(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NSTAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&tfull[0], 1);
    mbar_init(&tempty[0], 8 * NCTA);  // one arrival per epilogue warp (of both CTAs)
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (PAIR) cluster_sync();  // both CTAs' barriers exist before any remote arrive
  if (warp == 9) {  // TMEM allocation (whole warp), owner of the dealloc
    if constexpr (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)),
                   "r"(TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)),
                   "r"(TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem_base = *tmem_slot;
  // PAIR: tile (mc, n) of the cluster covers m-tiles 2 mc (leader) and
  // 2 mc + 1; every CTA of the pair runs the same trip count
  const int rank = PAIR ? (int)cluster_rank() : 0;
  const bool leader = rank == 0;
  const int64_t tiles_mc = (P.tiles_m + NCTA - 1) / NCTA;
  const int64_t tiles_b = tiles_mc * P.tiles_n;
  const int64_t ntiles = tiles_b * P.batch;
  const int64_t cid = blockIdx.x / NCTA, ncl = gridDim.x / NCTA;

  if (warp == 8) {
    if (lane == 0) {  // TMA producer
      int s = 0;
      uint32_t ph = 0;
      for (int64_t t = cid; t < ntiles; t += ncl) {
        const int b = (int)(t / tiles_b), tt = (int)(t % tiles_b);
        const int m0 = (int)(((tt / P.tiles_n) * NCTA + rank) * BM);
        const int n0 = (int)((tt % P.tiles_n) * BN + rank * B_ROWS);
        for (int kc = 0; kc < P.kchunks; ++kc) {
          mbar_wait(&empty[s], ph ^ 1);
          uint8_t *st = smem + s * STAGE_BYTES;
          if constexpr (PAIR) {
            // both CTAs' bytes complete on the leader's `full` barrier
            const uint32_t fb = mapa(smem_u32(&full[s]), 0);
            if (leader) mbar_expect_tx(&full[s], NCTA * STAGE_BYTES);
            tma_load_3d_pair(st, &mAhi, fb, kc * KC, m0, b);
            tma_load_3d_pair(st + A_BYTES, &mAlo, fb, kc * KC, m0, b);
            tma_load_3d_pair(st + 2 * A_BYTES, &mBhi, fb, kc * KC, n0, b);
            tma_load_3d_pair(st + 2 * A_BYTES + B_BYTES, &mBlo, fb, kc * KC, n0, b);
          } else {
            mbar_expect_tx(&full[s], STAGE_BYTES);
            tma_load_3d(st, &mAhi, &full[s], kc * KC, m0, b);
            tma_load_3d(st + A_BYTES, &mAlo, &full[s], kc * KC, m0, b);
            tma_load_3d(st + 2 * A_BYTES, &mBhi, &full[s], kc * KC, n0, b);
            tma_load_3d(st + 2 * A_BYTES + B_BYTES, &mBlo, &full[s], kc * KC, n0, b);
          }
          if (++s == NSTAGES) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 9) {
    if (lane == 0 && leader) {  // MMA issuer (PAIR: the leader CTA issues for both)
      int s = 0;
      uint32_t ph = 0, aph = 0;
      const uint32_t acc_main = tmem_base, acc_corr = tmem_base + (uint32_t)BN;
      for (int64_t t = cid; t < ntiles; t += ncl) {
        mbar_wait(&tempty[0], aph ^ 1);  // epilogue has drained the accumulators
        asm volatile("tcgen05.fence::after_thread_sync;");
        for (int kc = 0; kc < P.kchunks; ++kc) {
          mbar_wait(&full[s], ph);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint32_t sa = smem_u32(smem + s * STAGE_BYTES);
          const uint32_t sahi = sa, salo = sa + A_BYTES, sbhi = sa + 2 * A_BYTES,
                         sblo = sa + 2 * A_BYTES + B_BYTES;
#pragma unroll
          for (int ks = 0; ks < KC / 8; ++ks) {  // k-step of 8 tf32 = 32 bytes into the atom
            const uint32_t off = ks * 32;
            const uint64_t dah = sw128_desc(sahi + off), dal = sw128_desc(salo + off);
            const uint64_t dbh = sw128_desc(sbhi + off), dbl = sw128_desc(sblo + off);
            const uint32_t acc = (kc == 0 && ks == 0) ? 0u : 1u;
            mma_tf32(acc_corr, dal, dbh, acc);
            mma_tf32(acc_corr, dah, dbl, 1u);
            mma_tf32(acc_main, dah, dbh, acc);
          }
          mma_commit(&empty[s]);  // stage s is free once these MMAs retire
          if (++s == NSTAGES) {
            s = 0;
            ph ^= 1;
          }
        }
        mma_commit(&tfull[0]);  // both accumulators complete
        aph ^= 1;
      }
    }
  } else {  // epilogue warps 0-7: TMEM lanes 32*(warp%4).., columns 128*(warp/4)..
    const int quad = warp & 3, half = warp >> 2;
    uint32_t aph = 0;
    const uint32_t tempty_leader = PAIR ? mapa(smem_u32(&tempty[0]), 0) : 0u;
    for (int64_t t = cid; t < ntiles; t += ncl) {
      const int64_t b = t / tiles_b, tt = t % tiles_b;
      const int64_t m0 = ((tt / P.tiles_n) * NCTA + rank) * BM, n0 = (tt % P.tiles_n) * BN + 128 * half;
      float *Cb = P.C + b * P.c_bstride;
      mbar_wait(&tfull[0], aph);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t taddr = tmem_base + ((uint32_t)(quad * 32) << 16) + (uint32_t)(128 * half);
      float out[128];
#pragma unroll
      for (int c0 = 0; c0 < 128; c0 += 32) {  // two 16-column chunks of both accumulators per wait
        uint32_t v0[16], v1[16], w0[16], w1[16];
        tmem_ld16(taddr + (uint32_t)c0, v0);
        tmem_ld16(taddr + (uint32_t)(c0 + 16), v1);
        tmem_ld16(taddr + (uint32_t)(BN + c0), w0);
        tmem_ld16(taddr + (uint32_t)(BN + c0 + 16), w1);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          out[c0 + j] = __uint_as_float(v0[j]) + __uint_as_float(w0[j]);
          out[c0 + 16 + j] = __uint_as_float(v1[j]) + __uint_as_float(w1[j]);
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) {  // TMEM free: the next tile's MMAs may start
        if constexpr (PAIR)
          mbar_arrive_cluster(tempty_leader);
        else
          mbar_arrive(&tempty[0]);
      }
      aph ^= 1;
      // C is n-major: column j of this warp is one coalesced 128-byte row
      // segment; interior tiles store without per-element bounds checks
      const int64_t m = m0 + quad * 32 + lane;
      const int64_t nvalid = P.Ntot - n0;
      float *cp = Cb + n0 * P.ldc + m;
      if (m < P.Mtot) {
        if (nvalid >= 128) {
#pragma unroll
          for (int j = 0; j < 128; ++j) __stcs(cp + j * P.ldc, out[j]);
        } else {
#pragma unroll
          for (int j = 0; j < 128; ++j)
            if (j < nvalid) __stcs(cp + j * P.ldc, out[j]);
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  __syncwarp();  // the .aligned cluster barrier needs converged warps
  if (PAIR) cluster_sync();  // the peer is done with this CTA's smem, barriers and TMEM
  if (warp == 9) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    if constexpr (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "r"(TMEM_COLS));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "r"(TMEM_COLS));
  }
}

// split x into hi = rna_tf32(x) and lo = rna_tf32(x - hi)
__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

__global__ void split_tf32_kernel(const float *__restrict__ x, int64_t n, float *__restrict__ hi,
                                  float *__restrict__ lo) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    const float v = x[t];
    const float h = tf32_rna(v);
    hi[t] = h;
    lo[t] = tf32_rna(v - h);
  }
}

namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  });
  return fn;
}

// 3-D map over `batch` row-major (rows x K) fp32 matrices, box KC x box_rows x 1,
// 128B swizzle (rows beyond `rows` and K beyond `K` read as zeros)
int make_map(CUtensorMap *map, const float *base, int64_t rows, int K, int64_t batch, int box_rows) {
  auto fn = encode_fn();
  if (!fn) return fail(SK_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {(cuuint64_t)K, (cuuint64_t)rows, (cuuint64_t)batch};
  cuuint64_t strides[2] = {(cuuint64_t)K * 4, (cuuint64_t)rows * K * 4};
  cuuint32_t box[3] = {(cuuint32_t)KC, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void *)base, dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE,
                  SWZ_BYTES == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(SK_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return SK_OK;
}

}  // namespace
}  // namespace tc

int tf32_split(const float *x, int64_t n, float *hi, float *lo, cudaStream_t st) {
  if (n <= 0) return SK_OK;
  const int64_t blocks = std::min<int64_t>((n + 255) / 256, (int64_t)sm_count() * 16);
  tc::split_tf32_kernel<<<(unsigned)blocks, 256, 0, st>>>(x, n, hi, lo);
  SK_CHECK_LAUNCH();
  return SK_OK;
}

int tc_gemm_3xtf32(const float *Ahi, const float *Alo, int64_t Mtot, const float *Bhi,
                   const float *Blo, int64_t Ntot, int K, float *C, int64_t ldc, int64_t batch,
                   int64_t c_bstride, cudaStream_t st) {
  using namespace tc;
  if (Mtot <= 0 || Ntot <= 0 || batch <= 0) return SK_OK;
  if (K % 4) return fail(SK_ERR_INVALID, "tc_gemm: K must be a multiple of 4");
  CUtensorMap mAhi, mAlo, mBhi, mBlo;
  int rc;
  if ((rc = make_map(&mAhi, Ahi, Mtot, K, batch, BM)) || (rc = make_map(&mAlo, Alo, Mtot, K, batch, BM)) ||
      (rc = make_map(&mBhi, Bhi, Ntot, K, batch, B_ROWS)) ||
      (rc = make_map(&mBlo, Blo, Ntot, K, batch, B_ROWS)))
    return rc;
  TcParams P;
  P.Mtot = Mtot;
  P.Ntot = Ntot;
  P.ldc = ldc;
  P.kchunks = (K + KC - 1) / KC;
  P.tiles_m = (Mtot + BM - 1) / BM;
  P.tiles_n = (Ntot + BN - 1) / BN;
  P.batch = batch;
  P.c_bstride = c_bstride;
  P.C = C;
  const size_t smem = 1024 + (size_t)NSTAGES * STAGE_BYTES + 256;
  SK_CHECK_CUDA(cudaFuncSetAttribute(tc_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
  const int64_t clusters = ((P.tiles_m + NCTA - 1) / NCTA) * P.tiles_n * batch;
  cudaLaunchConfig_t lc = {};
  lc.blockDim = dim3(NTHREADS);
  lc.dynamicSmemBytes = smem;
  lc.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = NCTA;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  lc.attrs = attr;
  lc.numAttrs = 1;
  // persistent grid: as many CTA pairs as can be co-resident (cached per device)
  static std::atomic<int> resident_by_dev[64];
  int dev = 0;
  SK_CHECK_CUDA(cudaGetDevice(&dev));
  int resident = dev < 64 ? resident_by_dev[dev].load() : 0;
  if (resident == 0) {
    lc.gridDim = dim3((unsigned)(sm_count() / NCTA * NCTA));
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, (void *)tc_gemm_kernel, &lc) != cudaSuccess || n < 1) {
      (void)cudaGetLastError();
      n = sm_count() / NCTA;
    }
    resident = n;
    if (dev < 64) resident_by_dev[dev].store(n);
  }
  lc.gridDim = dim3((unsigned)(std::min<int64_t>(clusters, resident) * NCTA));
  SK_CHECK_CUDA(cudaLaunchKernelEx(&lc, tc_gemm_kernel, mAhi, mAlo, mBhi, mBlo, P));
  return SK_OK;
}

}  // namespace sk

// Development entry (tests/test_gpu_parity.py::test_tc_gemm_*): C = A B^T with
// fp32 inputs split here into hi/lo. Not part of the public ABI header.
extern "C" __attribute__((visibility("default"))) int sk_dev_tc_gemm(
    const float *A, int64_t M, const float *B, int64_t N, int32_t K, float *C, int64_t ldc,
    float *scratch, void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  float *ahi = scratch, *alo = ahi + M * K, *bhi = alo + M * K, *blo = bhi + N * K;
  int rc = sk::tf32_split(A, M * K, ahi, alo, st);
  if (!rc) rc = sk::tf32_split(B, N * K, bhi, blo, st);
  if (!rc) rc = sk::tc_gemm_3xtf32(ahi, alo, M, bhi, blo, N, K, C, ldc, 1, 0, st);
  return rc;
}
