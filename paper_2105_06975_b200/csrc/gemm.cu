// Batched / grouped FP64 GEMM on the DMMA tensor path with a fused epilogue
//   Y = alpha * A X + beta * Z[zrow]
// used for every covariance product of the hot path:
// D x1 (B on window-0 columns, Q on the rest -- two groups in one launch),
// R x2 + H x3 (the H gather is the zrow epilogue), D c1 inside S_hat^{-1} and
// P_I, and dense-M_w model products (batched over windows).
#include <algorithm>
#include <cstdlib>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "dmma.cuh"
#include "internal.h"

namespace wf {

struct GemmLaunch {
  GemmProb p[2];
  int tiles0;       // tiles of group 0 (per batch)
  int tm[2], tn[2];
  int gm;           // raster group height (M-tiles sharing each X panel in L2)
};

// Z (the beta term) loads of the epilogues.  -DGEMM_Z_LDCG (probe r02az): L2-only loads,
// so an in-place product (Z = Y) leaves no L1 lines of rows that a later kernel rewrites
__device__ __forceinline__ double ld_z(const double *p) {
#ifdef GEMM_Z_LDCG
  return __ldcg(p);
#else
  return *p;
#endif
}
__device__ __forceinline__ double2 ld_z2(const double *p) {
#ifdef GEMM_Z_LDCG
  return __ldcg(reinterpret_cast<const double2 *>(p));
#else
  return *reinterpret_cast<const double2 *>(p);
#endif
}

template <class C, bool V16>
__global__ void __launch_bounds__(C::NT) k_gemm(const GemmLaunch L) {
  extern __shared__ __align__(16) double smem[];
  int tile = blockIdx.x;
  int gi = 0;
  if (tile >= L.tiles0) { tile -= L.tiles0; gi = 1; }
  const GemmProb &P = L.p[gi];
  const int b = blockIdx.z;
  // grouped raster: GM M-tiles per group share X panels in L2 while the group's A
  // rows stay resident (ncu r01b: GM = 8 re-read X 8x from DRAM at configs[3])
  const int tm_all = L.tm[gi], tn_all = L.tn[gi];
  const int GM = L.gm;
  int group = tile / (GM * tn_all);
  int first_m = group * GM;
  int gsize = min(tm_all - first_m, GM);
  int tm = first_m + (tile % (GM * tn_all)) % gsize;
  int tn = (tile % (GM * tn_all)) / gsize;
  const int m0 = tm * C::BM, n0 = tn * C::BN;

  const double *A = P.A + (int64_t)b * P.sA;
  const double *X = P.X + (int64_t)b * P.sX;
  double *Y = P.Y + (int64_t)b * P.sY;
  const double *Z = P.Z ? P.Z + (int64_t)b * P.sZ : nullptr;

  double acc[C::FM][C::FN][2];
#pragma unroll
  for (int i = 0; i < C::FM; ++i)
#pragma unroll
    for (int j = 0; j < C::FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  if (P.kr) {   // banded A: only the K tiles its rows meet (zeros skipped exactly)
    int lo[2], hi[2];
    const int nint = kr_intervals(P.kr, m0, min(C::BM, P.M - m0), P.kr_c0, 0, P.K, lo, hi);
    for (int q = 0; q < nint; ++q)
      tile_mainloop<C, V16>(smem, acc, A, P.lda, X, P.ldx, m0, n0, lo[q], hi[q], P.M, P.N);
  } else {
    tile_mainloop<C, V16>(smem, acc, A, P.lda, X, P.ldx, m0, n0, 0, P.K, P.M, P.N);
  }

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = warp / C::WARPS_N, wn = warp % C::WARPS_N;
  const int g = lane >> 2, t = lane & 3;
  const bool y16 = pair_aligned(Y, P.ldy);
  const bool z16 = Z && pair_aligned(Z, P.ldz);
#pragma unroll
  for (int i = 0; i < C::FM; ++i) {
    int row = m0 + wm * C::WM + i * 8 + g;
    if (row >= P.M) continue;
    int zr = Z ? (P.zrow ? P.zrow[row] : row) : 0;
#pragma unroll
    for (int j = 0; j < C::FN; ++j) {
      const int col = n0 + wn * C::WN + j * 8 + 2 * t;
      double v[2] = {P.alpha * acc[i][j][0], P.alpha * acc[i][j][1]};
      if (Z) {
        const double *zp = Z + (int64_t)zr * P.ldz + col;
        if (z16 && col + 1 < P.N) {
          const double2 z = ld_z2(zp);
          v[0] += P.beta * z.x;
          v[1] += P.beta * z.y;
        } else {
          if (col < P.N) v[0] += P.beta * ld_z(zp);
          if (col + 1 < P.N) v[1] += P.beta * ld_z(zp + 1);
        }
      }
      store_pair(Y + (int64_t)row * P.ldy + col, col, P.N, v[0], v[1], y16);
    }
  }
}

// ------------------------------------------------------------------ stream-K hybrid
// Wave quantisation: 4160 tiles on 296 resident CTAs is 14.05 waves, run as 15
// (configs[3]'s D product; the TRSM couplings and the R product lose 4-14% the
// same way).  The hybrid launch keeps G = 296 persistent CTAs: CTA c first runs
// the data-parallel tiles c, c+G, ... of all but the last (G + r) tiles, then an
// equal share of the remaining tiles' k-iterations (stream-K).  A tile split
// between CTAs is finished by the CTA holding its last k-iteration: earlier pieces
// (each CTA has at most one, the start of its last tile) park their accumulators
// in a workspace slot and publish a flag; the finisher adds them in increasing
// CTA order (deterministic) and runs the epilogue.  Waits only ever target
// lower-numbered CTAs, which were dispatched earlier, so progress is guaranteed.
struct SkArgs {
  double *ws;                // [G][C::NT * FM*FN*2] parked partial accumulators
  unsigned *flags;           // [G]
  unsigned epoch;            // unused (kept for the layout); flags are 0 / 1, reset by
                             // their consumer, so a captured graph can replay the launch
  int G, dp_tiles, sk_tiles, nk;
  int dp_begin;              // first data-parallel tile this launch runs (dp_tiles: none)
};

template <class C>
__device__ __forceinline__ void tile_coords(const GemmLaunch &L, int tile, int &gi, int &m0,
                                            int &n0) {
  gi = 0;
  if (tile >= L.tiles0) { tile -= L.tiles0; gi = 1; }
  const int tm_all = L.tm[gi], tn_all = L.tn[gi];
  const int GM = L.gm;
  int group = tile / (GM * tn_all);
  int first_m = group * GM;
  int gsize = min(tm_all - first_m, GM);
  int tm = first_m + (tile % (GM * tn_all)) % gsize;
  int tn = (tile % (GM * tn_all)) / gsize;
  m0 = tm * C::BM;
  n0 = tn * C::BN;
}

template <class C>
__device__ __forceinline__ void tile_epilogue(const GemmProb &P, int m0, int n0,
                                              const double (&acc)[C::FM][C::FN][2]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = warp / C::WARPS_N, wn = warp % C::WARPS_N;
  const int g = lane >> 2, t = lane & 3;
  const bool y16 = pair_aligned(P.Y, P.ldy);
  const bool z16 = P.Z && pair_aligned(P.Z, P.ldz);
#pragma unroll
  for (int i = 0; i < C::FM; ++i) {
    int row = m0 + wm * C::WM + i * 8 + g;
    if (row >= P.M) continue;
    int zr = P.Z ? (P.zrow ? P.zrow[row] : row) : 0;
#pragma unroll
    for (int j = 0; j < C::FN; ++j) {
      const int col = n0 + wn * C::WN + j * 8 + 2 * t;
      double v[2] = {P.alpha * acc[i][j][0], P.alpha * acc[i][j][1]};
      if (P.Z) {
        const double *zp = P.Z + (int64_t)zr * P.ldz + col;
        if (z16 && col + 1 < P.N) {
          const double2 z = ld_z2(zp);
          v[0] += P.beta * z.x;
          v[1] += P.beta * z.y;
        } else {
          if (col < P.N) v[0] += P.beta * ld_z(zp);
          if (col + 1 < P.N) v[1] += P.beta * ld_z(zp + 1);
        }
      }
      store_pair(P.Y + (int64_t)row * P.ldy + col, col, P.N, v[0], v[1], y16);
    }
  }
}

template <class C, bool V16>
__global__ void __launch_bounds__(C::NT) k_gemm_sk(const GemmLaunch L, const SkArgs S) {
  extern __shared__ __align__(16) double smem[];
  const int c = blockIdx.x;
  constexpr int NACC = C::FM * C::FN * 2;
  double acc[C::FM][C::FN][2];
  auto zero = [&]() {
#pragma unroll
    for (int i = 0; i < C::FM; ++i)
#pragma unroll
      for (int j = 0; j < C::FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  };
  // ---- stream-K part first: iterations [range_lo(c), range_lo(c+1)) of the sk
  // tiles.  Every range spans >= nk iterations, so it holds at most: the END piece of
  // a tile started by CTA c-1 (c finishes it), full tiles, and the START piece of a
  // tile CTA c+1 finishes.  The start piece is computed and published FIRST, the
  // finisher piece LAST, so a finisher never waits behind its neighbour's full tiles.
  const int64_t T = (int64_t)S.sk_tiles * S.nk;
  auto range_lo = [&](int cc) { return (int64_t)cc * T / S.G; };
  const int64_t it0 = range_lo(c), it1 = range_lo(c + 1);
  auto piece = [&](int lt, int kb, int ke) {
    int gi, m0, n0;
    tile_coords<C>(L, S.dp_tiles + lt, gi, m0, n0);
    const GemmProb &P = L.p[gi];
    zero();
    tile_mainloop<C, V16>(smem, acc, P.A, P.lda, P.X, P.ldx, m0, n0, kb * C::BK,
                          min(P.K, ke * C::BK), P.M, P.N);
    if (ke < S.nk) {
      // start piece: park the accumulators, publish
      double *slot = S.ws + (int64_t)c * C::NT * NACC;
      int q = 0;
#pragma unroll
      for (int i = 0; i < C::FM; ++i)
#pragma unroll
        for (int j = 0; j < C::FN; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h, ++q) slot[(int64_t)q * C::NT + threadIdx.x] = acc[i][j][h];
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0) atomicExch(S.flags + c, 1u);
      return;
    }
    if (kb > 0) {
      // finisher: add the parked start piece(s) in a fixed order (c-1, c-2, ...)
      const int64_t tile_lo = (int64_t)lt * S.nk;
      int c0 = c;
      while (c0 > 0 && range_lo(c0) > tile_lo) --c0;
      for (int cc = c - 1; cc >= c0; --cc) {
        if (threadIdx.x == 0) {
          while (atomicAdd(S.flags + cc, 0u) != 1u) __nanosleep(64);
          // the only consumer of CTA cc's start piece: re-arm its flag for the next
          // launch on this stream (the slot is not rewritten before then)
          atomicExch(S.flags + cc, 0u);
        }
        __syncthreads();
        __threadfence();
        const double *slot = S.ws + (int64_t)cc * C::NT * NACC;
        int q = 0;
#pragma unroll
        for (int i = 0; i < C::FM; ++i)
#pragma unroll
          for (int j = 0; j < C::FN; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h, ++q)
              acc[i][j][h] += __ldcg(slot + (int64_t)q * C::NT + threadIdx.x);
      }
    }
    tile_epilogue<C>(P, m0, n0, acc);
  };
  const int lt_first = (int)(it0 / S.nk), kb_first = (int)(it0 - (int64_t)lt_first * S.nk);
  const int lt_last = (int)((it1 - 1) / S.nk);
  const int ke_last = (int)(it1 - (int64_t)lt_last * S.nk);
  const bool first_is_end = kb_first > 0;              // finisher piece
  const bool last_is_start = ke_last < S.nk;           // published piece
  if (last_is_start && !(lt_last == lt_first && first_is_end))
    piece(lt_last, lt_last == lt_first ? kb_first : 0, ke_last);
  for (int lt = lt_first + (first_is_end ? 1 : 0); lt <= lt_last - (last_is_start ? 1 : 0); ++lt)
    piece(lt, 0, S.nk);
  if (first_is_end) piece(lt_first, kb_first, lt_last == lt_first ? ke_last : S.nk);
  // ---- data-parallel part
  for (int tile = S.dp_begin + c; tile < S.dp_tiles; tile += S.G) {
    int gi, m0, n0;
    tile_coords<C>(L, tile, gi, m0, n0);
    const GemmProb &P = L.p[gi];
    zero();
    tile_mainloop<C, V16>(smem, acc, P.A, P.lda, P.X, P.ldx, m0, n0, 0, P.K, P.M, P.N);
    tile_epilogue<C>(P, m0, n0, acc);
  }
}

// ------------------------------------------------------------------ TMA-engine staging
// The same 64x128 / 4-warp DMMA tile, with the operand tiles staged by the TMA copy
// engine (cp.async.bulk, 1-D row copies into the padded, conflict-free shared layout)
// and an mbarrier ring instead of per-thread cp.async + __syncthreads: warp 0's lanes
// arm a stage's "full" barrier with its byte count and issue the row copies; every
// warp waits on "full", runs its DMMAs and arrives on the stage's "empty" barrier;
// warp 0 refills a stage once all four warps have released it.  No thread computes
// per-element addresses or bounds in the main loop.
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"((unsigned)__cvta_generic_to_shared(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n.reg .pred P;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
      "@!P bra WAIT_%=;\n}\n" ::"r"(a), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
               ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src), "r"(bytes),
               "r"((unsigned)__cvta_generic_to_shared(bar)) : "memory");
}

template <class C>
__global__ void __launch_bounds__(C::NT) k_gemm_bulk(const GemmLaunch L) {
  extern __shared__ __align__(16) double smem[];
  __shared__ __align__(8) uint64_t full[C::STAGES], empty[C::STAGES];
  int tile = blockIdx.x, gi, m0, n0;
  tile_coords<C>(L, tile, gi, m0, n0);
  const GemmProb &P = L.p[gi];
  const int b = blockIdx.z;
  const double *A = P.A + (int64_t)b * P.sA;
  const double *X = P.X + (int64_t)b * P.sX;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / C::WARPS_N, wn = warp % C::WARPS_N;
  const int nk = P.K / C::BK;                       // K % BK == 0 (host checks)
  const int rowsA = min(C::BM, P.M - m0);
  const int colsB = min(C::BN, P.N - n0);           // even (host checks)
  const unsigned bytes = (unsigned)(rowsA * C::BK * 8 + C::BK * colsB * 8);
  if (tid == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], C::NWARP);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int kt) {   // warp 0: arm + copy the rows of k-tile kt into stage kt % S
    const int s = kt % C::STAGES;
    double *sA = smem + s * C::STAGE, *sB = sA + C::A_STAGE;
    if (lane == 0) mbar_arrive_expect_tx(&full[s], bytes);
    __syncwarp();
    const int k0 = kt * C::BK;
    for (int r = lane; r < rowsA; r += 32)
      bulk_g2s(sA + r * C::LDA, A + (int64_t)(m0 + r) * P.lda + k0, C::BK * 8, &full[s]);
    for (int r = lane; r < C::BK; r += 32)
      bulk_g2s(sB + r * C::LDB, X + (int64_t)(k0 + r) * P.ldx + n0, (unsigned)colsB * 8, &full[s]);
  };
  if (warp == 0)
    for (int kt = 0; kt < C::STAGES - 1 && kt < nk; ++kt) issue(kt);
  double acc[C::FM][C::FN][2];
#pragma unroll
  for (int i = 0; i < C::FM; ++i)
#pragma unroll
    for (int j = 0; j < C::FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  for (int kt = 0; kt < nk; ++kt) {
    // refill: k-tile kt + S - 1 goes into the stage every warp released at kt - 1
    if (warp == 0 && kt + C::STAGES - 1 < nk) {
      const int kn = kt + C::STAGES - 1;
      if (kn >= C::STAGES) mbar_wait(&empty[kn % C::STAGES], ((kn / C::STAGES) - 1) & 1);
      issue(kn);
    }
    const int s = kt % C::STAGES;
    mbar_wait(&full[s], (kt / C::STAGES) & 1);
    const double *st = smem + s * C::STAGE;
    mma_stage<C>(st, st + C::A_STAGE, acc, wm, wn, lane);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  GemmProb Pb = P;
  Pb.Y = P.Y + (int64_t)b * P.sY;
  Pb.Z = P.Z ? P.Z + (int64_t)b * P.sZ : nullptr;
  tile_epilogue<C>(Pb, m0, n0, acc);
}

// ------------------------------------------------------------------ 2-D TMA staging
// The same 64x128 / 4-warp DMMA tile with each operand tile staged by ONE 2-D tensor
// copy per stage (cp.async.bulk.tensor, SASS UTMALDG) instead of 12 bounds-checked
// cp.async per thread: the SASS of the cp.async main loop spends ~6 integer
// instructions per DMMA on addresses and bounds (r02 count: 2400 IMAD/LEA/IADD3/ISETP
// per 384 DMMA), which is what keeps the DMMA pipe below cuBLAS's.  The padded,
// conflict-free fragment layout is kept without swizzling: the A box is BK + 4 = 20
// columns wide and the X box BN + 4 = 132, so the shared row strides are exactly LDA /
// LDB (the 4 extra columns are real data of the neighbouring k / n tile, never read by
// the DMMAs; past the matrix edge the TMA unit zero-fills, which also covers ragged M,
// N and K without a single bounds check in the kernel).  Stage s is armed by thread 0
// (expect_tx = both boxes' bytes) and refilled by it once every warp has released it
// (one "empty" arrival per warp).
struct TmaMaps {
  CUtensorMap a[2], x[2];   // per group: A (M x K) and X (K x N), row-major doubles
  // L2 eviction hints on the two operand streams (opt-in experiment, r02ar).  One raster
  // group of gm A row panels is re-read by every wave of the group, each X column panel
  // only by the CTAs of one wave (in k lock-step): A evict_last / X evict_first was meant to
  // keep the group's A panels resident (ncu r02ae: 1.47 GB of DRAM traffic per configs[3]
  // covariance product against 0.70 GB algorithmic); measured without effect.
  int hint;   // 1: A evict_last, X evict_first
};

__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, int c0, int c1,
                                            uint64_t *bar, unsigned long long pol) {
  if (pol) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        ".L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5;\n" ::"r"(
            (unsigned)__cvta_generic_to_shared(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"((unsigned)__cvta_generic_to_shared(bar)), "l"(pol)
        : "memory");
    return;
  }
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];\n" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"((unsigned)__cvta_generic_to_shared(bar))
      : "memory");
}

template <class C>
__global__ void __launch_bounds__(C::NT) k_gemm_tma(const GemmLaunch L,
                                                   const __grid_constant__ TmaMaps T,
                                                   const TmaMaps *Tg) {
  extern __shared__ __align__(1024) double smem[];
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + C::SMEM_DOUBLES);
  uint64_t *empty = full + C::STAGES;
  int gi, m0, n0;
  tile_coords<C>(L, blockIdx.x, gi, m0, n0);
  const GemmProb &P = L.p[gi];
  // Tg (probe r02au, WF4DVAR_TMA_DESC_GLOBAL=1): the same maps in global memory
  const CUtensorMap *ma = Tg ? &Tg->a[gi] : &T.a[gi], *mx = Tg ? &Tg->x[gi] : &T.x[gi];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / C::WARPS_N, wn = warp % C::WARPS_N;
  const int nk = (P.K + C::BK - 1) / C::BK;
  constexpr unsigned kBytes = (unsigned)(C::STAGE * sizeof(double));
  if (tid == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], C::NWARP);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  unsigned long long pol_a = 0, pol_x = 0;
  if (tid == 0 && T.hint) {
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol_a));
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol_x));
  }
  auto issue = [&](int kt) {   // thread 0
    const int s = kt % C::STAGES;
    double *sA = smem + s * C::STAGE, *sB = sA + C::A_STAGE;
    mbar_arrive_expect_tx(&full[s], kBytes);
    tma_load_2d(sA, ma, kt * C::BK, m0, &full[s], pol_a);
    tma_load_2d(sB, mx, n0, kt * C::BK, &full[s], pol_x);
  };
#ifdef TMA_FENCE
  asm volatile("fence.proxy.async.global;\n" ::: "memory");
#endif
  if (tid == 0)
    for (int kt = 0; kt < C::STAGES - 1 && kt < nk; ++kt) issue(kt);
  double acc[C::FM][C::FN][2];
#pragma unroll
  for (int i = 0; i < C::FM; ++i)
#pragma unroll
    for (int j = 0; j < C::FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  for (int kt = 0; kt < nk; ++kt) {
    if (tid == 0 && kt + C::STAGES - 1 < nk) {
      const int kn = kt + C::STAGES - 1;
      if (kn >= C::STAGES) mbar_wait(&empty[kn % C::STAGES], ((kn / C::STAGES) - 1) & 1);
      issue(kn);
    }
    const int s = kt % C::STAGES;
    mbar_wait(&full[s], (kt / C::STAGES) & 1);
    const double *st = smem + s * C::STAGE;
    mma_stage<C>(st, st + C::A_STAGE, acc, wm, wn, lane);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
#ifdef TMA_INVAL
  __syncthreads();
  if (tid == 0)
    for (int s = 0; s < C::STAGES; ++s) {
      asm volatile("mbarrier.inval.shared::cta.b64 [%0];\n" ::"r"((unsigned)__cvta_generic_to_shared(&full[s])) : "memory");
      asm volatile("mbarrier.inval.shared::cta.b64 [%0];\n" ::"r"((unsigned)__cvta_generic_to_shared(&empty[s])) : "memory");
    }
#endif
  tile_epilogue<C>(P, m0, n0, acc);
}

// host: encode the 2-D tensor maps of one problem (row-major, 16-byte aligned rows)
static bool encode_tma(CUtensorMap *map, const double *base, int64_t rows, int64_t cols,
                       int64_t ld, unsigned box_cols, unsigned box_rows) {
  static PFN_cuTensorMapEncodeTiled fn = []() -> PFN_cuTensorMapEncodeTiled {
    void *f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) !=
            cudaSuccess || q != cudaDriverEntryPointSuccess)
      return nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled>(f);
  }();
  if (!fn || ((uintptr_t)base & 15) || (ld & 1) || rows < 1 || cols < 1) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * 8};
  const cuuint32_t box[2] = {box_cols, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  // probes only (r02as): 0 = no L2 promotion, 1 = 64 B, 2 = 128 B, 3 (default) = 256 B
  static const int promo_env = env_int("WF4DVAR_TMA_L2PROMO", 3);
  const CUtensorMapL2promotion promo =
      promo_env == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
      : promo_env == 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
      : promo_env == 2 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double *>(base), dims, strides,
            box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

// Y = A X (+ Z) for the tiles [0, tiles) of L through k_gemm_tma; false (nothing
// launched) when a problem does not meet the TMA alignment rules or is banded/batched
template <class C>
static bool run_tma(Ctx &c, const GemmLaunch &L, int nprob, int tiles) {
  // 1 = every eligible GEMM; 2 (default) = not the blocked TRSM's coupling GEMMs; 3 = only
  // those.  r02y-r02ab: with the coupling GEMMs TMA-staged, configs[4]'s P_I apply
  // (R_hat^{-1} blocked TRSM on an aux stream concurrent with the L_hat chains and the D
  // product) was not reproducible -- 60 chained applies differed by up to 6e-3 between
  // runs, and GMRES histories drifted from the oracle recurrence -- while the cp.async
  // coupling GEMMs, serialised streams (WF4DVAR_FORK=0) or a single TRSM segment were
  // bitwise reproducible and equal to each other.  Root cause not identified (see
  // DESIGN.md section 10); the covariance products keep the TMA staging (reproducible in
  // every probe)
  static const int env = env_int("WF4DVAR_GEMM_TMA", 2);
  if (!env || tiles <= 0) return false;
  if (env == 2 && c.gemm_cls == K_TRSM_UPD) return false;
  if (env == 3 && c.gemm_cls != K_TRSM_UPD) return false;
  TmaMaps T{};
  for (int i = 0; i < nprob; ++i) {
    const GemmProb &p = L.p[i];
    if (p.kr) return false;
    if (!encode_tma(&T.a[i], p.A, p.M, p.K, p.lda, C::BK + 4, C::BM)) return false;
    if (!encode_tma(&T.x[i], p.X, p.K, p.N, p.ldx, C::BN + 4, C::BK)) return false;
  }
  // only where a raster group spans several waves (otherwise there is nothing to keep).
  // OPT-IN (WF4DVAR_GEMM_L2HINT=1; 2 = every TMA GEMM): r02ar measured no gain on
  // configs[3] -- DRAM reads per covariance product 1.6-1.9 GB without and 1.8-2.2 GB
  // with the hints (raster groups of 16 / 24 / 32 row panels alike), step 30.56 ms in
  // every setting
  static const int hint_env = env_int("WF4DVAR_GEMM_L2HINT", 0);
  T.hint = hint_env == 2 || (hint_env == 1 && tiles > 4 * 148 && c.gemm_cls != K_TRSM_UPD);
  // WF4DVAR_TMA_SMEM_PAD (probe r02au): extra dynamic shared memory, e.g. 40000 -> one
  // k_gemm_tma CTA per SM
  static const int pad_env = env_int("WF4DVAR_TMA_SMEM_PAD", 0);
  const size_t smem =
      C::SMEM_DOUBLES * sizeof(double) + 2 * C::STAGES * sizeof(uint64_t) + (size_t)pad_env;
  static const cudaError_t attr =
      cudaFuncSetAttribute(k_gemm_tma<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  WF_CUDA(attr);
  // WF4DVAR_TMA_CARVEOUT (probe r02aw): preferred shared-memory carve-out of the kernel in
  // percent (100 = the maximum, so the SM's L1 / shared split never changes under it)
  static const int carve_env = env_int("WF4DVAR_TMA_CARVEOUT", -1);
  static const cudaError_t attr_carve =
      carve_env >= 0 ? cudaFuncSetAttribute(k_gemm_tma<C>,
                                            cudaFuncAttributePreferredSharedMemoryCarveout, carve_env)
                     : cudaSuccess;
  WF_CUDA(attr_carve);
  // probe (r02au): descriptors read from a per-launch slot in global memory instead of the
  // kernel parameter space (slot ring: pinned host copy -> device copy on the launch stream)
  static const int desc_global = env_int("WF4DVAR_TMA_DESC_GLOBAL", 0);
  const TmaMaps *Tg = nullptr;
  if (desc_global) {
    constexpr int kSlots = 4096;
    static TmaMaps *hring = nullptr, *dring = nullptr;
    static unsigned next = 0;
    if (!hring) {
      WF_CUDA(cudaMallocHost(&hring, sizeof(TmaMaps) * kSlots));
      WF_CUDA(cudaMalloc(&dring, sizeof(TmaMaps) * kSlots));
    }
    const unsigned slot = next++ % kSlots;
    hring[slot] = T;
    WF_CUDA(cudaMemcpyAsync(dring + slot, hring + slot, sizeof(TmaMaps), cudaMemcpyHostToDevice,
                            c.st));
    Tg = dring + slot;
  }
  k_gemm_tma<C><<<tiles, C::NT, smem, c.st>>>(L, T, Tg);
  WF_CUDA(cudaGetLastError());
  return true;
}

// Large problems: 64x128 CTA tile, 4 warps of 32x64 (32 independent DMMA
// accumulator tiles per warp per k-step), BK = 16, 3-stage cp.async ring,
// 81 KB smem -> 2 CTAs (8 warps) per SM.  Chosen by measurement (tools/kbench.py,
// r01): 32.5 TFLOP/s at 4096x8128x4096 = 90% of cuBLAS DGEMM on the same box,
// vs 30.2 for 128x128/8x(64x32) and 28.7 for 128x128/8x(32x64).
using CfgHuge = TileCfg<64, 128, 16, 32, 64, 3>;
// 16 warps of 32x32 (4 per SMSP): more warps to hide LDS->DMMA latency
using CfgWide = TileCfg<128, 128, 32, 32, 32, 3>;


using CfgBig = TileCfg<128, 64, 16, 32, 32, 4>;
using CfgSmall = TileCfg<64, 32, 16, 32, 16, 4>;

template <class C>
static int tiles_of(const GemmProb &p, int &tm, int &tn) {
  tm = (p.M + C::BM - 1) / C::BM;
  tn = (p.N + C::BN - 1) / C::BN;
  return tm * tn;
}

static bool aligned16(const GemmProb &p) {
  auto al = [](const void *q) { return ((uintptr_t)q & 15) == 0; };
  return al(p.A) && al(p.X) && (p.lda % 2 == 0) && (p.ldx % 2 == 0) &&
         (p.sA % 2 == 0) && (p.sX % 2 == 0);
}

template <class C>
static void run(Ctx &c, const GemmProb *probs, int nprob, int batch, bool v16) {
  GemmLaunch L{};
  int tiles = 0;
  for (int i = 0; i < nprob; ++i) {
    L.p[i] = probs[i];
    int t = tiles_of<C>(probs[i], L.tm[i], L.tn[i]);
    if (i == 0) L.tiles0 = t;
    tiles += t;
  }
  if (nprob == 1) L.tiles0 = tiles;
  // raster group height: one wave of resident CTAs (~2 per SM) touches gm A row
  // panels and (2*148/gm) X column panels; pick the gm minimising that L2 footprint
  // (~sqrt(2*148*BN/BM)), capped at the M-tiles of the problem
  {
    static const int gm_env = env_int("WF4DVAR_GEMM_GM", -1);   // tuning experiments only
    int best = 1;
    double best_fp = 1e300;
    for (int g = 1; g <= 64; g *= 2) {
      double fp = (double)g * C::BM + std::max(1.0, 2.0 * 148 / g) * C::BN;
      if (fp <= best_fp) { best_fp = fp; best = g; }
    }
    L.gm = std::max(1, std::min(gm_env > 0 ? gm_env : best, L.tm[0]));
  }
  size_t smem = C::SMEM_DOUBLES * sizeof(double);
  // stream-K hybrid when one batch of large tiles quantises badly onto the waves
  // Split launch (default): the data-parallel waves run in the plain k_gemm (its main
  // loop keeps 214 registers and ~95% DMMA-pipe occupancy in steady state, ncu r01ak),
  // then the stream-K kernel runs only the last G + r tiles split evenly by
  // k-iterations.  The single persistent kernel (WF4DVAR_GEMM_SK=2) runs its DP tiles
  // at 254 registers / 81% pipe and lost (r01ak: 29.9 vs 30.8 TFLOP/s at
  // 4096 x 8256 x 4096).  Only when the tail wave is nearly empty (r < 0.3 G): the
  // stream-K part costs (G + r) / G tile-times at lower efficiency.
  static const int sk_env = env_int("WF4DVAR_GEMM_SK", 1);   // 0 disables
  const int G = 2 * 148;   // resident CTAs of the 64x128 / 81 KB configuration
  const int nk = (probs[0].K + C::BK - 1) / C::BK;
  bool same_k = nprob == 1 || probs[0].K == probs[1].K;
  bool banded = false;
  for (int i = 0; i < nprob; ++i) banded = banded || probs[i].kr;
  if constexpr (C::BM == 64 && C::BN == 128 && C::STAGES == 3 && C::BK == 16) {
  static const int sk_tail_env = env_int("WF4DVAR_GEMM_SK_TAIL", 30);   // percent of G
  const double sk_max_tail = sk_env == 2 ? 0.75 : sk_tail_env / 100.0;
  if (sk_env && !banded && v16 && batch == 1 && same_k && tiles > G &&
      (tiles % G) != 0 && (double)(tiles % G) / G < sk_max_tail && nk >= 8) {
    const int r = tiles % G;
    SkArgs S{};
    S.G = G;
    S.sk_tiles = G + r;
    S.dp_tiles = tiles - S.sk_tiles;
    S.nk = nk;
    constexpr int NACC = C::FM * C::FN * 2;
    const size_t need = (size_t)G * C::NT * NACC;
    // one workspace per stream: stream-K GEMMs on the fork/join streams may run
    // concurrently (D product on the main stream, D_hat / R_hat coupling GEMMs on the
    // aux streams) and must not share parked partials or flags
    Ctx::SkState *st = nullptr;
    for (auto &e : c.sk_states)
      if (e.stream == c.st) st = &e;
    if (!st) {
      c.sk_states.push_back(Ctx::SkState{});
      st = &c.sk_states.back();
      st->stream = c.st;
    }
    if (st->cap < need) {
      if (st->ws) c.retired.push_back(st->ws);
      if (st->flags) c.retired.push_back(st->flags);
      st->ws = nullptr; st->flags = nullptr; st->cap = 0;
      WF_CUDA(cudaMalloc(&st->ws, need * 8));
      WF_CUDA(cudaMalloc(&st->flags, G * sizeof(unsigned)));
      WF_CUDA(cudaMemsetAsync(st->flags, 0, G * sizeof(unsigned), c.st));
      st->cap = need;
    }
    S.ws = st->ws;
    S.flags = st->flags;
    S.epoch = 1;
    static const cudaError_t attr = cudaFuncSetAttribute(k_gemm_sk<C, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    WF_CUDA(attr);
    S.dp_begin = 0;
    if (sk_env != 2 && S.dp_tiles > 0) {
      if (!run_tma<C>(c, L, nprob, S.dp_tiles)) {
        static const cudaError_t attr_dp = cudaFuncSetAttribute(k_gemm<C, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        WF_CUDA(attr_dp);
        k_gemm<C, true><<<dim3(S.dp_tiles, 1, 1), C::NT, smem, c.st>>>(L);   // tiles [0, dp_tiles)
        WF_CUDA(cudaGetLastError());
      }
      c.launches++;
      S.dp_begin = S.dp_tiles;
    }
    k_gemm_sk<C, true><<<G, C::NT, smem, c.st>>>(L, S);
    WF_CUDA(cudaGetLastError());
    return;
  }
  }
  if constexpr (C::BM == 64 && C::BN == 128 && C::BK == 16 && C::STAGES == 3) {
    // measured r01x: 20.0 vs 32.5 TFLOP/s at 4096x8128x4096 -- 80 small (128 B / 1 KB)
    // bulk copies per stage through the copy engine cost more than the per-thread
    // cp.async issue they replace -> opt-in only (WF4DVAR_GEMM_BULK=1)
    static const int bulk_env = env_int("WF4DVAR_GEMM_BULK", 0);   // tuning experiments only
    bool ok = bulk_env && v16 && !banded;
    for (int i = 0; i < nprob; ++i)
      ok = ok && probs[i].K % C::BK == 0 && probs[i].N % 2 == 0 && probs[i].K > 0 &&
           ((uintptr_t)probs[i].A % 16 == 0) && ((uintptr_t)probs[i].X % 16 == 0);
    if (ok) {
      static const cudaError_t attr =
          cudaFuncSetAttribute(k_gemm_bulk<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      WF_CUDA(attr);
      k_gemm_bulk<C><<<dim3(tiles, 1, batch), C::NT, smem, c.st>>>(L);
      WF_CUDA(cudaGetLastError());
      return;
    }
  }
  if constexpr (C::BK == 16) {   // every BK = 16 tile shape (64x128, 128x64, 64x32)
    if (batch == 1 && !banded && run_tma<C>(c, L, nprob, tiles)) return;
  }
  dim3 grid(tiles, 1, batch);
  if (v16) {
    static const cudaError_t attr = cudaFuncSetAttribute(k_gemm<C, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    WF_CUDA(attr);
    k_gemm<C, true><<<grid, C::NT, smem, c.st>>>(L);
  } else {
    static const cudaError_t attr = cudaFuncSetAttribute(k_gemm<C, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    WF_CUDA(attr);
    k_gemm<C, false><<<grid, C::NT, smem, c.st>>>(L);
  }
  WF_CUDA(cudaGetLastError());
}

// Small operators (M, K <= 64: the s x s and p x p covariances of the L96 configs,
// s = 40, 50).  A 64x128 DMMA tile with K <= 64 never fills its cp.async ring and
// wastes most of its M rows; the product is HBM bound, so this kernel is the
// streaming form: one thread per (column, group of GR rows) streams x[0:K] of its
// column and accumulates its GR outputs (two partial sums each), the GR x K block of
// A resident in shared memory (broadcast 16-byte pairs).  The row groups of one
// column read x from L2 after the first; they exist for memory-level parallelism
// (ncu r01ad: one thread per column = 11 warps per SM, 0.5 TB/s).
constexpr int kSmallGR = 8;
template <int KMAX>
__global__ void __launch_bounds__(128) k_gemm_small(const GemmLaunch L) {
  constexpr int LD = KMAX + 2;
  __shared__ __align__(16) double sA[kSmallGR * LD];
  int chunk = blockIdx.x, gi = 0;
  if (chunk >= L.tiles0) { chunk -= L.tiles0; gi = 1; }
  const GemmProb &P = L.p[gi];
  const int r0 = blockIdx.y * kSmallGR;
  if (r0 >= P.M) return;
  const int b = blockIdx.z;
  const double *A = P.A + (int64_t)b * P.sA;
  const double *X = P.X + (int64_t)b * P.sX;
  double *Y = P.Y + (int64_t)b * P.sY;
  const double *Z = P.Z ? P.Z + (int64_t)b * P.sZ : nullptr;
  for (int e = threadIdx.x; e < kSmallGR * KMAX; e += 128) {
    const int r = e / KMAX, k = e % KMAX;
    sA[r * LD + k] = (r0 + r < P.M && k < P.K) ? A[(int64_t)(r0 + r) * P.lda + k] : 0.0;
  }
  __syncthreads();
  const int col = chunk * 128 + threadIdx.x;
  if (col >= P.N) return;
  double acc0[kSmallGR], acc1[kSmallGR];
#pragma unroll
  for (int r = 0; r < kSmallGR; ++r) acc0[r] = acc1[r] = 0.0;
#pragma unroll
  for (int k = 0; k < KMAX; k += 2) {
    const double x0 = k < P.K ? X[(int64_t)k * P.ldx + col] : 0.0;
    const double x1 = k + 1 < P.K ? X[(int64_t)(k + 1) * P.ldx + col] : 0.0;
#pragma unroll
    for (int r = 0; r < kSmallGR; ++r) {
      const double2 g = *reinterpret_cast<const double2 *>(&sA[r * LD + k]);
      acc0[r] = fma(g.x, x0, acc0[r]);
      acc1[r] = fma(g.y, x1, acc1[r]);
    }
  }
#pragma unroll
  for (int r = 0; r < kSmallGR; ++r) {
    const int row = r0 + r;
    if (row < P.M) {
      double v = P.alpha * (acc0[r] + acc1[r]);
      if (Z) v += P.beta * Z[(int64_t)(P.zrow ? P.zrow[row] : row) * P.ldz + col];
      Y[(int64_t)row * P.ldy + col] = v;
    }
  }
}

// The same small products on the FP64 tensor pipe (round 2, r02ao): with K <= 64 the
// streaming kernel above issues one FMA per multiply and one shared-memory A pair per
// two FMAs, so its issue slots, not HBM, bound it (configs[2]: 29 us per 40 x 40 x 52k
// product against ~5 us of HBM traffic).  Here each warp owns 16-column slabs of X (two
// 8-column DMMA tiles): it loads the slab's B fragments for all of K (2 KMAX / 4
// independent 8-byte loads per lane, in flight together; every 128-byte row segment is
// read by one warp), then runs ceil(M/8) x K/4 pairs of DMMA.8x8x4 against A fragments
// read from shared memory (A staged once per CTA with the conflict-free padded stride),
// and writes its M x 16 outputs (+ beta Z, 16-byte stores when aligned).  A warp owns
// ALL M rows of its columns, so the product may be in place (Y = X): every B fragment
// is in registers before the first store.  Slabs per warp are set by the host so the
// grid is ~2 waves of 8-warp CTAs.
template <int KMAX>
__global__ void __launch_bounds__(256) k_gemm_small_dmma(const GemmLaunch L, int tpw) {
  constexpr int KS = KMAX / 4, LDA = KMAX + 4;
  __shared__ __align__(16) double sA[64 * LDA];
  int chunk = blockIdx.x, gi = 0;
  if (chunk >= L.tiles0) { chunk -= L.tiles0; gi = 1; }
  const GemmProb &P = L.p[gi];
  const int b = blockIdx.z;
  const double *A = P.A + (int64_t)b * P.sA;
  const double *X = P.X + (int64_t)b * P.sX;
  double *Y = P.Y + (int64_t)b * P.sY;
  const double *Z = P.Z ? P.Z + (int64_t)b * P.sZ : nullptr;
  const int M = P.M, K = P.K, N = P.N;
  const int mt = (M + 7) / 8;
  for (int e = threadIdx.x; e < mt * 8 * KMAX; e += 256) {
    const int r = e / KMAX, k = e % KMAX;
    sA[r * LDA + k] = (r < M && k < K) ? A[(int64_t)r * P.lda + k] : 0.0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  // 16 columns per warp pass (two 8-column DMMA tiles): every 128-byte row segment of X
  // is read by one warp, and 2 KS loads per lane are in flight together
  const bool y16 = ((P.ldy & 1) == 0) && (((uintptr_t)Y & 15) == 0) &&
                   (!Z || (((P.ldz & 1) == 0) && (((uintptr_t)Z & 15) == 0)));
  for (int it = 0; it < tpw; ++it) {
    const int n0 = ((chunk * tpw + it) * 8 + warp) * 16;
    if (n0 >= N) break;
    double bf[2][KS];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int cb = n0 + 8 * h + g;            // B fragment column of this lane
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        const int k = 4 * ks + t;
        bf[h][ks] = (k < K && cb < N) ? X[(int64_t)k * P.ldx + cb] : 0.0;
      }
    }
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      if (m >= mt) break;
      double c[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        const double a = sA[(8 * m + g) * LDA + 4 * ks + t];
        dmma884(c[0][0], c[0][1], a, bf[0][ks]);
        dmma884(c[1][0], c[1][1], a, bf[1][ks]);
      }
      const int row = 8 * m + g;
      if (row >= M) continue;
      const int64_t zr = Z ? (int64_t)(P.zrow ? P.zrow[row] : row) * P.ldz : 0;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col = n0 + 8 * h + 2 * t;
        double v0 = P.alpha * c[h][0], v1 = P.alpha * c[h][1];
        if (y16 && col + 1 < N) {
          if (Z) {
            const double2 zz = *reinterpret_cast<const double2 *>(Z + zr + col);
            v0 += P.beta * zz.x;
            v1 += P.beta * zz.y;
          }
          *reinterpret_cast<double2 *>(Y + (int64_t)row * P.ldy + col) = make_double2(v0, v1);
        } else {
          if (col < N) {
            if (Z) v0 += P.beta * Z[zr + col];
            Y[(int64_t)row * P.ldy + col] = v0;
          }
          if (col + 1 < N) {
            if (Z) v1 += P.beta * Z[zr + col + 1];
            Y[(int64_t)row * P.ldy + col + 1] = v1;
          }
        }
      }
    }
  }
}

static void run_small_dmma(Ctx &c, const GemmProb *probs, int nprob, int batch, int kmax) {
  GemmLaunch L{};
  int64_t tiles = 0;   // 16-column warp tiles over all problems and the batch
  for (int i = 0; i < nprob; ++i) tiles += (int64_t)((probs[i].N + 15) / 16) * batch;
  // ~2 waves of 8-warp CTAs (each CTA stages A once; more tiles per warp amortise it)
  const int tpw = (int)std::max<int64_t>(1, tiles / (8 * 2 * 2 * 148));
  const int cols_per_cta = tpw * 128;
  int chunks = 0;
  for (int i = 0; i < nprob; ++i) {
    L.p[i] = probs[i];
    const int ci = (probs[i].N + cols_per_cta - 1) / cols_per_cta;
    if (i == 0) L.tiles0 = ci;
    chunks += ci;
  }
  if (nprob == 1) L.tiles0 = chunks;
  const dim3 grid(chunks, 1, batch);
  switch ((kmax + 7) / 8) {
    case 1: k_gemm_small_dmma<8><<<grid, 256, 0, c.st>>>(L, tpw); break;
    case 2: k_gemm_small_dmma<16><<<grid, 256, 0, c.st>>>(L, tpw); break;
    case 3: k_gemm_small_dmma<24><<<grid, 256, 0, c.st>>>(L, tpw); break;
    case 4: k_gemm_small_dmma<32><<<grid, 256, 0, c.st>>>(L, tpw); break;
    case 5: k_gemm_small_dmma<40><<<grid, 256, 0, c.st>>>(L, tpw); break;
    case 6: k_gemm_small_dmma<48><<<grid, 256, 0, c.st>>>(L, tpw); break;
    case 7: k_gemm_small_dmma<56><<<grid, 256, 0, c.st>>>(L, tpw); break;
    default: k_gemm_small_dmma<64><<<grid, 256, 0, c.st>>>(L, tpw); break;
  }
  WF_CUDA(cudaGetLastError());
}

static void run_small(Ctx &c, const GemmProb *probs, int nprob, int batch, int mmax, int kmax) {
  GemmLaunch L{};
  int chunks = 0;
  for (int i = 0; i < nprob; ++i) {
    L.p[i] = probs[i];
    const int ci = (probs[i].N + 127) / 128;
    if (i == 0) L.tiles0 = ci;
    chunks += ci;
  }
  if (nprob == 1) L.tiles0 = chunks;
  const dim3 grid(chunks, (mmax + kSmallGR - 1) / kSmallGR, batch);
  switch ((kmax + 7) / 8) {
    case 1: k_gemm_small<8><<<grid, 128, 0, c.st>>>(L); break;
    case 2: k_gemm_small<16><<<grid, 128, 0, c.st>>>(L); break;
    case 3: k_gemm_small<24><<<grid, 128, 0, c.st>>>(L); break;
    case 4: k_gemm_small<32><<<grid, 128, 0, c.st>>>(L); break;
    case 5: k_gemm_small<40><<<grid, 128, 0, c.st>>>(L); break;
    case 6: k_gemm_small<48><<<grid, 128, 0, c.st>>>(L); break;
    case 7: k_gemm_small<56><<<grid, 128, 0, c.st>>>(L); break;
    default: k_gemm_small<64><<<grid, 128, 0, c.st>>>(L); break;
  }
  WF_CUDA(cudaGetLastError());
}

// ---- split-K for GEMMs with too few tiles to fill the GPU (configs[1]: 1000 x 336 x
// 1000 is 48 tiles of 64x128 on 148 SMs).  Split z of S runs the K range
// [z kc, (z+1) kc) of every tile and parks its 64x128 partial in a per-stream
// workspace; the reduction adds the S partials in a fixed order and applies the
// epilogue (deterministic, no atomics, graph-replay safe).
template <class C, bool V16>
__global__ void __launch_bounds__(C::NT) k_gemm_splitk(const GemmLaunch L, double *ws, int kc) {
  extern __shared__ __align__(16) double smem[];
  const int tiles = gridDim.x, tile = blockIdx.x, z = blockIdx.z;
  int gi, m0, n0;
  tile_coords<C>(L, tile, gi, m0, n0);
  const GemmProb &P = L.p[gi];
  double acc[C::FM][C::FN][2];
#pragma unroll
  for (int i = 0; i < C::FM; ++i)
#pragma unroll
    for (int j = 0; j < C::FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int kb = z * kc, ke = min(P.K, kb + kc);
  if (ke > kb)
    tile_mainloop<C, V16>(smem, acc, P.A, P.lda, P.X, P.ldx, m0, n0, kb, ke, P.M, P.N);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = warp / C::WARPS_N, wn = warp % C::WARPS_N;
  const int g = lane >> 2, t = lane & 3;
  double *slot = ws + ((int64_t)z * tiles + tile) * (C::BM * C::BN);
#pragma unroll
  for (int i = 0; i < C::FM; ++i)
#pragma unroll
    for (int j = 0; j < C::FN; ++j) {
      const int rr = wm * C::WM + i * 8 + g, cc = wn * C::WN + j * 8 + 2 * t;
      *reinterpret_cast<double2 *>(slot + rr * C::BN + cc) = make_double2(acc[i][j][0], acc[i][j][1]);
    }
}

template <class C>
__global__ void k_gemm_splitk_reduce(const GemmLaunch L, const double *ws, int tiles, int S) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)tiles * C::BM * C::BN) return;
  const int tile = (int)(e / (C::BM * C::BN));
  const int loc = (int)(e % (C::BM * C::BN));
  int gi, m0, n0;
  tile_coords<C>(L, tile, gi, m0, n0);
  const GemmProb &P = L.p[gi];
  const int row = m0 + loc / C::BN, col = n0 + loc % C::BN;
  if (row >= P.M || col >= P.N) return;
  double sum = 0.0;
  for (int z = 0; z < S; ++z) sum += ws[((int64_t)z * tiles + tile) * (C::BM * C::BN) + loc];
  double v = P.alpha * sum;
  if (P.Z) v += P.beta * P.Z[(int64_t)(P.zrow ? P.zrow[row] : row) * P.ldz + col];
  P.Y[(int64_t)row * P.ldy + col] = v;
}

// true if launched (S >= 2 splits fit); the caller falls back to the tile configs
template <class C>
static bool run_splitk(Ctx &c, const GemmProb *probs, int nprob, bool v16) {
  // opt-in: r01bd measured 1000 x 320 x 1000 alone 10.5 -> 12.2 TFLOP/s, but configs[1]'s
  // step 0.318 -> 0.365 ms -- its small GEMMs already overlap on the fork/join streams,
  // and the split grids crowd out the concurrent blocks (NEXT-1: 0.898 -> 0.889 ms)
  static const int env = env_int("WF4DVAR_GEMM_SPLITK", 0);
  if (!env) return false;
  GemmLaunch L{};
  int tiles = 0, kmax = 0;
  for (int i = 0; i < nprob; ++i) {
    L.p[i] = probs[i];
    if (probs[i].kr) return false;
    const int t = tiles_of<C>(probs[i], L.tm[i], L.tn[i]);
    if (i == 0) L.tiles0 = t;
    tiles += t;
    kmax = std::max(kmax, probs[i].K);
  }
  if (nprob == 1) L.tiles0 = tiles;
  L.gm = 1;
  const int G = 2 * 148;
  // S splits of >= 8 k-steps each, S x tiles <= one wave of resident CTAs
  int S = std::min(G / std::max(1, tiles), kmax / (8 * C::BK));
  if (S < 2) return false;
  const int nk = (kmax + C::BK - 1) / C::BK;
  const int kc = ((nk + S - 1) / S) * C::BK;
  S = (kmax + kc - 1) / kc;
  if (S < 2) return false;
  Ctx::SkState *st = nullptr;
  for (auto &e : c.sk_states)
    if (e.stream == c.st) st = &e;
  if (!st) {
    c.sk_states.push_back(Ctx::SkState{});
    st = &c.sk_states.back();
    st->stream = c.st;
  }
  const size_t need = (size_t)S * tiles * C::BM * C::BN;
  if (st->splitk_cap < need) {
    if (st->splitk) c.retired.push_back(st->splitk);
    st->splitk = nullptr;
    st->splitk_cap = 0;
    WF_CUDA(cudaMalloc(&st->splitk, need * 8));
    st->splitk_cap = need;
  }
  const size_t smem = C::SMEM_DOUBLES * sizeof(double);
  auto kern = v16 ? k_gemm_splitk<C, true> : k_gemm_splitk<C, false>;
  static const cudaError_t a1 = cudaFuncSetAttribute(k_gemm_splitk<C, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  static const cudaError_t a2 = cudaFuncSetAttribute(k_gemm_splitk<C, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  WF_CUDA(v16 ? a1 : a2);
  kern<<<dim3(tiles, 1, S), C::NT, smem, c.st>>>(L, st->splitk, kc);
  WF_CUDA(cudaGetLastError());
  const int64_t nel = (int64_t)tiles * C::BM * C::BN;
  k_gemm_splitk_reduce<C><<<(unsigned)((nel + 255) / 256), 256, 0, c.st>>>(L, st->splitk, tiles, S);
  WF_CUDA(cudaGetLastError());
  c.launches++;
  return true;
}

// ---- tile column ranges (banded covariances and factors)
// flag[t][j] = 1 iff G[64 t : 64 t + 64, 16 j : 16 j + 16] has a non-zero
__global__ void k_tile_mask(const double *G, int64_t ld, int rows, int cols, unsigned char *flag) {
  const int t = blockIdx.x, nj = (cols + 15) / 16;
  for (int j = threadIdx.x; j < nj; j += blockDim.x) {
    unsigned char f = 0;
    for (int r = t * 64; r < min(rows, t * 64 + 64) && !f; ++r)
      for (int k = j * 16; k < min(cols, j * 16 + 16); ++k)
        if (G[(int64_t)r * ld + k] != 0.0) { f = 1; break; }
    flag[(int64_t)t * nj + j] = f;
  }
}

void register_tile_ranges(Ctx &c, const double *G, int rows, int cols, int64_t ld) {
  static const int env = env_int("WF4DVAR_BANDED", 1);   // 0: dense K loops always
  if (!env || !G || rows <= 0 || cols <= 0) return;
  unregister_tile_ranges(c, G);
  const int nt = (rows + 63) / 64, nj = (cols + 15) / 16;
  unsigned char *dflag = nullptr;
  WF_CUDA(cudaMalloc(&dflag, (size_t)nt * nj));
  k_tile_mask<<<nt, 128, 0, c.st>>>(G, ld, rows, cols, dflag);
  std::vector<unsigned char> f((size_t)nt * nj);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = memcpy_sync(c, f.data(), dflag, f.size(), cudaMemcpyDeviceToHost);
  cudaFree(dflag);
  WF_CUDA(e);
  // per tile: the non-zero chunks as two intervals split at the largest internal gap
  TileRanges tr;
  tr.base = G; tr.ld = ld; tr.rows = rows; tr.cols = cols;
  tr.h.resize(nt);
  double covered = 0;
  for (int t = 0; t < nt; ++t) {
    const unsigned char *ft = &f[(size_t)t * nj];
    int first = -1, last = -1, gap = 0, gs = -1, ge = -1, prev = -1;
    for (int j = 0; j < nj; ++j) {
      if (!ft[j]) continue;
      if (first < 0) first = j;
      if (prev >= 0 && j - prev - 1 > gap) { gap = j - prev - 1; gs = prev + 1; ge = j; }
      prev = last = j;
    }
    KRange k{0, 0, 0, 0};
    if (first >= 0) {
      if (gap >= 2) k = KRange{first * 16, gs * 16, ge * 16, std::min(cols, (last + 1) * 16)};
      else k = KRange{first * 16, std::min(cols, (last + 1) * 16), 0, 0};
    }
    tr.h[t] = k;
    covered += (double)std::min(64, rows - t * 64) * ((k.a1 - k.a0) + (k.b1 - k.b0));
  }
  if (covered > 0.75 * (double)rows * cols) return;   // not worth the bookkeeping
  tr.coverage = covered / ((double)rows * cols);
  tr.d = c.alloc<KRange>(nt);
  WF_CUDA(memcpy_sync(c, tr.d, tr.h.data(), nt * sizeof(KRange), cudaMemcpyHostToDevice));
  c.tranges.push_back(std::move(tr));
}

void unregister_tile_ranges(Ctx &c, const void *G) {
  for (size_t i = 0; i < c.tranges.size();) {
    if (c.tranges[i].base == G) {
      auto it = std::find(c.allocs.begin(), c.allocs.end(), (void *)c.tranges[i].d);
      if (it != c.allocs.end()) c.allocs.erase(it);
      cudaFree(c.tranges[i].d);
      c.tranges.erase(c.tranges.begin() + i);
    } else {
      ++i;
    }
  }
}

const TileRanges *find_tile_ranges(const Ctx &c, const double *A, int *row0, int *col0) {
  for (const TileRanges &t : c.tranges) {
    if (A < t.base || A >= t.base + (int64_t)t.rows * t.ld) continue;
    const int64_t off = A - t.base;
    const int r = (int)(off / t.ld), q = (int)(off % t.ld);
    if (r % 64 != 0 || q >= t.cols) return nullptr;
    *row0 = r;
    *col0 = q;
    return &t;
  }
  return nullptr;
}

// sum over the 64-row tiles of rows [r0, r0 + nrows) of rows x covered columns in
// [k0, k1): the algorithmic (non-zero tile) work of a banded product
double kr_work(const TileRanges &t, int r0, int nrows, int k0, int k1) {
  double w = 0;
  for (int r = r0; r < r0 + nrows;) {
    const int tt = r / 64, re = std::min(r0 + nrows, tt * 64 + 64);
    const KRange &k = t.h[tt];
    const int ca = std::max(0, std::min(k.a1, k1) - std::max(k.a0, k0));
    const int cb = std::max(0, std::min(k.b1, k1) - std::max(k.b0, k0));
    w += (double)(re - r) * (ca + cb);
    r = re;
  }
  return w;
}

void launch_gemm(Ctx &c, const GemmProb *probs, int nprob, int batch, double flops_hint) {
  int valid = 0;
  GemmProb ps[2];
  for (int i = 0; i < nprob; ++i)
    if (probs[i].M > 0 && probs[i].N > 0) ps[valid++] = probs[i];
  if (!valid || batch <= 0) return;
  double flops = 0, bytes = 0;
  bool v16 = true;
  int tm, tn, huge_tiles = 0, big_tiles = 0;
  for (int i = 0; i < valid; ++i) {
    GemmProb &p = ps[i];
    int r0 = 0, c0 = 0;
    const TileRanges *t = (!p.kr && batch == 1 && !c.tranges.empty() && p.M > 64)
                              ? find_tile_ranges(c, p.A, &r0, &c0) : nullptr;
    // attach only where the ranges skip work: the off-diagonal blocks a blocked TRSM
    // couples with are dense even when the (triangular) factor is registered, and a
    // dense GEMM keeps the stream-K tail (r01am: the coupling GEMMs had lost it)
    const double w = (t && c0 % 16 == 0 && p.lda == t->ld && r0 + p.M <= t->rows &&
                      c0 + p.K <= t->cols) ? kr_work(*t, r0, p.M, c0, c0 + p.K) : -1.0;
    if (w >= 0 && w < 0.9 * (double)p.M * p.K) {
      p.kr = t->d + r0 / 64;
      p.kr_c0 = c0;
      flops += 2.0 * p.N * w;
    } else {
      flops += 2.0 * p.M * (double)p.N * p.K * batch;
    }
    bytes += 8.0 * batch * ((double)p.M * p.K + (double)p.K * p.N + (double)p.M * p.N * (p.Z ? 2 : 1));
    v16 = v16 && aligned16(p);
    huge_tiles += tiles_of<CfgHuge>(p, tm, tn);
    big_tiles += tiles_of<CfgBig>(p, tm, tn);
  }
  if (flops_hint >= 0) flops = flops_hint;
  LaunchScope ls(c, c.gemm_cls, flops, bytes);
  static const int small_env = env_int("WF4DVAR_GEMM_SMALL", 2);   // 0: DMMA tiles always
  int mmax = 0, kmax = 0;
  for (int i = 0; i < valid; ++i) {
    mmax = std::max(mmax, ps[i].M);
    kmax = std::max(kmax, ps[i].K);
  }
  if (small_env && mmax <= 64 && kmax <= 64 && kmax > 0) {
    // 2 (default): the DMMA form; 1: the streaming FMA kernel (round 1)
    if (small_env == 2) run_small_dmma(c, ps, valid, batch, kmax);
    else run_small(c, ps, valid, batch, mmax, kmax);
    c.launches++;
    return;
  }
  static const int force = env_int("WF4DVAR_GEMM_CFG", -1);   // tuning experiments only
  if (force >= 0 && huge_tiles * batch >= 2 * 148) {
    if (force == 1) run<CfgWide>(c, ps, valid, batch, v16);
    else if (force == 3) run<TileCfg<64, 128, 16, 32, 64, 3>>(c, ps, valid, batch, v16);
    else if (force == 4) run<TileCfg<128, 128, 16, 64, 32, 4>>(c, ps, valid, batch, v16);
    else if (force == 5) run<TileCfg<64, 128, 16, 32, 64, 4>>(c, ps, valid, batch, v16);
    else if (force == 6) run<TileCfg<128, 64, 16, 64, 32, 3>>(c, ps, valid, batch, v16);
    else if (force == 7) run<TileCfg<64, 128, 16, 32, 64, 2>>(c, ps, valid, batch, v16);
    else if (force == 8) run<TileCfg<64, 256, 16, 32, 64, 3>>(c, ps, valid, batch, v16);
    else if (force == 9) run<TileCfg<128, 128, 16, 32, 64, 3>>(c, ps, valid, batch, v16);
    else if (force == 10) run<TileCfg<64, 128, 32, 32, 64, 2>>(c, ps, valid, batch, v16);
    else run<CfgHuge>(c, ps, valid, batch, v16);
  } else if (huge_tiles * batch >= 2 * 148) run<CfgHuge>(c, ps, valid, batch, v16);
  else if (batch == 1 && huge_tiles < 148 && run_splitk<CfgHuge>(c, ps, valid, v16)) {}
  else if (big_tiles * batch >= 148) run<CfgBig>(c, ps, valid, batch, v16);
  else run<CfgSmall>(c, ps, valid, batch, v16);
  c.launches++;
}

}  // namespace wf
