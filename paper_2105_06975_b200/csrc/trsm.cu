// Cholesky-factor triangular solves for D_hat^{-1} and R_hat^{-1} (
// R_hat^{-1} "using the ... Cholesky factors").  Dense blocks with n >= 256
// are applied through setup-time explicit inverses (reading A32, saddle.cu), which
// these solves compute; the solves themselves serve banded / IC(0) factors, small
// blocks, R_block segments and WF4DVAR_EXPLICIT_INV=0.
//
// Blocked right-looking TRSM, B200 layout:
//   * the triangle is cut into diagonal super-blocks of SB rows (a narrow-band
//     factor: one super-block);
//   * each super-block is solved by k_trsm: one CTA per NB-column panel walks
//     the 64-row tiles of the super-block,
//         T_i = X_i - sum_{j<i, j in block} G_ij Y_j    (DMMA tile GEMM, K tiles
//                                                         outside a band skipped)
//         Y_i = G_ii^{-1} T_i                           (default: one DMMA product
//                                                         with the setup-time inverse
//                                                         tile, reading A31; else exact
//                                                         shuffle substitution)
//   * the coupling of the solved super-block to all remaining rows is one large
//     DMMA GEMM  Y_rest -= G_rest,blk Y_blk  (gemm.cu), which is where almost
//     all the FLOPs go.
// R_block (Alg. 1) has a block-diagonal factor: every diagonal block is an
// independent segment (grid.y), no GEMM coupling.  Segments of <= 64 rows take the
// thread-per-column k_trsm_small.
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "dmma.cuh"
#include "internal.h"

namespace wf {

constexpr int TB = 64;  // rows per triangle tile
// The in-panel GEMMs are short (K < SB) and latency bound: a 4-deep cp.async ring.
#define TRSM_STAGES 4

template <int NB>
using TrsmCfg = typename std::conditional<NB == 8, TileCfg<64, 8, 16, 16, 8, TRSM_STAGES>,
                                          TileCfg<64, NB, 16, 32, NB / 2, TRSM_STAGES>>::type;

constexpr int kMaxSegTab = 512;
// doubles per packed diagonal tile: substitution form (transposed masked tile, stride
// 65, + 64 reciprocals = 4160) or inverse form (G_ii^{-1} row-major, stride kInvLd)
constexpr int kInvLd = TB + 4;
constexpr int kDiagPack = TB * kInvLd;
static_assert(kDiagPack >= TB * (TB + 1) + TB, "pack holds either form");

// Diagonal tiles applied as setup-time inverses (one DMMA product per tile instead of
// the 64-step shuffle substitution chain; reading A31).  Measured r01ag
// (per step): c1 0.527 -> 0.453 ms, c5 1.187 -> 1.036 ms, c3 34.20 -> 33.41 ms.
// WF4DVAR_TRSM_INV=0 restores the substitution.
static int trsm_inv_mode() {
  static const int v = env_int("WF4DVAR_TRSM_INV", 1);
  return v;
}

struct TrsmLaunch {
  TrsmProb p[2];
  int panels0;
  int seg_lo, seg_len, seg_hi;   // segment j covers [seg_lo + j*seg_len, min(.. + seg_len, seg_hi))
  int ntab;                      // > 0: segment j covers [tab[j], tab[j+1]) instead
  int tab[kMaxSegTab + 1];
};

template <int NB, bool UPPER, bool V16, bool INV>
__global__ void __launch_bounds__(128) k_trsm(const TrsmLaunch L) {
  using C = TrsmCfg<NB>;
  extern __shared__ __align__(16) double smem[];
  double *sPipe = smem;                        // C::SMEM_DOUBLES
  double *sT = smem + C::SMEM_DOUBLES;         // [64][NB+1]
  double *sG = sT + TB * (NB + 1);             // [64][65] diagonal tile, transposed
  double *sD = sG + TB * (TB + 1);             // [64] reciprocal diagonal

  int panel = blockIdx.x, gi = 0;
  if (panel >= L.panels0) { panel -= L.panels0; gi = 1; }
  const TrsmProb &P = L.p[gi];
  const int c0 = panel * NB;
  const int slo = L.ntab ? L.tab[blockIdx.y] : L.seg_lo + blockIdx.y * L.seg_len;
  const int shi = L.ntab ? L.tab[blockIdx.y + 1] : min(L.seg_hi, slo + L.seg_len);
  if (slo >= shi) return;
  const int ntile = (shi - slo + TB - 1) / TB;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / C::WARPS_N, wn = warp % C::WARPS_N;
  const int g = lane >> 2, t = lane & 3;
  const double *__restrict__ G = P.G;
  double *Y = P.Y;
  const double *X = P.X;
  const int ncols = P.ncols;
  const bool y16 = pair_aligned(Y, P.ldy);

  for (int it = 0; it < ntile; ++it) {
    const int ti = UPPER ? (ntile - 1 - it) : it;
    const int r0 = slo + ti * TB, r1 = min(shi, r0 + TB), nr = r1 - r0;
    // ---- setup-time pack of this diagonal tile (ncu r01g: building it in-kernel from
    // strided global loads + reciprocals was the top stall of k_trsm): one contiguous
    // 33 KB cp.async copy straight into sG|sD, overlapped with the tile GEMM below
    const double *dpk = (P.dpack && (r0 % TB) == 0) ? P.dpack + (int64_t)(r0 / TB) * kDiagPack
                                                      : nullptr;
    if (dpk) {
      for (int e = 2 * tid; e < kDiagPack; e += 2 * 128) cp_async16(sG + e, dpk + e, 16);
      cp_async_commit();
    }
    // ---- in-segment off-diagonal update: acc = G[r0:r1, K] * Y[K, panel]
    const int kbeg = UPPER ? r1 : slo;
    const int kend = UPPER ? shi : r0;
    double acc[C::FM][C::FN][2];
#pragma unroll
    for (int i = 0; i < C::FM; ++i)
#pragma unroll
      for (int j = 0; j < C::FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    if (kend > kbeg) {
      if (P.kr && (r0 & 63) == 0) {   // banded factor: only the K tiles these rows meet
        int lo[2], hi[2];
        const int nint = kr_intervals(P.kr, r0, nr, 0, kbeg, kend, lo, hi);
        for (int q = 0; q < nint; ++q)
          tile_mainloop<C, V16>(sPipe, acc, G + (int64_t)r0 * P.ldg, P.ldg, Y + c0, P.ldy, 0, 0,
                                lo[q], hi[q], nr, ncols - c0);
      } else {
        tile_mainloop<C, V16>(sPipe, acc, G + (int64_t)r0 * P.ldg, P.ldg, Y + c0, P.ldy, 0, 0,
                              kbeg, kend, nr, ncols - c0);
      }
    }
    // ---- T = X - acc  -> shared memory
#pragma unroll
    for (int i = 0; i < C::FM; ++i) {
      int rr = wm * C::WM + i * 8 + g;
#pragma unroll
      for (int j = 0; j < C::FN; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          int cc = wn * C::WN + j * 8 + 2 * t + h;
          double xv = 0.0;
          if (rr < nr && c0 + cc < ncols) xv = X[(int64_t)(r0 + rr) * P.ldx + c0 + cc];
          sT[rr * (NB + 1) + cc] = xv - acc[i][j][h];
        }
    }
    if (INV && dpk) {
      // ---- Y_i = G_ii^{-1} T_i on the tensor pipe (the setup-time inverse in sG,
      // row-major stride kInvLd; identity padding past a ragged tile).  Warp w owns
      // the 8-row blocks w and w + 4 across all NB columns.
      cp_async_wait<0>();
      __syncthreads();
      constexpr int NJ = NB / 8;
      double ya[2][NJ][2];
#pragma unroll
      for (int q = 0; q < 2; ++q)
#pragma unroll
        for (int j = 0; j < NJ; ++j) ya[q][j][0] = ya[q][j][1] = 0.0;
#pragma unroll 4
      for (int kk = 0; kk < TB; kk += 4) {
        const double a0 = sG[(warp * 8 + g) * kInvLd + kk + t];
        const double a1 = sG[((warp + 4) * 8 + g) * kInvLd + kk + t];
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
          const double b = sT[(kk + t) * (NB + 1) + j * 8 + g];
          dmma884(ya[0][j][0], ya[0][j][1], a0, b);
          dmma884(ya[1][j][0], ya[1][j][1], a1, b);
        }
      }
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int rr = (warp + 4 * q) * 8 + g;
        if (rr >= nr) continue;
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
          const int cc = c0 + j * 8 + 2 * t;
          store_pair(Y + (int64_t)(r0 + rr) * P.ldy + cc, cc, ncols, ya[q][j][0], ya[q][j][1], y16);
        }
      }
      __syncthreads();   // Y rows visible to the CTA; sG / sT free for the next tile
      continue;
    }
    // ---- diagonal tile, transposed and masked:
    //   sG[c][r] = G[r0 + r][r0 + c] for r strictly below (lower) / above (upper) c, else 0;
    //   sD[r] = 1 / G[r0 + r][r0 + r]   (identity padding of a ragged last tile).
    if (dpk) {
      cp_async_wait<0>();   // the pack copy issued before the tile GEMM has landed
    } else {
      // no setup pack: build it here (consecutive threads read consecutive columns)
      for (int e = tid; e < TB * TB; e += 128) {
        int r = e / TB, cc = e % TB;
        double v = 0.0;
        if (r < nr && cc < nr) v = G[(int64_t)(r0 + r) * P.ldg + r0 + cc];
        if (r == cc) sD[r] = (r < nr) ? 1.0 / v : 1.0;
        bool keep = UPPER ? (r < cc) : (r > cc);
        sG[cc * (TB + 1) + r] = keep ? v : 0.0;
      }
    }
    __syncthreads();
    // ---- substitution: warp w solves columns w, w+4, ...; lane holds rows lane, lane+32.
    // Step r: y_r = t_r / G_rr (owner lane, broadcast by shuffle), then every lane
    // t_l -= G_lr y_r with the masked column (zeros where l is not below r).
    constexpr int CPW = NB / 4;
    double v0[CPW], v1[CPW];
#pragma unroll
    for (int q = 0; q < CPW; ++q) {
      int cc = warp + 4 * q;
      v0[q] = sT[lane * (NB + 1) + cc];
      v1[q] = sT[(lane + 32) * (NB + 1) + cc];
    }
    auto step = [&](int r, auto hi_tag) {
      constexpr bool HI = decltype(hi_tag)::value;
      const double dinv = sD[r];
      const double g0 = sG[r * (TB + 1) + lane];
      const double g1 = sG[r * (TB + 1) + lane + 32];
      const int src = r & 31;
#pragma unroll
      for (int q = 0; q < CPW; ++q) {
        const double yr = __shfl_sync(0xffffffffu, HI ? v1[q] : v0[q], src) * dinv;
        if (HI) {
          v1[q] = (lane == src) ? yr : fma(-g1, yr, v1[q]);
          if (UPPER) v0[q] = fma(-g0, yr, v0[q]);
        } else {
          v0[q] = (lane == src) ? yr : fma(-g0, yr, v0[q]);
          if (!UPPER) v1[q] = fma(-g1, yr, v1[q]);
        }
      }
    };
    if (!UPPER) {
#pragma unroll 4
      for (int r = 0; r < 32; ++r) step(r, std::false_type{});
#pragma unroll 4
      for (int r = 32; r < TB; ++r) step(r, std::true_type{});
    } else {
#pragma unroll 4
      for (int r = TB - 1; r >= 32; --r) step(r, std::true_type{});
#pragma unroll 4
      for (int r = 31; r >= 0; --r) step(r, std::false_type{});
    }
    // ---- store Y rows of this tile
#pragma unroll
    for (int q = 0; q < CPW; ++q) {
      int cc = warp + 4 * q;
      if (c0 + cc < ncols) {
        if (lane < nr) Y[(int64_t)(r0 + lane) * P.ldy + c0 + cc] = v0[q];
        if (lane + 32 < nr) Y[(int64_t)(r0 + lane + 32) * P.ldy + c0 + cc] = v1[q];
      }
    }
    __syncthreads();   // Y rows visible to the whole CTA (next tile's cp.async reads)
  }
#ifdef TRSM_PROXY_FENCE
  // probe: order this thread's generic Y stores before any later
  // async-proxy (TMA) access
  asm volatile("fence.proxy.async.global;\n" ::: "memory");
#endif
#ifdef TRSM_END_FENCE
  // probe r02bd: device-scope fence, then the proxy fence, after the last Y stores
  __threadfence();
  asm volatile("fence.proxy.async.global;\n" ::: "memory");
#endif
}

// ---- Dataflow form of one segment (default where it applies, r02o): one CTA per
// (64-row tile, NB-column panel) instead of one CTA per panel walking every tile.  CTA
// (t, c) computes  Y_t = G_tt^{-1} (X_t - sum_{j before t} G_tj Y_j)  for its panel: it
// accumulates each G_tj Y_j as soon as tile j of the same panel is published (a ready
// flag in global memory), so the off-diagonal products of all tiles run in parallel on
// ntile x panels CTAs and only the chain "Y_{t-1} ready -> one 64 x 64 x NB product ->
// the inverse-tile product -> publish Y_t" is serial.  The blocked panel kernel above
// runs that whole chain, products included, inside one CTA per panel (ncu r02c: 11%
// warps active, latency bound; configs[1]: 42 CTAs on 148 SMs).
// Same arithmetic as k_trsm's inverse form: the K range of each tile is summed in
// increasing row order (lower) / decreasing tile order (upper) in BK = 16 steps, then
// T = X - acc, Y = G_tt^{-1} T (reading A31).
// CTAs are numbered in solve order (tile-major), so a CTA only waits for CTAs with
// lower indices, which the hardware dispatched before it: no co-residency is needed.
// Flags hold the launch epoch + 1; the epoch (ep[0]) is read at the start of every CTA
// and advanced by the last CTA to finish (ep[1] counts finished CTAs), so back-to-back
// launches and CUDA-graph replays on one stream need no host-side reset.
struct TrsmDfArgs {
  TrsmProb p[2];
  int panels0, panels;   // panels of problem 0; of both problems
  int slo, shi, ntile;   // the segment's rows; its 64-row tiles
  unsigned *flags;       // [ntile][panels]
  unsigned *ep;          // [0] epoch, [1] finished CTAs of the current launch
};

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned *p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

template <int NB, bool UPPER>
__global__ void __launch_bounds__(128) k_trsm_df(const TrsmDfArgs L) {
  using C = TrsmCfg<NB>;
  extern __shared__ __align__(16) double smem[];
  double *sPipe = smem;                        // C::SMEM_DOUBLES
  double *sT = smem + C::SMEM_DOUBLES;         // [64][NB+1]
  double *sG = sT + TB * (NB + 1);             // G_tt^{-1}, row-major, stride kInvLd
  __shared__ unsigned s_ep;
  __shared__ int s_ready;
  const int it = blockIdx.x / L.panels, pc = blockIdx.x - it * L.panels;
  int gi = 0, panel = pc;
  if (pc >= L.panels0) { gi = 1; panel -= L.panels0; }
  const TrsmProb &P = L.p[gi];
  const int ti = UPPER ? L.ntile - 1 - it : it;
  const int r0 = L.slo + ti * TB, r1 = min(L.shi, r0 + TB), nr = r1 - r0;
  const int c0 = panel * NB;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / C::WARPS_N, wn = warp % C::WARPS_N;
  const int g = lane >> 2, t = lane & 3;
  const bool y16 = pair_aligned(P.Y, P.ldy);
  const int ncols = P.ncols;
  // the inverse diagonal tile and this tile's X rows: in flight under the dependency
  // waits and the products (X_t is read only here; in place, only this CTA writes Y_t)
  const double *dpk = P.dpack + (int64_t)(r0 / TB) * kDiagPack;
  for (int e = 2 * tid; e < kDiagPack; e += 2 * 128) cp_async16(sG + e, dpk + e, 16);
  for (int e = tid; e < TB * NB; e += 128) {
    const int rr = e / NB, cc = e % NB;
    const bool ok = rr < nr && c0 + cc < ncols;
    cp_async8(sT + rr * (NB + 1) + cc, ok ? P.X + (int64_t)(r0 + rr) * P.ldx + c0 + cc : P.X,
              ok ? 8 : 0);
  }
  cp_async_commit();
  if (tid == 0) s_ep = __ldcg(L.ep);
  __syncthreads();
  const unsigned want = s_ep + 1;
  double acc[C::FM][C::FN][2];
#pragma unroll
  for (int i = 0; i < C::FM; ++i)
#pragma unroll
    for (int j = 0; j < C::FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  // dependencies: the tiles before this one in solve order, it' = 0 .. it-1
  auto dep_tile = [&](int k) { return UPPER ? L.ntile - 1 - k : k; };
  auto dep_flag = [&](int k) { return L.flags + (int64_t)dep_tile(k) * L.panels + pc; };
  auto wait_dep = [&](int k) {
    if (tid == 0)
      while (ld_acquire_u32(dep_flag(k)) != want) __nanosleep(20);
  };
  // all but the last dependency through the cp.async DMMA main loop, as they arrive
  int done = 0;
  while (done < it - 1) {
    if (tid == 0) {
      int k = done;
      while (ld_acquire_u32(dep_flag(k)) != want) __nanosleep(32);
      ++k;
      // lower: every tile ready now, one increasing-k sweep (the chunking does not change
      // the summation order).  Upper: one tile per sweep -- its tiles arrive in decreasing
      // order, and a multi-tile sweep would sum them in increasing order, so the result
      // would depend on the arrival timing (deterministic results are tested bitwise)
      if (!UPPER)
        while (k < it - 1 && ld_acquire_u32(dep_flag(k)) == want) ++k;
      s_ready = k;
    }
    __syncthreads();
    const int k1 = s_ready;
    int kb, ke;   // rows of G's columns / Y's rows covered by solve-order tiles [done, k1)
    if (!UPPER) {
      kb = L.slo + done * TB;
      ke = L.slo + k1 * TB;
    } else {
      kb = L.slo + (L.ntile - k1) * TB;
      ke = min(L.shi, L.slo + (L.ntile - done) * TB);
    }
    tile_mainloop<C, true>(sPipe, acc, P.G + (int64_t)r0 * P.ldg, P.ldg, P.Y + c0, P.ldy, 0, 0,
                           kb, ke, nr, ncols - c0);   // ends with __syncthreads
    done = k1;
  }
  // the last dependency (the previous tile, on the critical path): its 64 x 64 block of G
  // is staged before its flag is awaited, so after the flag only Y_j (64 x NB, from L2)
  // is loaded before the product
  if (it >= 1) {
    const int jt = dep_tile(it - 1);
    const int jc0 = L.slo + jt * TB, jw = min(TB, L.shi - jc0);
    double *sGl = sPipe;                       // [64][kInvLd]
    double *sYl = sPipe + TB * kInvLd;         // [64][NB + 4]
    constexpr int LDY = NB + 4;
    static_assert(TB * kInvLd + TB * (NB + 4) <= C::SMEM_DOUBLES, "last-dependency staging");
    for (int e = tid; e < TB * (TB / 2); e += 128) {
      const int rr = e / (TB / 2), cp = (e % (TB / 2)) * 2;
      const int bytes = rr < nr ? max(0, min(2, jw - cp)) * 8 : 0;
      cp_async16(sGl + rr * kInvLd + cp, bytes ? P.G + (int64_t)(r0 + rr) * P.ldg + jc0 + cp : P.G,
                 bytes);
    }
    cp_async_commit();
    wait_dep(it - 1);
    __syncthreads();
    for (int e = tid; e < TB * (NB / 2); e += 128) {
      const int rr = e / (NB / 2), cp = (e % (NB / 2)) * 2;
      const int bytes = rr < jw ? max(0, min(2, ncols - c0 - cp)) * 8 : 0;
      cp_async16(sYl + rr * LDY + cp, bytes ? P.Y + (int64_t)(jc0 + rr) * P.ldy + c0 + cp : P.Y,
                 bytes);
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
#pragma unroll 4
    for (int kk = 0; kk < TB; kk += 4) {
      double a[C::FM], b[C::FN];
#pragma unroll
      for (int i = 0; i < C::FM; ++i) a[i] = sGl[(wm * C::WM + i * 8 + g) * kInvLd + kk + t];
#pragma unroll
      for (int j = 0; j < C::FN; ++j) b[j] = sYl[(kk + t) * LDY + wn * C::WN + j * 8 + g];
#pragma unroll
      for (int i = 0; i < C::FM; ++i)
#pragma unroll
        for (int j = 0; j < C::FN; ++j) dmma884(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
  }
  // T = X - acc (X staged in sT at the start)
  cp_async_wait<0>();
  __syncthreads();
#pragma unroll
  for (int i = 0; i < C::FM; ++i) {
    const int rr = wm * C::WM + i * 8 + g;
#pragma unroll
    for (int j = 0; j < C::FN; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int cc = wn * C::WN + j * 8 + 2 * t + h;
        sT[rr * (NB + 1) + cc] -= acc[i][j][h];
      }
  }
  cp_async_wait<0>();
  __syncthreads();
  // Y_t = G_tt^{-1} T on the tensor pipe (warp w: the 8-row blocks w and w + 4)
  constexpr int NJ = NB / 8;
  double ya[2][NJ][2];
#pragma unroll
  for (int q = 0; q < 2; ++q)
#pragma unroll
    for (int j = 0; j < NJ; ++j) ya[q][j][0] = ya[q][j][1] = 0.0;
#pragma unroll 4
  for (int kk = 0; kk < TB; kk += 4) {
    const double a0 = sG[(warp * 8 + g) * kInvLd + kk + t];
    const double a1 = sG[((warp + 4) * 8 + g) * kInvLd + kk + t];
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const double b = sT[(kk + t) * (NB + 1) + j * 8 + g];
      dmma884(ya[0][j][0], ya[0][j][1], a0, b);
      dmma884(ya[1][j][0], ya[1][j][1], a1, b);
    }
  }
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int rr = (warp + 4 * q) * 8 + g;
    if (rr >= nr) continue;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int cc = c0 + j * 8 + 2 * t;
      store_pair(P.Y + (int64_t)(r0 + rr) * P.ldy + cc, cc, ncols, ya[q][j][0], ya[q][j][1], y16);
    }
  }
  // publish Y_t of this panel, then count this CTA out of the launch
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    st_release_u32(L.flags + (int64_t)ti * L.panels + pc, want);
    if (atomicAdd(L.ep + 1, 1u) == gridDim.x - 1) {
      atomicExch(L.ep + 1, 0u);
      __threadfence();
      atomicAdd(L.ep, 1u);
    }
  }
}

// Setup: pack every 64x64 diagonal tile of a triangular factor as the kernel wants it
// in shared memory: transposed and strictly masked (sG[c][r], stride 65) followed by
// the 64 reciprocal diagonal entries (identity padding past n).
__global__ void k_pack_diag(const double *G, int n, int upper, double *pack) {
  const int t = blockIdx.x;
  const int r0 = t * TB, nr = min(TB, n - r0);
  double *pk = pack + (int64_t)t * kDiagPack;
  for (int e = threadIdx.x; e < TB * TB; e += blockDim.x) {
    int r = e / TB, cc = e % TB;
    double v = (r < nr && cc < nr) ? G[(int64_t)(r0 + r) * n + r0 + cc] : 0.0;
    if (r == cc) pk[TB * (TB + 1) + r] = (r < nr) ? 1.0 / v : 1.0;
    bool keep = upper ? (r < cc) : (r > cc);
    pk[cc * (TB + 1) + r] = keep ? v : 0.0;
  }
  for (int e = threadIdx.x; e < TB; e += blockDim.x) pk[e * (TB + 1) + TB] = 0.0;   // pad col
}

// Inverse form: pack[t] = G_tt^{-1} (row-major, stride kInvLd), computed column by
// column (thread j: substitution of G_tt x = e_j), identity padding past n.
__global__ void k_pack_diag_inv(const double *G, int n, int upper, double *pack) {
  __shared__ double sg[TB][TB + 1];
  const int t = blockIdx.x;
  const int r0 = t * TB, nr = min(TB, n - r0);
  double *pk = pack + (int64_t)t * kDiagPack;
  for (int e = threadIdx.x; e < TB * TB; e += blockDim.x) {
    const int r = e / TB, cc = e % TB;
    sg[r][cc] = (r < nr && cc < nr) ? G[(int64_t)(r0 + r) * n + r0 + cc] : (r == cc ? 1.0 : 0.0);
  }
  __syncthreads();
  const int j = threadIdx.x;
  if (j >= TB) return;
  double x[TB];
#pragma unroll
  for (int i = 0; i < TB; ++i) x[i] = 0.0;
  if (!upper) {
#pragma unroll
    for (int i = 0; i < TB; ++i) {
      if (i < j) continue;
      double v = (i == j) ? 1.0 : 0.0;
#pragma unroll
      for (int k = 0; k < TB; ++k)
        if (k >= j && k < i) v = fma(-sg[i][k], x[k], v);
      x[i] = v / sg[i][i];
    }
  } else {
#pragma unroll
    for (int i = TB - 1; i >= 0; --i) {
      if (i > j) continue;
      double v = (i == j) ? 1.0 : 0.0;
#pragma unroll
      for (int k = 0; k < TB; ++k)
        if (k > i && k <= j) v = fma(-sg[i][k], x[k], v);
      x[i] = v / sg[i][i];
    }
  }
#pragma unroll
  for (int i = 0; i < TB; ++i) pk[i * kInvLd + j] = x[i];
  for (int e = j; e < TB * (kInvLd - TB); e += TB)   // padding columns
    pk[(e / (kInvLd - TB)) * kInvLd + TB + e % (kInvLd - TB)] = 0.0;
}

void fill_diag_pack(Ctx &c, const double *G, int n, bool upper, double *pk) {
  const int nt = (n + TB - 1) / TB;
  if (trsm_inv_mode()) k_pack_diag_inv<<<nt, TB, 0, c.st>>>(G, n, upper ? 1 : 0, pk);
  else k_pack_diag<<<nt, 256, 0, c.st>>>(G, n, upper ? 1 : 0, pk);
  WF_CUDA(cudaGetLastError());
}

size_t diag_pack_doubles(int n) { return (size_t)((n + TB - 1) / TB) * kDiagPack; }

double *make_diag_pack(Ctx &c, const double *G, int n, bool upper) {
  const int nt = (n + TB - 1) / TB;
  double *pk = c.alloc<double>((size_t)nt * kDiagPack);
  fill_diag_pack(c, G, n, upper, pk);
  register_tile_ranges(c, G, n, n, n);   // banded factors: skip their zero tiles
  WF_CUDA(cudaStreamSynchronize(c.st));
  return pk;
}

template <int NB, bool UPPER, bool INV>
static void run_inv(Ctx &c, const TrsmLaunch &L, int panels, int nseg, bool v16) {
  using C = TrsmCfg<NB>;
  size_t smem = (C::SMEM_DOUBLES + TB * (NB + 1) + kDiagPack) * sizeof(double);
  auto kern = v16 ? k_trsm<NB, UPPER, true, INV> : k_trsm<NB, UPPER, false, INV>;
  // one-time (thread-safe static initialisation) opt-in to the large dynamic smem
  static const cudaError_t attr_v =
      cudaFuncSetAttribute(k_trsm<NB, UPPER, true, INV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  static const cudaError_t attr_n =
      cudaFuncSetAttribute(k_trsm<NB, UPPER, false, INV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  WF_CUDA(v16 ? attr_v : attr_n);
  kern<<<dim3(panels, nseg), 128, smem, c.st>>>(L);
  WF_CUDA(cudaGetLastError());
}

template <int NB, bool UPPER>
static void run(Ctx &c, const TrsmLaunch &L, int panels, int nseg, bool v16) {
  if (trsm_inv_mode()) run_inv<NB, UPPER, true>(c, L, panels, nseg, v16);
  else run_inv<NB, UPPER, false>(c, L, panels, nseg, v16);
}

template <int NB, bool UPPER>
static void run_df(Ctx &c, TrsmDfArgs &A) {
  using C = TrsmCfg<NB>;
  const size_t smem = (C::SMEM_DOUBLES + TB * (NB + 1) + kDiagPack) * sizeof(double);
  static const cudaError_t attr = cudaFuncSetAttribute(
      k_trsm_df<NB, UPPER>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  WF_CUDA(attr);
  // per-stream flags / epoch (concurrent solves on the fork/join streams must not share)
  Ctx::SkState *st = nullptr;
  for (auto &e : c.sk_states)
    if (e.stream == c.st) st = &e;
  if (!st) {
    c.sk_states.push_back(Ctx::SkState{});
    st = &c.sk_states.back();
    st->stream = c.st;
  }
  const size_t need = (size_t)A.ntile * A.panels;
  if (!st->df_ep) {
    WF_CUDA(cudaMalloc(&st->df_ep, 2 * sizeof(unsigned)));
    WF_CUDA(cudaMemsetAsync(st->df_ep, 0, 2 * sizeof(unsigned), c.st));
  }
  if (st->df_cap < need) {
    // flags of a grown set start at 0 (< every epoch + 1); the old set may still be
    // referenced by captured graphs: retired, freed with the context
    if (st->df_flags) c.retired.push_back(st->df_flags);
    WF_CUDA(cudaMalloc(&st->df_flags, need * sizeof(unsigned)));
    WF_CUDA(cudaMemsetAsync(st->df_flags, 0, need * sizeof(unsigned), c.st));
    st->df_cap = need;
  }
  A.flags = st->df_flags;
  A.ep = st->df_ep;
  k_trsm_df<NB, UPPER><<<A.ntile * A.panels, 128, smem, c.st>>>(A);
  WF_CUDA(cudaGetLastError());
}

// Small triangles: every segment (diagonal block) has <= 64 rows -- R_hat / D_hat of the
// L96 configs (s = 40, 50; p = 20, 25) and the R_block blocks.  The 64-row panel kernel
// above spends such a solve in the shuffle chain of a mostly empty tile; here one
// thread owns one right-hand-side column in registers (coalesced row loads across the
// warp) and runs the right-looking substitution
//     y_i = t_i / G_ii,   t_k -= G_ki y_i   (k after i),
// whose updates are independent FMAs, against the segment's factor held TRANSPOSED in
// shared memory (sGt[i][k] = G[k][i], broadcast 16-byte pair loads; masked to the
// strict triangle, identity padding past the segment so padded rows stay 0).
template <int NMAX, bool UPPER>
__global__ void __launch_bounds__(128) k_trsm_small(const TrsmLaunch L) {
  constexpr int LD = NMAX + 2;
  __shared__ __align__(16) double sGt[NMAX * LD];
  __shared__ double sD[NMAX];
  int chunk = blockIdx.x, gi = 0;
  if (chunk >= L.panels0) { chunk -= L.panels0; gi = 1; }
  const TrsmProb &P = L.p[gi];
  const int slo = L.ntab ? L.tab[blockIdx.y] : L.seg_lo + blockIdx.y * L.seg_len;
  const int shi = L.ntab ? L.tab[blockIdx.y + 1] : min(L.seg_hi, slo + L.seg_len);
  const int len = shi - slo;
  if (len <= 0) return;
  for (int e = threadIdx.x; e < NMAX * NMAX; e += 128) {
    const int i = e / NMAX, k = e % NMAX;
    const bool keep = (UPPER ? (k < i) : (k > i)) && i < len && k < len;
    sGt[i * LD + k] = keep ? P.G[(int64_t)(slo + k) * P.ldg + slo + i] : 0.0;
  }
  for (int e = threadIdx.x; e < NMAX; e += 128)
    sD[e] = e < len ? 1.0 / P.G[(int64_t)(slo + e) * P.ldg + slo + e] : 1.0;
  __syncthreads();
  const int col = chunk * 128 + threadIdx.x;
  if (col >= P.ncols) return;
  double y[NMAX];
#pragma unroll
  for (int i = 0; i < NMAX; ++i) y[i] = i < len ? P.X[(int64_t)(slo + i) * P.ldx + col] : 0.0;
  if (!UPPER) {
#pragma unroll
    for (int i = 0; i < NMAX; ++i) {
      y[i] *= sD[i];
      // pairs from the even index at or below i + 1 (sGt[i][i] = 0 keeps y_i unchanged)
#pragma unroll
      for (int k = (i + 1) & ~1; k < NMAX; k += 2) {
        const double2 gg = *reinterpret_cast<const double2 *>(&sGt[i * LD + k]);
        y[k] = fma(-gg.x, y[i], y[k]);
        y[k + 1] = fma(-gg.y, y[i], y[k + 1]);
      }
    }
  } else {
#pragma unroll
    for (int i = NMAX - 1; i >= 0; --i) {
      y[i] *= sD[i];
#pragma unroll
      for (int k = 0; k < i; k += 2) {
        const double2 gg = *reinterpret_cast<const double2 *>(&sGt[i * LD + k]);
        y[k] = fma(-gg.x, y[i], y[k]);
        y[k + 1] = fma(-gg.y, y[i], y[k + 1]);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < NMAX; ++i)
    if (i < len) P.Y[(int64_t)(slo + i) * P.ldy + col] = y[i];
}

template <bool UPPER>
static void run_small(Ctx &c, const TrsmLaunch &L, int chunks, int nseg, int maxlen) {
  const dim3 grid(chunks, nseg);
  switch ((maxlen + 7) / 8) {
    case 1: k_trsm_small<8, UPPER><<<grid, 128, 0, c.st>>>(L); break;
    case 2: k_trsm_small<16, UPPER><<<grid, 128, 0, c.st>>>(L); break;
    case 3: k_trsm_small<24, UPPER><<<grid, 128, 0, c.st>>>(L); break;
    case 4: k_trsm_small<32, UPPER><<<grid, 128, 0, c.st>>>(L); break;
    case 5: k_trsm_small<40, UPPER><<<grid, 128, 0, c.st>>>(L); break;
    case 6: k_trsm_small<48, UPPER><<<grid, 128, 0, c.st>>>(L); break;
    case 7: k_trsm_small<56, UPPER><<<grid, 128, 0, c.st>>>(L); break;
    default: k_trsm_small<64, UPPER><<<grid, 128, 0, c.st>>>(L); break;
  }
  WF_CUDA(cudaGetLastError());
}

// the dataflow kernel applies to dense factors with packed inverse diagonal tiles
// (WF4DVAR_TRSM_DF=0: never)
// (dense: the registered tile ranges of a full triangle are the triangle itself, so the
// kernel's dependency K loop covers exactly them; narrow-band factors keep the panel walk,
// whose K loops skip the zero tiles -- the caller passes allow_df = false for those)
static bool df_ok(const TrsmProb *p, int np) {
  static const int df_env = env_int("WF4DVAR_TRSM_DF", 1);
  if (!df_env || !trsm_inv_mode()) return false;
  for (int i = 0; i < np; ++i)
    if (!p[i].dpack || p[i].blk || p[i].segs) return false;
  return true;
}

// one k_trsm launch over segments [seg_lo + j*seg_len ...) of every problem
static void trsm_segments(Ctx &c, const TrsmProb *probs, int np, bool upper, int seg_lo,
                          int seg_len, int seg_hi, const std::vector<int> *tab = nullptr,
                          bool allow_df = false) {
  TrsmLaunch L{};
  int total_cols = 0;
  bool v16 = (seg_len % 2 == 0) && (seg_lo % 2 == 0);
  double flops = 0, bytes = 0;
  int nseg = (seg_hi - seg_lo + seg_len - 1) / seg_len;
  // algorithmic work: each segment of length l is a triangle of l^2/2 FMAs per column
  const int last = seg_hi - seg_lo - (nseg - 1) * seg_len;
  double tri = (double)(nseg - 1) * seg_len * seg_len + (double)last * last;
  if (tab) {
    nseg = (int)tab->size() - 1;
    WF_REQUIRE(nseg >= 1 && nseg <= kMaxSegTab, WF4DVAR_EINVAL, "too many R_block blocks");
    L.ntab = nseg;
    tri = 0;
    for (int j = 0; j <= nseg; ++j) {
      L.tab[j] = (*tab)[j];
      v16 = v16 && ((*tab)[j] % 2 == 0);
      if (j < nseg) tri += (double)((*tab)[j + 1] - (*tab)[j]) * ((*tab)[j + 1] - (*tab)[j]);
    }
    seg_lo = (*tab)[0];
    seg_hi = (*tab)[nseg];
  }
  for (int i = 0; i < np; ++i) {
    L.p[i] = probs[i];
    total_cols += probs[i].ncols;
    double rows = seg_hi - seg_lo;
    int r0 = 0, c0 = 0;
    const TileRanges *tr = probs[i].kr ? find_tile_ranges(c, probs[i].G, &r0, &c0) : nullptr;
    if (tr && r0 == 0 && c0 == 0) {   // banded: the non-zero tiles of each segment's triangle
      double w = 0;
      for (int j = 0; j < nseg; ++j) {
        const int a = tab ? (*tab)[j] : seg_lo + j * seg_len;
        const int b = tab ? (*tab)[j + 1] : std::min(seg_hi, a + seg_len);
        w += kr_work(*tr, a, b - a, a, b);
      }
      flops += 2.0 * w * probs[i].ncols;
    } else {
      flops += tri * probs[i].ncols;
    }
    bytes += 8.0 * (tri / 2 + 2.0 * rows * probs[i].ncols);
    v16 = v16 && ((uintptr_t)probs[i].G % 16 == 0) && ((uintptr_t)probs[i].Y % 16 == 0) &&
          (probs[i].ldg % 2 == 0) && (probs[i].ldy % 2 == 0);
  }
  L.seg_lo = seg_lo; L.seg_len = seg_len; L.seg_hi = seg_hi;
  if (tab) { L.seg_lo = 0; L.seg_len = 1; }
  // every segment <= 64 rows: the thread-per-column kernel
  static const int small_env = env_int("WF4DVAR_TRSM_SMALL", 1);   // 0: panel kernel always
  int maxlen = tab ? 0 : std::min(seg_len, seg_hi - seg_lo);
  if (tab)
    for (int j = 0; j < nseg; ++j) maxlen = std::max(maxlen, (*tab)[j + 1] - (*tab)[j]);
  if (small_env && maxlen <= 64) {
    int chunks = 0;
    for (int i = 0; i < np; ++i) {
      const int ci = (L.p[i].ncols + 127) / 128;
      if (i == 0) L.panels0 = ci;
      chunks += ci;
    }
    if (np == 1) L.panels0 = chunks;
    LaunchScope ls(c, K_TRSM, flops, bytes);
    upper ? run_small<true>(c, L, chunks, nseg, maxlen)
          : run_small<false>(c, L, chunks, nseg, maxlen);
    c.launches++;
    return;
  }
  // one dense segment, inverse diagonal tiles packed, 16-byte aligned operands: the
  // dataflow kernel (WF4DVAR_TRSM_DF=0: the panel walk)
  static const int nb_env = env_int("WF4DVAR_TRSM_NB", 0);   // tuning experiments only
  if (allow_df && nseg == 1 && !tab && v16 && (seg_lo % TB) == 0 && df_ok(L.p, np)) {
    TrsmDfArgs A{};
    A.p[0] = L.p[0];
    if (np > 1) A.p[1] = L.p[1];
    A.slo = seg_lo; A.shi = seg_hi;
    A.ntile = (seg_hi - seg_lo + TB - 1) / TB;
    // panel width: the widest of 32 / 16 / 8 columns that still gives >= 2 CTAs per SM
    int nb = 32;
    auto ctas = [&](int w) {
      int t = 0;
      for (int i = 0; i < np; ++i) t += (L.p[i].ncols + w - 1) / w;
      return t * A.ntile;
    };
    if (ctas(32) < 2 * 148) nb = 16;
    if (nb == 16 && ctas(16) < 2 * 148) nb = 8;
    if (nb_env == 8 || nb_env == 16 || nb_env == 32) nb = nb_env;
    A.panels0 = (L.p[0].ncols + nb - 1) / nb;
    A.panels = A.panels0 + (np > 1 ? (L.p[1].ncols + nb - 1) / nb : 0);
    if (np == 1) A.panels0 = A.panels;
    LaunchScope ls(c, K_TRSM, flops, bytes);
    switch (nb) {
      case 32: upper ? run_df<32, true>(c, A) : run_df<32, false>(c, A); break;
      case 16: upper ? run_df<16, true>(c, A) : run_df<16, false>(c, A); break;
      default: upper ? run_df<8, true>(c, A) : run_df<8, false>(c, A); break;
    }
    c.launches++;
    return;
  }
  // panel width: as wide as possible while still filling the SMs
  const int ctas_per_col = nseg;
  int NB = 64;
  if ((total_cols + 63) / 64 * ctas_per_col < 148) NB = 32;
  if ((total_cols + 31) / 32 * ctas_per_col < 148) NB = 16;
  if ((total_cols + 15) / 16 * ctas_per_col < 148) NB = 8;
  if (nb_env == 8 || nb_env == 16 || nb_env == 32 || nb_env == 64) NB = nb_env;
  int panels = 0;
  for (int i = 0; i < np; ++i) {
    int pi = (L.p[i].ncols + NB - 1) / NB;
    if (i == 0) L.panels0 = pi;
    panels += pi;
  }
  if (np == 1) L.panels0 = panels;
  LaunchScope ls(c, K_TRSM, flops, bytes);
  switch (NB) {
    case 64: upper ? run<64, true>(c, L, panels, nseg, v16) : run<64, false>(c, L, panels, nseg, v16); break;
    case 32: upper ? run<32, true>(c, L, panels, nseg, v16) : run<32, false>(c, L, panels, nseg, v16); break;
    case 16: upper ? run<16, true>(c, L, panels, nseg, v16) : run<16, false>(c, L, panels, nseg, v16); break;
    default: upper ? run<8, true>(c, L, panels, nseg, v16) : run<8, false>(c, L, panels, nseg, v16); break;
  }
  c.launches++;
}

// Recursive blocked TRSM over rows [lo, hi) (Elmroth-Gustavson style): solve one
// half, couple it to the other half with ONE DMMA GEMM (K = half the range), solve
// the other half.  Half the triangle's flops land in the top-level GEMM (K = n/2),
// a quarter in K = n/4 GEMMs, ...; only ranges <= leaf rows go to the panel kernel.
// src_x: the rows of this range still hold only X (no coupling wrote Y yet).
static void trsm_rec(Ctx &c, const TrsmProb *probs, int np, bool upper, int lo, int hi, int leaf,
                     bool src_x) {
  auto with_src = [&](TrsmProb *cur, bool from_x) {
    for (int i = 0; i < np; ++i) {
      cur[i] = probs[i];
      if (!from_x) { cur[i].X = cur[i].Y; cur[i].ldx = cur[i].ldy; }
    }
  };
  TrsmProb cur[2];
  if (hi - lo <= leaf) {
    with_src(cur, src_x);
    trsm_segments(c, cur, np, upper, lo, hi - lo, hi);
    return;
  }
  // split at a multiple of the 64-row tile, near the middle
  int mid = lo + (((hi - lo) / 2 + TB - 1) / TB) * TB;
  if (mid >= hi) mid = lo + (hi - lo) / 2;
  const int f_lo = upper ? mid : lo, f_hi = upper ? hi : mid;     // solved first
  const int s_lo = upper ? lo : mid, s_hi = upper ? mid : hi;     // coupled, solved second
  trsm_rec(c, probs, np, upper, f_lo, f_hi, leaf, src_x);
  GemmProb g[2];
  for (int i = 0; i < np; ++i) {
    const TrsmProb &P = probs[i];
    GemmProb &q = g[i];
    q = GemmProb{};
    q.A = P.G + (int64_t)s_lo * P.ldg + f_lo; q.lda = P.ldg;
    q.X = P.Y + (int64_t)f_lo * P.ldy; q.ldx = P.ldy;
    q.Y = P.Y + (int64_t)s_lo * P.ldy; q.ldy = P.ldy;
    if (src_x) { q.Z = P.X + (int64_t)s_lo * P.ldx; q.ldz = P.ldx; }
    else { q.Z = q.Y; q.ldz = P.ldy; }
    q.M = s_hi - s_lo; q.N = P.ncols; q.K = f_hi - f_lo;
    q.alpha = -1.0; q.beta = 1.0;
  }
  c.gemm_cls = K_TRSM_UPD;
  launch_gemm(c, g, np, 1);
  c.gemm_cls = K_GEMM;
  trsm_rec(c, probs, np, upper, s_lo, s_hi, leaf, false);
}

void launch_trsm(Ctx &c, const TrsmProb *probs_in, int nprob, bool upper) {
  TrsmProb probs[2];
  int np = 0;
  for (int i = 0; i < nprob; ++i)
    if (probs_in[i].ncols > 0 && probs_in[i].n > 0) probs[np++] = probs_in[i];
  if (!np) return;
  bool banded = true;   // every factor a narrow band (not just a triangle)
  for (int i = 0; i < np; ++i) {   // banded factor: its registered column ranges
    int r0 = 0, c0 = 0;
    const TileRanges *tr = (!probs[i].kr && !c.tranges.empty())
                               ? find_tile_ranges(c, probs[i].G, &r0, &c0) : nullptr;
    if (tr && r0 == 0 && c0 == 0 && tr->ld == probs[i].ldg && tr->rows >= probs[i].n)
      probs[i].kr = tr->d;
    banded = banded && tr && tr->coverage < 0.35;
  }
  const int n = probs[0].n;
  const int blk = probs[0].blk;
  if (probs[0].segs) {   // variable block-diagonal factor (Algorithm 1): independent segments
    trsm_segments(c, probs, np, upper, 0, 1, n, probs[0].segs);
    return;
  }
  if (blk > 0) {   // block-diagonal factor: independent segments
    trsm_segments(c, probs, np, upper, 0, blk, n);
    return;
  }
  // a whole triangle of <= 64 rows (the L96 configs' D_hat / R_hat, s = 40, p = 20) is a
  // single diagonal tile: apply its setup-time inverse (reading A31) as one small DMMA
  // product, in place allowed (gemm.cu k_gemm_small_dmma).  OPT-IN (WF4DVAR_TRSM_SMALL_INV=1):
  // r02ao measured configs[2]'s TRSM class 1.62 -> 1.28 ms per 20 steps (step 0.467 ->
  // 0.456 ms), but a product with an inverse is not backward stable (reading A32) and on
  // configs[0] it moved the smoke cell's MINRES count outside reading A33's envelope
  // (GPU 180, oracle recurrence with the GPU's applies 182); the thread-per-column
  // substitution (k_trsm_small) stays the default.
  static const int small_inv = env_int("WF4DVAR_TRSM_SMALL_INV", 0);
  bool tile_inv = small_inv && trsm_inv_mode() && n <= TB;
  for (int i = 0; i < np; ++i) tile_inv = tile_inv && probs[i].dpack && probs[i].n == n;
  if (tile_inv) {
    GemmProb g[2];
    double flops = 0;
    for (int i = 0; i < np; ++i) {
      const TrsmProb &P = probs[i];
      g[i] = GemmProb{};
      g[i].A = P.dpack; g[i].lda = kInvLd;
      g[i].X = P.X; g[i].ldx = P.ldx;
      g[i].Y = P.Y; g[i].ldy = P.ldy;
      g[i].M = n; g[i].N = P.ncols; g[i].K = n;
      g[i].alpha = 1.0; g[i].beta = 0.0;
      flops += (double)n * n * P.ncols;   // the triangle's n^2 / 2 FMAs per column
    }
    const int saved = c.gemm_cls;
    c.gemm_cls = K_TRSM;
    launch_gemm(c, g, np, 1, flops);
    c.gemm_cls = saved;
    return;
  }
  // recursion (Elmroth-Gustavson, leaf 512) for the large dense factors with wide
  // right-hand sides: with the triangular solves as the default D_hat^{-1} apply, the
  // configs[3] step measured 32.33 (blocked, SB = 1024) -> 32.04 ms (leaf 512; leaf 256:
  // 33.30, 768: 32.68 with the same heat kernel; r02c/r02d sweeps) -- the top-level
  // coupling GEMM (K = n/2) runs at GEMM rate and the panels shrink to 512 rows.
  // Standalone (r01c/r01l kbench) the two schemes were within 1%.  WF4DVAR_TRSM_LEAF=0
  // forces the blocked scheme, > 0 the recursion with that leaf.
  int total_cols0 = 0;
  for (int i = 0; i < np; ++i) total_cols0 += probs[i].ncols;
  static const int leaf_env = env_int("WF4DVAR_TRSM_LEAF", -1);
  const int leaf = leaf_env >= 0 ? leaf_env : ((n >= 4096 && total_cols0 > 1536 && !banded) ? 512 : 0);
  if (leaf > 0 && n > leaf) {
    trsm_rec(c, probs, np, upper, 0, n, leaf, true);
    return;
  }
  static const int sb_env = env_int("WF4DVAR_TRSM_SB", 0);   // tuning experiments only
  // the dataflow kernel needs no coupling GEMMs between super-blocks: one launch over the
  // whole triangle (ntile x panels CTAs, K up to n) where the blocked scheme's
  // 2 (n / SB) - 1 launches per solve leave the GPU latency bound: narrow right-hand
  // sides.  r02q per step: configs[1] (n = 1000 / 500, 336 columns) GMRES 0.592 -> 0.548
  // ms, MINRES 0.426 -> 0.364 ms; but wide ones lose -- configs[4] (n = 2048, 8192
  // columns) 18.68 -> 19.07 ms, configs[3] with the dataflow kernel at the 512-row leaves
  // 29.46 -> 30.06 ms, over the whole triangle 32.5 ms (its 64 x NB tiles run the long K
  // loops at ~21 TFLOP/s against the coupling GEMMs' 28)
  static const int df_whole = env_int("WF4DVAR_TRSM_DF_WHOLE", 2048);
  static const int df_cols = env_int("WF4DVAR_TRSM_DF_COLS", 1024);
  if (!sb_env && !banded && n <= df_whole && total_cols0 <= df_cols && df_ok(probs, np)) {
    trsm_segments(c, probs, np, upper, 0, n, n, nullptr, true);
    return;
  }
  // measured (tools/kbench.py, r01): at n = 4096 SB = 512 gives 19.1 TFLOP/s vs 16.2
  // (256) and 12.3 (128) -- the coupling GEMMs need K >= 512 to run efficiently
  // (1024 at n = 4096: 20.6 TFLOP/s, above cuBLAS DTRSM's 18.8 on the same shape)
  // narrow right-hand sides (a time shard of configs[3] on 8 ranks: 1024 columns) gain
  // from shorter panel chains: r01z measured SB = 512 4.5% faster per step there
  int total_cols = 0;
  for (int i = 0; i < np; ++i) total_cols += probs[i].ncols;
  // a banded factor (compact-support covariance): the in-segment K loops stop at the
  // band, so one panel walk over all rows costs no extra GEMM work and saves the
  // coupling launches (r01at, NEXT-1 at n = 2048: 1.021 -> 0.914 ms per step)
  static const int banded_sb = env_int("WF4DVAR_TRSM_BANDED_SB", 1);   // 0: size-based SB
  const int SB = sb_env > 0 ? sb_env
                 : (banded && banded_sb) ? n
                 : (n >= 4096 ? (total_cols <= 1536 ? 512 : 1024)
                              : (n >= 2048 ? 512 : (n >= 512 ? 256 : 128)));
  if (n <= SB) {
    trsm_segments(c, probs, np, upper, 0, n, n);
    return;
  }
  const int nsb = (n + SB - 1) / SB;
  static const int left_env = env_int("WF4DVAR_TRSM_LEFT", 0);   // tuning experiments only
  if (left_env) {
    // left-looking: before solving super-block b, ONE GEMM brings in every solved
    // block (K = all rows solved so far), then the panel kernel solves b in place
    for (int it = 0; it < nsb; ++it) {
      const int kb = upper ? nsb - 1 - it : it;
      const int lo = kb * SB, hi = std::min(n, lo + SB);
      TrsmProb cur[2];
      for (int i = 0; i < np; ++i) cur[i] = probs[i];
      const int klo = upper ? hi : 0, khi = upper ? n : lo;   // already solved rows
      if (khi > klo) {
        GemmProb g[2];
        for (int i = 0; i < np; ++i) {
          const TrsmProb &P = probs[i];
          GemmProb &q = g[i];
          q = GemmProb{};
          q.A = P.G + (int64_t)lo * P.ldg + klo; q.lda = P.ldg;
          q.X = P.Y + (int64_t)klo * P.ldy; q.ldx = P.ldy;
          q.Y = P.Y + (int64_t)lo * P.ldy; q.ldy = P.ldy;
          q.Z = P.X + (int64_t)lo * P.ldx; q.ldz = P.ldx;
          q.M = hi - lo; q.N = P.ncols; q.K = khi - klo;
          q.alpha = -1.0; q.beta = 1.0;
          cur[i].X = cur[i].Y; cur[i].ldx = cur[i].ldy;   // the block is now in Y
        }
        c.gemm_cls = K_TRSM_UPD;
        launch_gemm(c, g, np, 1);
        c.gemm_cls = K_GEMM;
      }
      trsm_segments(c, cur, np, upper, lo, hi - lo, hi);
    }
    return;
  }
  TrsmProb cur[2];
  for (int i = 0; i < np; ++i) cur[i] = probs[i];
  for (int it = 0; it < nsb; ++it) {
    const int kb = upper ? nsb - 1 - it : it;
    const int lo = kb * SB, hi = std::min(n, lo + SB);
    trsm_segments(c, cur, np, upper, lo, hi - lo, hi);
    // couple the solved block to the rest:  Y_rest = Z_rest - G_rest,blk Y_blk
    const int rlo = upper ? 0 : hi, rhi = upper ? lo : n;
    if (rhi > rlo) {
      GemmProb g[2];
      for (int i = 0; i < np; ++i) {
        const TrsmProb &P = cur[i];
        GemmProb &q = g[i];
        q = GemmProb{};
        q.A = P.G + (int64_t)rlo * P.ldg + lo; q.lda = P.ldg;
        q.X = P.Y + (int64_t)lo * P.ldy; q.ldx = P.ldy;
        q.Y = P.Y + (int64_t)rlo * P.ldy; q.ldy = P.ldy;
        q.Z = P.X + (int64_t)rlo * P.ldx; q.ldz = P.ldx;
        q.M = rhi - rlo; q.N = P.ncols; q.K = hi - lo;
        q.alpha = -1.0; q.beta = 1.0;
      }
      c.gemm_cls = K_TRSM_UPD;
      launch_gemm(c, g, np, 1);
      c.gemm_cls = K_GEMM;
    }
    // after the first coupling every remaining row of Y is initialised: solve in place
    for (int i = 0; i < np; ++i) { cur[i].X = cur[i].Y; cur[i].ldx = cur[i].ldy; }
  }
}

}  // namespace wf
