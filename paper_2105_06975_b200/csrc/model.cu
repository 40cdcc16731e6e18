// Model term kernels: M_w / M_w^T products fused into L, L^T (Eq. 2.3,
// P:L108-117), the chain substitutions of L_M(k)^{-1} (Def. 4.1, Lemma 4.2,
// P:L255-276), the L_I prefix scan and the H^T scatter of A's
// third block.
//
// Heat (BJ.c0-c4): M = (I - r Lap)^{-1} is a symmetric circulant whose row
// decays like rho^|d|, rho = (1+2r-sqrt(1+4r))/(2r) (0.1716 at r = 0.25).  It
// is applied as its exact circulant stencil truncated at |d| <= D where the
// dropped tail is < 1e-17 relative (D = 22 at r = 0.25): a coalesced,
// register-windowed 1-D stencil along the state index, one thread per
// (window, RHS) column -- FP64-ALU/HBM balanced, no tensor cores (not a GEMM).
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include <type_traits>

#include "dmma.cuh"
#include "internal.h"

namespace wf {

struct Taps { double t[65]; };

// out_w = base_w + sign * sum_d taps[d] in_{w_src}[(i+d) mod s]   (+ add2[row_map[i]])
template <int D, int TI>
__global__ void __launch_bounds__(128) k_heat_step(double *out, const double *base,
                                                   const double *in, const double *add2,
                                                   const int *row_map, const Taps taps, double sign,
                                                   int s, int W, int m, int w_first, int w_step,
                                                   int nw, int dir, const double *halo, int w0,
                                                   int WG) {
  const int64_t ld = (int64_t)W * m;
  const int cc = blockIdx.x * blockDim.x + threadIdx.x;
  if (cc >= nw * m) return;
  const int tt = cc / m, r = cc - tt * m;
  const int w = w_first + tt * w_step;
  const int ws = w + dir;   // dir = -1 (M_w in_{w-1}) or +1 (M_{w+1}^T in_{w+1}); local
  const bool has = (w0 + ws >= 0 && w0 + ws < WG);   // the global source window exists
  // a source outside the local windows belongs to the neighbour rank: its state
  // was received into the [s][m] halo buffer
  const bool from_halo = (ws < 0 || ws >= W);
  const int64_t col = (int64_t)w * m + r, cols = (int64_t)ws * m + r;
  const int i0 = blockIdx.y * TI;
  double v[TI + 2 * D];
  if (has) {
#pragma unroll
    for (int j = 0; j < TI + 2 * D; ++j) {
      int row = i0 - D + j;
      row = row < 0 ? row + s : (row >= s ? row - s : row);
      row = row < 0 ? row + s : (row >= s ? row - s : row);
      v[j] = from_halo ? __ldg(halo + (int64_t)row * m + r) : __ldg(in + row * ld + cols);
    }
  }
  // tap-outer / row-inner: TI independent accumulation chains advance together
  // (ILP TI instead of one 2D+1-long dependent FMA chain at a time; ncu r01 showed
  // the row-outer form stalled on fixed-latency FMA dependencies)
  double acc[TI];
#pragma unroll
  for (int o = 0; o < TI; ++o) acc[o] = 0.0;
  if (has) {
#pragma unroll
    for (int d = 0; d <= 2 * D; ++d) {
      const double td = taps.t[d];
#pragma unroll
      for (int o = 0; o < TI; ++o) acc[o] = fma(td, v[o + d], acc[o]);
    }
  }
#pragma unroll
  for (int o = 0; o < TI; ++o) {
    const int i = i0 + o;
    if (i < s) {
      double val = base[i * ld + col];
      if (has) val = fma(sign, acc[o], val);
      if (add2) {
        int j = row_map[i];
        if (j >= 0) val += add2[(int64_t)j * ld + col];
      }
      out[i * ld + col] = val;
    }
  }
}

// Same operator through its factorisation (I - r Lap) = (r/rho)(1 - rho S)(1 - rho S^-1)
// (S the periodic shift, rho as above): M x = (rho/r) * anticausal(causal(x)) with the
// first-order recursions u_j = x_j + rho u_{j-1}, v_i = u_i + rho v_{i+1}.  Each thread
// owns TI consecutive rows of one (window, RHS) column and starts each recursion H rows
// early from zero: the dropped tail is rho^(H+1)/(1-rho) relative (< 1e-17 for the H
// the stencil uses), so this is the stencil's operator to rounding, at ~4 FMAs per
// output instead of 2H+1 (ncu r01: the stencil was FP64-ALU bound).
template <int H, int TI>
__global__ void __launch_bounds__(128) k_heat_iir(double *out, const double *base,
                                                  const double *in, const double *add2,
                                                  const int *row_map, double rho, double gain,
                                                  int s, int W, int m, int w_first, int w_step,
                                                  int nw, int dir, const double *halo, int w0,
                                                  int WG) {
  const int64_t ld = (int64_t)W * m;
  const int cc = blockIdx.x * blockDim.x + threadIdx.x;
  if (cc >= nw * m) return;
  const int tt = cc / m, r = cc - tt * m;
  const int w = w_first + tt * w_step;
  const int ws = w + dir;
  const bool has = (w0 + ws >= 0 && w0 + ws < WG);
  const bool from_halo = (ws < 0 || ws >= W);
  const int64_t col = (int64_t)w * m + r;
  const double *src = from_halo ? halo + r : in + (int64_t)ws * m + r;
  const int64_t sld = from_halo ? (int64_t)m : ld;
  const int i0 = blockIdx.y * TI;
  auto wrap = [&](int i) { i %= s; return i < 0 ? i + s : i; };
  double ub[TI + H + 1];
  if (has) {
    double u = 0.0;
#pragma unroll 4
    for (int j = i0 - H; j < i0; ++j) u = fma(rho, u, __ldg(src + wrap(j) * sld));
#pragma unroll
    for (int t = 0; t <= TI + H; ++t) {
      u = fma(rho, u, __ldg(src + wrap(i0 + t) * sld));
      ub[t] = u;
    }
  }
  double v = 0.0;
  if (has) {
#pragma unroll
    for (int t = TI + H; t >= TI; --t) v = fma(rho, v, ub[t]);
  }
#pragma unroll
  for (int t = TI - 1; t >= 0; --t) {
    if (has) v = fma(rho, v, ub[t]);
    const int i = i0 + t;
    if (i < s) {
      double val = base[i * ld + col];
      if (has) val = fma(gain, v, val);
      if (add2) {
        int j = row_map[i];
        if (j >= 0) val += add2[(int64_t)j * ld + col];
      }
      out[i * ld + col] = val;
    }
  }
}

// CTA-tiled form of k_heat_iir with warp-parallel recursions (default).  A CTA owns 32
// consecutive (window, RHS) columns and R output rows.  The input rows [i0 - H,
// i0 + R + H] are staged once into shared memory, coalesced (one 256-byte row segment
// per warp load): 1 + (2H + 1)/R input reads per output instead of the (TI + 2H + 1)/TI
// of the thread-per-chunk form, whose warm-ups re-read the neighbours' rows from L2.
// Then each warp takes whole columns and runs both first-order recursions
// (u_j = x_j + rho u_{j-1} forward, v_i = u_i + rho v_{i+1} backward) in parallel over
// its 32 lanes: lane l owns CH consecutive rows, runs the recursion locally from zero,
// the lanes' end values are combined by a shuffle scan of the affine maps
// (a, b) o (a', b') = (a a', b a' + b') with a = rho^len, and each lane adds its carry
// times rho^(t+1).  Same operator (restart H rows outside the output range, dropped tail
// < 1e-17 relative), other rounding order than k_heat_iir.  Results go back to shared
// memory and leave as coalesced rows: out = base + gain * v (+ the H^T scatter).
template <int H, int R, int WARPS>
__global__ void __launch_bounds__(WARPS * 32, R <= 128 ? 4 : 2) k_heat_iir_scan(
    double *out, const double *base, const double *in, const double *add2, const int *row_map,
    double rho, double gain, int s, int W, int m, int w_first, int w_step, int nw, int dir,
    const double *halo, int w0, int WG) {
  constexpr int NS = R + 2 * H + 1;          // staged rows i0 - H .. i0 + R + H
  constexpr int LD = 33;                     // padded row stride (doubles)
  constexpr int CH0 = (NS + 31) / 32;
  constexpr int CH = CH0 | 1;                // odd: lane strides CH*LD hit distinct banks
  extern __shared__ double tile[];           // [NS][LD]
  const int64_t ld = (int64_t)W * m;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int i0 = blockIdx.y * R;
  // this lane's column (load / store phases)
  const int cc = blockIdx.x * 32 + lane;
  const bool live = cc < nw * m;
  const int tt = live ? cc / m : 0, r = live ? cc - tt * m : 0;
  const int w = w_first + tt * w_step, ws = w + dir;
  const bool has = live && (w0 + ws >= 0 && w0 + ws < WG);
  const bool from_halo = (ws < 0 || ws >= W);
  // this thread's rows of `base` (and of the H^T scatter) are loaded into registers now,
  // in flight together with the staged tile: the store phase then issues no dependent
  // loads (r02n: one base load per store left every warp waiting ~1 us per row).  Each
  // element of base / out is read and written only by this thread, so in-place calls
  // (out == base) stay exact.
  constexpr int RPW = (R + WARPS - 1) / WARPS;
  const int64_t ocol = (int64_t)w * m + r;
  double bv[RPW];
#pragma unroll
  for (int k = 0; k < RPW; ++k) {
    const int i = i0 + warp + k * WARPS;
    bv[k] = (live && warp + k * WARPS < R && i < s) ? base[(int64_t)i * ld + ocol] : 0.0;
  }
  {
    // all NS x 32 loads in flight at once: cp.async straight into shared memory (ncu
    // r02e: register-staged loads left this kernel long-scoreboard bound at 12% of DRAM
    // bandwidth); a missing source (no M term, or a dead lane) zero-fills
    const double *src = has ? (from_halo ? halo + r : in + (int64_t)ws * m + r) : in;
    const int64_t sld = from_halo ? (int64_t)m : ld;
    int row = (i0 - H + warp) % s;
    row = row < 0 ? row + s : row;
#pragma unroll 4
    for (int j = warp; j < NS; j += WARPS) {
      cp_async8(tile + j * LD + lane, has ? src + (int64_t)row * sld : src, has ? 8 : 0);
      row += WARPS;
      while (row >= s) row -= s;
    }
    cp_async_commit();
    cp_async_wait<0>();
  }
  __syncthreads();
  // recursions, one column per warp at a time; lane l owns rows [l*CH, l*CH + len)
  const int j0 = lane * CH;
  const int len = max(0, min(CH, NS - j0));
  double rl = 1.0;                           // rho^len
  for (int t = 0; t < len; ++t) rl *= rho;
  // two columns per pass: their recursions and shuffle scans are independent (ILP 2)
  static_assert((32 / WARPS) % 2 == 0, "columns per warp must be even");
  for (int c = warp; c < 32; c += 2 * WARPS) {
    double *col[2] = {tile + c, tile + c + WARPS};
    // forward, local from zero
    double u[2] = {0.0, 0.0};
#pragma unroll
    for (int t = 0; t < CH; ++t)
      if (t < len) {
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          u[q] = fma(rho, u[q], col[q][(j0 + t) * LD]);
          col[q][(j0 + t) * LD] = u[q];
        }
      }
    // inclusive scan of (a, b) = (rho^len, u_end) over the lanes
    double a = rl, b[2] = {u[0], u[1]};
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double ap = __shfl_up_sync(0xffffffffu, a, o);
      const double b0 = __shfl_up_sync(0xffffffffu, b[0], o);
      const double b1 = __shfl_up_sync(0xffffffffu, b[1], o);
      if (lane >= o) { b[0] = fma(b0, a, b[0]); b[1] = fma(b1, a, b[1]); a *= ap; }
    }
    double carry[2];   // state entering this lane's rows
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      carry[q] = __shfl_up_sync(0xffffffffu, b[q], 1);
      if (lane == 0) carry[q] = 0.0;
    }
    double pw = rho;
#pragma unroll
    for (int t = 0; t < CH; ++t)
      if (t < len) {
#pragma unroll
        for (int q = 0; q < 2; ++q)
          col[q][(j0 + t) * LD] = fma(carry[q], pw, col[q][(j0 + t) * LD]);
        pw *= rho;
      }
    __syncwarp();
    // backward, local from zero, then the carry from the lanes above
    double v[2] = {0.0, 0.0};
#pragma unroll
    for (int t = CH - 1; t >= 0; --t)
      if (t < len) {
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          v[q] = fma(rho, v[q], col[q][(j0 + t) * LD]);
          col[q][(j0 + t) * LD] = v[q];
        }
      }
    a = rl; b[0] = v[0]; b[1] = v[1];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double an = __shfl_down_sync(0xffffffffu, a, o);
      const double b0 = __shfl_down_sync(0xffffffffu, b[0], o);
      const double b1 = __shfl_down_sync(0xffffffffu, b[1], o);
      if (lane + o < 32) { b[0] = fma(b0, a, b[0]); b[1] = fma(b1, a, b[1]); a *= an; }
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      carry[q] = __shfl_down_sync(0xffffffffu, b[q], 1);
      if (lane == 31) carry[q] = 0.0;
    }
    pw = rho;
#pragma unroll
    for (int t = CH - 1; t >= 0; --t)
      if (t < len) {
#pragma unroll
        for (int q = 0; q < 2; ++q)
          col[q][(j0 + t) * LD] = fma(carry[q], pw, col[q][(j0 + t) * LD]);
        pw *= rho;
      }
    __syncwarp();
  }
  __syncthreads();
  if (!live) return;
  if (!add2) {
#pragma unroll
    for (int k = 0; k < RPW; ++k) {
      const int j = H + warp + k * WARPS;
      const int i = i0 + j - H;
      if (j < H + R && i < s)
        out[(int64_t)i * ld + ocol] = has ? fma(gain, tile[j * LD + lane], bv[k]) : bv[k];
    }
    return;
  }
  // H^T scatter (the L^T x1 pass): its rows loaded 8 at a time ahead of their stores
  constexpr int KB = RPW < 8 ? RPW : 8;
#pragma unroll
  for (int k0 = 0; k0 < RPW; k0 += KB) {
    double a2[KB];
#pragma unroll
    for (int kk = 0; kk < KB; ++kk) {
      const int k = k0 + kk, i = i0 + warp + k * WARPS;
      a2[kk] = 0.0;
      if (k < RPW && warp + k * WARPS < R && i < s) {
        const int q = row_map[i];
        if (q >= 0) a2[kk] = add2[(int64_t)q * ld + ocol];
      }
    }
#pragma unroll
    for (int kk = 0; kk < KB; ++kk) {
      const int k = k0 + kk;
      const int j = H + warp + k * WARPS;
      const int i = i0 + j - H;
      if (k < RPW && j < H + R && i < s) {
        double val = has ? fma(gain, tile[j * LD + lane], bv[k]) : bv[k];
        out[(int64_t)i * ld + ocol] = val + a2[kk];   // (base + gain v) + scatter, as before
      }
    }
  }
}

// Column-sequential form (default, r02o): the same two first-order recursions as
// k_heat_iir, but every lane runs its column's recursions serially over rows staged in
// shared memory, instead of splitting a column over a warp with a shuffle scan (ncu r02n:
// k_heat_iir_scan issued ~150 thread instructions per output and sat at 78% L1 / shared
// memory busy with DRAM at 26%).  A CTA owns 32 consecutive (window, RHS) columns (lane =
// column) and WARPS * R output rows; warp w owns rows [wR, wR + R) of the tile.  The
// input rows [i0 - H, i0 + WARPS R + H] land in shared memory by cp.async (one
// coalesced row of 32 columns per warp instruction, zero-filled where there is no
// source); meanwhile each lane loads its R rows of `base` into registers.  Then
//   1. warm-up: u from zero over the H rows before the warp's own rows (the previous
//      warp's rows -- read before step 2 overwrites them);
//   2. forward over the own rows, u written back in place (the last warp continues
//      over the H + 1 rows below the tile);
//   3. backward from H + 1 rows below the own rows (the next warp's u) down through
//      the own rows, each output leaving as out = base + gain v (+ the H^T scatter).
// This is k_heat_iir's arithmetic with TI = R (restart H rows early, dropped tail
// < 1e-17 relative), at ~(2H + 1) / R + 2 serial FMAs per output and one shared load
// each; the tile is read from DRAM once (plus its 2H-row halo, mostly L2 hits).
// resident CTAs per SM: as many as shared memory allows (228 KB, 1 KB reserved per CTA),
// but never fewer than 64 registers per thread (R = 16's 16 staged base rows)
template <int H, int R, int WARPS>
constexpr int heat_seq_ctas() {
  constexpr int by_smem = (228 * 1024) / ((WARPS * R + 2 * H + 1) * 256 + 1024);
  constexpr int by_reg = 1024 / (WARPS * 32);   // keep >= 64 registers per thread
  return by_smem < by_reg ? by_smem : by_reg;
}

// -DHEAT_SEQ_MAXNREG=n (probe r02ay): cap the kernel's registers below the 64 that, with
// two 4-warp k_gemm_tma CTAs at 192, fill an SM's register file exactly
template <int H, int R, int WARPS>
__global__ void
#ifdef HEAT_SEQ_MAXNREG
__maxnreg__(HEAT_SEQ_MAXNREG)
#else
__launch_bounds__(WARPS * 32, heat_seq_ctas<H, R, WARPS>())
#endif
k_heat_iir_seq(double *out, const double *base, const double *in, const double *add2,
               const int *row_map, double rho, double gain, int s, int W, int m, int w_first,
               int w_step, int nw, int dir, const double *halo, int w0, int WG) {
  constexpr int T = WARPS * R + 2 * H + 1;   // staged rows i0 - H .. i0 + WARPS R + H
  extern __shared__ double tile[];           // [T][32]
  const int64_t ld = (int64_t)W * m;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int i0 = blockIdx.y * (WARPS * R);
  const int cc = blockIdx.x * 32 + lane;
  const bool live = cc < nw * m;
  const int tt = live ? cc / m : 0, r = live ? cc - tt * m : 0;
  const int w = w_first + tt * w_step, ws = w + dir;
  const bool has = live && (w0 + ws >= 0 && w0 + ws < WG);
  const bool from_halo = (ws < 0 || ws >= W);
  const int64_t ocol = (int64_t)w * m + r;
  {
    const double *src = has ? (from_halo ? halo + r : in + (int64_t)ws * m + r) : in;
    const int64_t sld = from_halo ? (int64_t)m : ld;
    int row = (i0 - H + warp) % s;
    row = row < 0 ? row + s : row;
#pragma unroll 4
    for (int j = warp; j < T; j += WARPS) {
      cp_async8(tile + j * 32 + lane, has ? src + (int64_t)row * sld : src, has ? 8 : 0);
      row += WARPS;
      while (row >= s) row -= s;
    }
    cp_async_commit();
  }
  const int ob = i0 + warp * R;   // first output row of this warp
  double bv[R];
#pragma unroll
  for (int k = 0; k < R; ++k)
    bv[k] = (live && ob + k < s) ? base[(int64_t)(ob + k) * ld + ocol] : 0.0;
  cp_async_wait<0>();
  __syncthreads();
  const int t0 = H + warp * R;    // tile row of the warp's first output row
  // 1. warm-up over the H rows above (the previous warp's own rows, still x)
  double u = 0.0;
#pragma unroll
  for (int t = 0; t < H; ++t) u = fma(rho, u, tile[(t0 - H + t) * 32 + lane]);
  __syncthreads();
  // 2. forward over the own rows, in place (+ the tail below the tile: last warp)
#pragma unroll
  for (int t = 0; t < R; ++t) {
    u = fma(rho, u, tile[(t0 + t) * 32 + lane]);
    tile[(t0 + t) * 32 + lane] = u;
  }
  if (warp == WARPS - 1) {
#pragma unroll
    for (int t = 0; t <= H; ++t) {
      u = fma(rho, u, tile[(t0 + R + t) * 32 + lane]);
      tile[(t0 + R + t) * 32 + lane] = u;
    }
  }
  __syncthreads();
  // 3. backward: warm-up over the H + 1 rows below, then the own rows -> out
  double v = 0.0;
#pragma unroll
  for (int t = H; t >= 0; --t) v = fma(rho, v, tile[(t0 + R + t) * 32 + lane]);
  if (!live) return;
  if (!add2) {
#pragma unroll
    for (int t = R - 1; t >= 0; --t) {
      v = fma(rho, v, tile[(t0 + t) * 32 + lane]);
      if (ob + t < s) out[(int64_t)(ob + t) * ld + ocol] = has ? fma(gain, v, bv[t]) : bv[t];
    }
    return;
  }
  // H^T scatter (the L^T x1 pass): its rows loaded 8 at a time ahead of their stores
  constexpr int KB = R < 8 ? R : 8;
#pragma unroll
  for (int t1 = R; t1 > 0; t1 -= KB) {
    double a2[KB];
#pragma unroll
    for (int q = 0; q < KB; ++q) {
      const int t = t1 - 1 - q;
      a2[q] = 0.0;
      if (t >= 0 && ob + t < s) {
        const int qq = row_map[ob + t];
        if (qq >= 0) a2[q] = add2[(int64_t)qq * ld + ocol];
      }
    }
#pragma unroll
    for (int q = 0; q < KB; ++q) {
      const int t = t1 - 1 - q;
      if (t < 0) break;
      v = fma(rho, v, tile[(t0 + t) * 32 + lane]);
      if (ob + t < s) {
        const double val = has ? fma(gain, v, bv[t]) : bv[t];
        out[(int64_t)(ob + t) * ld + ocol] = val + a2[q];   // (base + gain v) + scatter
      }
    }
  }
}

// The paper's own heat model: M = M_dt^NS, M_dt the forward-Euler
// Dirichlet step (rows 0 and s-1 zero; interior (r, 1-2r, r), the boundary columns
// carrying coefficient 0).  M_dt is symmetric, so M^T = M.  One thread per (window,
// RHS) column and TI consecutive rows; the NS sweeps run in registers on the rows
// [i0 - NS, i0 + TI + NS) (the light cone of the chunk), boundary and out-of-range
// rows held at zero.
template <int NS, int TI>
__global__ void __launch_bounds__(128) k_heat_explicit(double *out, const double *base,
                                                       const double *in, const double *add2,
                                                       const int *row_map, double r, double sign,
                                                       int s, int W, int m, int w_first,
                                                       int w_step, int nw, int dir,
                                                       const double *halo, int w0, int WG) {
  const int64_t ld = (int64_t)W * m;
  const int cc = blockIdx.x * blockDim.x + threadIdx.x;
  if (cc >= nw * m) return;
  const int tt = cc / m, rr = cc - tt * m;
  const int w = w_first + tt * w_step;
  const int ws = w + dir;
  const bool has = (w0 + ws >= 0 && w0 + ws < WG);
  const bool from_halo = (ws < 0 || ws >= W);
  const int64_t col = (int64_t)w * m + rr;
  const double *src = from_halo ? halo + rr : in + (int64_t)ws * m + rr;
  const int64_t sld = from_halo ? (int64_t)m : ld;
  const int i0 = blockIdx.y * TI;
  constexpr int L = TI + 2 * NS;
  double v[L];
  if (has) {
#pragma unroll
    for (int j = 0; j < L; ++j) {
      const int i = i0 - NS + j;
      v[j] = (i >= 1 && i <= s - 2) ? __ldg(src + (int64_t)i * sld) : 0.0;
    }
    const double d = 1.0 - 2.0 * r;
#pragma unroll
    for (int st = 0; st < NS; ++st) {
      double prev = v[st];
#pragma unroll
      for (int j = st + 1; j < L - 1 - st; ++j) {
        const int i = i0 - NS + j;
        const double nv = (i >= 1 && i <= s - 2) ? fma(r, prev + v[j + 1], d * v[j]) : 0.0;
        prev = v[j];
        v[j] = nv;
      }
    }
  }
#pragma unroll
  for (int o = 0; o < TI; ++o) {
    const int i = i0 + o;
    if (i < s) {
      double val = base[i * ld + col];
      if (has) val = fma(sign, v[NS + o], val);
      if (add2) {
        int j = row_map[i];
        if (j >= 0) val += add2[(int64_t)j * ld + col];
      }
      out[i * ld + col] = val;
    }
  }
}

template <int NS>
static void heat_explicit_launch(Ctx &c, bool transpose, double sign, const double *in,
                                 const double *base, double *out, int w_first, int w_step,
                                 int nw, const double *add2, const int *row_map) {
  // r01bh, NEXT-1 per step: TI = 32 / 16 / 8 -> 0.901 / 0.887 / 0.876 ms
  static const int ti_env = env_int("WF4DVAR_HEAT_EXPL_TI", 8);   // tuning experiments only
  int cols = nw * c.m;
  auto go = [&](auto ti_tag) {
    constexpr int TI = decltype(ti_tag)::value;
    dim3 grid((cols + 127) / 128, (c.s + TI - 1) / TI);
    k_heat_explicit<NS, TI><<<grid, 128, 0, c.st>>>(out, base, in, add2, row_map, c.heat_r,
                                                     sign, c.s, c.W, c.m, w_first, w_step, nw,
                                                     transpose ? 1 : -1,
                                                     transpose ? c.halo_hi : c.halo_lo, c.w0,
                                                     c.WG);
  };
  if (ti_env == 32) go(std::integral_constant<int, 32>{});
  else if (ti_env == 16) go(std::integral_constant<int, 16>{});
  else go(std::integral_constant<int, 8>{});
  WF_CUDA(cudaGetLastError());
}

// Same recursions, the forward one streamed over register batches of 16 independent
// loads (coalesced across the CTA's 128 columns) and its results kept in shared
// memory only for the rows the backward pass reads (each thread owns one column:
// no barriers) -- the register version exposed one global-load latency per step.
template <int H, int TI>
__global__ void __launch_bounds__(128) k_heat_iir_smem(double *out, const double *base,
                                                       const double *in, const double *add2,
                                                       const int *row_map, double rho,
                                                       double gain, int s, int W, int m,
                                                       int w_first, int w_step, int nw, int dir,
                                                       const double *halo, int w0, int WG) {
  constexpr int R = TI + 2 * H + 1;      // rows i0 - H .. i0 + TI + H
  constexpr int RU = TI + H + 1;         // rows kept for the backward pass (i0 ..)
  extern __shared__ double tile[];       // [RU][128]; thread t owns column t (no barrier)
  const int64_t ld = (int64_t)W * m;
  const int tid = threadIdx.x;
  const int i0 = blockIdx.y * TI;
  const int cc = blockIdx.x * 128 + tid;
  if (cc >= nw * m) return;
  const int tt = cc / m, r = cc - tt * m;
  const int w = w_first + tt * w_step, ws = w + dir;
  const bool has = (w0 + ws >= 0 && w0 + ws < WG);
  const int64_t col = (int64_t)w * m + r;
  double *tc = tile + tid;
  double v = 0.0;
  if (has) {
    // forward recursion streamed over the input rows, 16 loads in flight per thread;
    // u is kept (in shared memory) only for the rows the backward pass needs
    const double *src = (ws < 0 || ws >= W) ? halo + r : in + (int64_t)ws * m + r;
    const int64_t sld = (ws < 0 || ws >= W) ? (int64_t)m : ld;
    int row0 = (i0 - H) % s;
    row0 = row0 < 0 ? row0 + s : row0;
    double u = 0.0;
    for (int j = 0; j < R; j += 16) {
      double x[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        int row = row0 + j + q;
        row = row >= s ? row - s : row;
        row = row >= s ? row % s : row;
        x[q] = (j + q < R) ? __ldg(src + (int64_t)row * sld) : 0.0;
      }
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        if (j + q < R) {
          u = fma(rho, u, x[q]);
          if (j + q >= H) tc[(j + q - H) * 128] = u;
        }
      }
    }
    // backward: v_i = u_i + rho v_{i+1} from the last kept row; outputs rows i0..i0+TI-1
#pragma unroll 8
    for (int j = RU - 1; j >= TI; --j) v = fma(rho, v, tc[j * 128]);
  }
#pragma unroll 4
  for (int j = TI - 1; j >= 0; --j) {
    if (has) v = fma(rho, v, tc[j * 128]);
    const int i = i0 + j;
    if (i < s) {
      double val = base[(int64_t)i * ld + col];
      if (has) val = fma(gain, v, val);
      if (add2) {
        int jj = row_map[i];
        if (jj >= 0) val += add2[(int64_t)jj * ld + col];
      }
      out[(int64_t)i * ld + col] = val;
    }
  }
}

// z_w += z_{w-1} (forward, w ascending) or z_w += z_{w+1} (backward): L_I^{-1} / L_I^{-T}
__global__ void k_window_scan(double *z, int rows, int W, int m, int dir) {
  const int64_t ld = (int64_t)W * m;
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)rows * m) return;
  int64_t i = e / m, r = e % m;
  double *p = z + i * ld + r;
  if (dir > 0) {
    double acc = p[0];
    for (int w = 1; w < W; ++w) { acc += p[(int64_t)w * m]; p[(int64_t)w * m] = acc; }
  } else {
    double acc = p[(int64_t)(W - 1) * m];
    for (int w = W - 2; w >= 0; --w) { acc += p[(int64_t)w * m]; p[(int64_t)w * m] = acc; }
  }
}

// out[H_idx[j]][col] += add2[j][col] for every column (dense-model path of H^T)
__global__ void k_scatter_add(double *out, const double *add2, const int *H_idx, int p,
                              int64_t ld) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)p * ld) return;
  int64_t j = e / ld, c = e % ld;
  out[(int64_t)H_idx[j] * ld + c] += add2[e];
}

template <int H>
static void heat_iir_launch(Ctx &c, bool transpose, double sign, const double *in,
                            const double *base, double *out, int w_first, int w_step, int nw,
                            const double *add2, const int *row_map) {
  int cols = nw * c.m;
  // r01t: the staged variant measured no faster (15.4 vs 14.5 ms per 11 steps) -> opt-in
  static const int smem_env = env_int("WF4DVAR_HEAT_IIR_SMEM", 0);   // tuning experiments only
  if (smem_env) {
    constexpr int TI = 32;
    constexpr size_t smem = (size_t)(TI + H + 1) * 128 * sizeof(double);
    static const cudaError_t attr = cudaFuncSetAttribute(k_heat_iir_smem<H, TI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem);
    WF_CUDA(attr);
    dim3 grid((cols + 127) / 128, (c.s + TI - 1) / TI);
    k_heat_iir_smem<H, TI><<<grid, 128, smem, c.st>>>(out, base, in, add2, row_map, c.heat_rho,
                                                      sign * c.heat_gain, c.s, c.W, c.m, w_first,
                                                      w_step, nw, transpose ? 1 : -1,
                                                      transpose ? c.halo_hi : c.halo_lo, c.w0,
                                                      c.WG);
  } else {
    // rows per thread: r01bf/bg per step, TI = 32 / 16 / 8: c3 30.39 / 30.09 / 30.03 ms,
    // c1 0.318 / 0.290 / 0.276 ms, c0 0.151 / 0.137 / 0.128 ms -- the recursions are
    // latency-bound chains; shorter chunks (the H-row warm-ups re-read from L2) give
    // more independent chains and fewer registers (higher occupancy)
    // r02f (configs[3] per step): thread-per-chunk 1.264 ms (2.31 TB/s) -> warp-scan with
    // cp.async staging R = 128: 1.110 ms (2.63 TB/s), R = 256: 1.431 ms (fewer CTAs per SM)
    // r02o: column-sequential kernel (WF4DVAR_HEAT_SEQ = rows per warp, 0: off)
    static const int seq_env = env_int("WF4DVAR_HEAT_SEQ", 16);   // r02p: R = 16 4.92 TB/s, 32: 4.61
    static const int seqw_env = env_int("WF4DVAR_HEAT_SEQW", 8);   // warps per CTA (4 / 8 / 16)
    // small launches (configs[1]'s chain steps: 80 columns x 1000 rows = 24 CTAs of 32 x 128)
    // leave most SMs idle; WF4DVAR_HEAT_SEQ_MINCTA=K sends launches of fewer than K such
    // CTAs to the thread-per-chunk form (8 rows per thread, 128 columns per CTA: 125 CTAs
    // there).  r02w, configs[1] MINRES step: K = 148 0.340 ms, off (default) 0.336 ms
    static const int seq_min = env_int("WF4DVAR_HEAT_SEQ_MINCTA", 0);
    const int seq_ctas = ((cols + 31) / 32) * ((c.s + 8 * seq_env - 1) / (8 * std::max(seq_env, 1)));
    if ((seq_env == 16 || seq_env == 32) && seq_ctas >= seq_min) {
      auto go2 = [&](auto r_tag, auto w_tag) {
        constexpr int R = decltype(r_tag)::value;
        constexpr int WARPS = decltype(w_tag)::value;
        constexpr size_t smem = (size_t)(WARPS * R + 2 * H + 1) * 32 * sizeof(double);
        static const cudaError_t attr = cudaFuncSetAttribute(
            k_heat_iir_seq<H, R, WARPS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        WF_CUDA(attr);
        dim3 grid((cols + 31) / 32, (c.s + WARPS * R - 1) / (WARPS * R));
        k_heat_iir_seq<H, R, WARPS><<<grid, WARPS * 32, smem, c.st>>>(
            out, base, in, add2, row_map, c.heat_rho, sign * c.heat_gain, c.s, c.W, c.m, w_first,
            w_step, nw, transpose ? 1 : -1, transpose ? c.halo_hi : c.halo_lo, c.w0, c.WG);
      };
      using I16 = std::integral_constant<int, 16>;
      if (seq_env == 32) go2(std::integral_constant<int, 32>{}, std::integral_constant<int, 8>{});
      else if (seqw_env == 4) go2(I16{}, std::integral_constant<int, 4>{});
      else if (seqw_env == 16) go2(I16{}, std::integral_constant<int, 16>{});
      else go2(I16{}, std::integral_constant<int, 8>{});
      WF_CUDA(cudaGetLastError());
      return;
    }
    static const int tile_env = env_int("WF4DVAR_HEAT_TILE", 128);   // 0: thread-per-chunk form
    // (the warp-scan form: opt-in, WF4DVAR_HEAT_SEQ=0; launches too small for the
    // column-sequential kernel take the thread-per-chunk form below)
    const bool small = (seq_env == 16 || seq_env == 32);   // seq default, too few CTAs
    if (!small && (tile_env == 64 || tile_env == 128 || tile_env == 256)) {
      constexpr int WARPS = 8;
      auto go = [&](auto r_tag) {
        constexpr int R = decltype(r_tag)::value;
        constexpr size_t smem = (size_t)(R + 2 * H + 1) * 33 * sizeof(double);
        static const cudaError_t attr = cudaFuncSetAttribute(
            k_heat_iir_scan<H, R, WARPS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        WF_CUDA(attr);
        dim3 grid((cols + 31) / 32, (c.s + R - 1) / R);
        k_heat_iir_scan<H, R, WARPS><<<grid, WARPS * 32, smem, c.st>>>(
            out, base, in, add2, row_map, c.heat_rho, sign * c.heat_gain, c.s, c.W, c.m, w_first,
            w_step, nw, transpose ? 1 : -1, transpose ? c.halo_hi : c.halo_lo, c.w0, c.WG);
      };
      if (tile_env == 128) go(std::integral_constant<int, 128>{});
      else if (tile_env == 64) go(std::integral_constant<int, 64>{});
      else go(std::integral_constant<int, 256>{});
      WF_CUDA(cudaGetLastError());
      return;
    }
    static const int ti_env = env_int("WF4DVAR_HEAT_TI", 8);   // tuning experiments only
    auto go = [&](auto ti_tag) {
      constexpr int TI = decltype(ti_tag)::value;
      dim3 grid((cols + 127) / 128, (c.s + TI - 1) / TI);
      k_heat_iir<H, TI><<<grid, 128, 0, c.st>>>(out, base, in, add2, row_map, c.heat_rho,
                                                sign * c.heat_gain, c.s, c.W, c.m, w_first,
                                                w_step, nw, transpose ? 1 : -1,
                                                transpose ? c.halo_hi : c.halo_lo, c.w0, c.WG);
    };
    if (ti_env == 16) go(std::integral_constant<int, 16>{});
    else if (ti_env == 64) go(std::integral_constant<int, 64>{});
    else if (ti_env == 48) go(std::integral_constant<int, 48>{});
    else if (ti_env == 32) go(std::integral_constant<int, 32>{});
    else go(std::integral_constant<int, 8>{});
  }
  WF_CUDA(cudaGetLastError());
}

template <int D>
static void heat_launch(Ctx &c, bool transpose, double sign, const double *in, const double *base,
                        double *out, int w_first, int w_step, int nw, const double *add2,
                        const int *row_map) {
  constexpr int TI = 16;
  Taps taps;
  for (int d = 0; d <= 2 * D; ++d) taps.t[d] = c.heat_taps[d - D + c.heat_D];
  int cols = nw * c.m;
  dim3 grid((cols + 127) / 128, (c.s + TI - 1) / TI);
  k_heat_step<D, TI><<<grid, 128, 0, c.st>>>(out, base, in, add2, row_map, taps, sign, c.s, c.W,
                                              c.m, w_first, w_step, nw, transpose ? 1 : -1,
                                              transpose ? c.halo_hi : c.halo_lo, c.w0, c.WG);
  WF_CUDA(cudaGetLastError());
}

void model_step(Ctx &c, bool transpose, double sign, const double *in, const double *base,
                double *out, int w_first, int w_step, int nw, const double *add2,
                const int *row_map) {
  if (nw <= 0) return;
  const int s = c.s, m = c.m;
  const int64_t ld = c.ncol;
  if (c.model == WF4DVAR_M_L96) {
    l96_step(c, transpose, sign, in, base, out, w_first, w_step, nw, add2, row_map);
    return;
  }
  if (c.model == WF4DVAR_M_HEAT_EXPLICIT) {
    double elems = (double)nw * s * m;
    LaunchScope ls(c, K_MODEL, elems * 4.0 * c.heat_nsteps, elems * 8.0 * 3);
    switch (c.heat_nsteps) {
      case 1: heat_explicit_launch<1>(c, transpose, sign, in, base, out, w_first, w_step, nw, add2, row_map); break;
      case 2: heat_explicit_launch<2>(c, transpose, sign, in, base, out, w_first, w_step, nw, add2, row_map); break;
      case 3: heat_explicit_launch<3>(c, transpose, sign, in, base, out, w_first, w_step, nw, add2, row_map); break;
      case 4: heat_explicit_launch<4>(c, transpose, sign, in, base, out, w_first, w_step, nw, add2, row_map); break;
      case 5: heat_explicit_launch<5>(c, transpose, sign, in, base, out, w_first, w_step, nw, add2, row_map); break;
      case 6: heat_explicit_launch<6>(c, transpose, sign, in, base, out, w_first, w_step, nw, add2, row_map); break;
      case 7: heat_explicit_launch<7>(c, transpose, sign, in, base, out, w_first, w_step, nw, add2, row_map); break;
      default: heat_explicit_launch<8>(c, transpose, sign, in, base, out, w_first, w_step, nw, add2, row_map); break;
    }
    c.launches++;
    return;
  }
  if (c.model == WF4DVAR_M_HEAT && c.heat_D > 0 && c.heat_iir) {
    // algorithmic work per output: the two first-order recursions (2 FMAs) and the
    // epilogue FMA; bytes: read in, read base, write out
    double elems = (double)nw * s * m;
    LaunchScope ls(c, K_MODEL, elems * 2.0 * 3, elems * 8.0 * 3);
    switch (c.heat_D) {
      case 8: heat_iir_launch<8>(c, transpose, sign, in, base, out, w_first, w_step, nw, add2, row_map); break;
      case 16: heat_iir_launch<16>(c, transpose, sign, in, base, out, w_first, w_step, nw, add2, row_map); break;
      case 24: heat_iir_launch<24>(c, transpose, sign, in, base, out, w_first, w_step, nw, add2, row_map); break;
      default: heat_iir_launch<32>(c, transpose, sign, in, base, out, w_first, w_step, nw, add2, row_map); break;
    }
    c.launches++;
    return;
  }
  if (c.model == WF4DVAR_M_HEAT && c.heat_D > 0) {
    double elems = (double)nw * s * m;
    LaunchScope ls(c, K_MODEL, elems * 2.0 * (2 * c.heat_D + 1), elems * 8.0 * 3);
    switch (c.heat_D) {
      case 8: heat_launch<8>(c, transpose, sign, in, base, out, w_first, w_step, nw, add2, row_map); break;
      case 16: heat_launch<16>(c, transpose, sign, in, base, out, w_first, w_step, nw, add2, row_map); break;
      case 24: heat_launch<24>(c, transpose, sign, in, base, out, w_first, w_step, nw, add2, row_map); break;
      default: heat_launch<32>(c, transpose, sign, in, base, out, w_first, w_step, nw, add2, row_map); break;
    }
    c.launches++;
    return;
  }
  if (c.model == WF4DVAR_M_DENSE || c.model == WF4DVAR_M_HEAT) {
    // Windows without a (global) source -- w = 0 forward, w = N transposed -- are a
    // copy of base; a source owned by the neighbour rank comes from the halo.
    const int dir = transpose ? 1 : -1;
    auto src_ok = [&](int t) {
      int ws = c.w0 + w_first + t * w_step + dir;
      return ws >= 0 && ws < c.WG;
    };
    auto src_halo = [&](int t) {
      int ws = w_first + t * w_step + dir;
      return ws < 0 || ws >= c.W;
    };
    auto mat = [&](int w) {   // M_w at Mdense[w-1]; M_{w+1}^T at MdenseT[w]  (global w)
      return transpose ? c.MdenseT + (int64_t)(c.w0 + w) * s * s
                       : c.Mdense + (int64_t)(c.w0 + w - 1) * s * s;
    };
    int t0 = 0, t1 = nw;
    for (int t = 0; t < nw; ++t) {
      int w = w_first + t * w_step;
      if (!src_ok(t)) {
        if (out != base)
          WF_CUDA(cudaMemcpy2DAsync(out + (int64_t)w * m, ld * 8, base + (int64_t)w * m, ld * 8,
                                    m * 8, s, cudaMemcpyDeviceToDevice, c.st));
      } else if (src_halo(t)) {
        GemmProb g{};
        g.A = mat(w); g.lda = s;
        g.X = transpose ? c.halo_hi : c.halo_lo; g.ldx = m;
        g.Y = out + (int64_t)w * m; g.ldy = ld;
        g.Z = base + (int64_t)w * m; g.ldz = ld;
        g.M = s; g.N = m; g.K = s; g.alpha = sign; g.beta = 1.0;
        launch_gemm(c, &g, 1, 1);
      }
    }
    auto plain = [&](int t) { return src_ok(t) && !src_halo(t); };
    while (t0 < t1 && !plain(t0)) ++t0;
    while (t1 > t0 && !plain(t1 - 1)) --t1;
    if (t1 > t0) {
      int wf0 = w_first + t0 * w_step;
      GemmProb g{};
      g.A = mat(wf0);
      g.lda = s; g.sA = (int64_t)w_step * s * s;
      g.X = in + (int64_t)(wf0 + dir) * m; g.ldx = ld; g.sX = (int64_t)w_step * m;
      g.Y = out + (int64_t)wf0 * m; g.ldy = ld; g.sY = (int64_t)w_step * m;
      g.Z = base + (int64_t)wf0 * m; g.ldz = ld; g.sZ = (int64_t)w_step * m;
      g.zrow = nullptr;
      g.M = s; g.N = m; g.K = s;
      g.alpha = sign; g.beta = 1.0;
      launch_gemm(c, &g, 1, t1 - t0);
    }
    if (add2) {
      // H^T scatter on every target window (only used with w_step == 1 over all windows)
      LaunchScope ls(c, K_VEC, 0, (double)c.p * ld * 16);
      int64_t tot = (int64_t)c.p * ld;
      k_scatter_add<<<(unsigned)((tot + 255) / 256), 256, 0, c.st>>>(out, add2, c.H_idx, c.p, ld);
      WF_CUDA(cudaGetLastError());
      c.launches++;
    }
    return;
  }
  throw Error{WF4DVAR_EINVAL, "model not supported by model_step"};
}

// out[i][w][r] += sum_{q in [qlo, qhi)} tot[q][i][r] for every local window w
__global__ void k_add_totals(double *z, const double *tot, int qlo, int qhi, int s, int W, int m) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)s * m) return;
  int64_t i = e / m, r = e % m;
  double add = 0.0;
  for (int q = qlo; q < qhi; ++q) add += tot[(int64_t)q * s * m + e];   // fixed rank order
  if (add == 0.0 && qlo >= qhi) return;
  double *p = z + i * (int64_t)W * m + r;
  for (int w = 0; w < W; ++w) p[(int64_t)w * m] += add;
}

void pack_window(Ctx &c, double *dst, const double *seg, int wl) {
  WF_CUDA(cudaMemcpy2DAsync(dst, (size_t)c.m * 8, seg + (int64_t)wl * c.m, (size_t)c.ncol * 8,
                            (size_t)c.m * 8, c.s, cudaMemcpyDeviceToDevice, c.st));
}

void partition(int W, int world, int rank, int *w_begin, int *w_end) {
  const int base = W / world, rem = W % world;
  *w_begin = rank * base + std::min(rank, rem);
  *w_end = *w_begin + base + (rank < rem ? 1 : 0);
}

std::vector<ChainStep> chain_plan(int WG, int k, int w0, int w1, bool transpose) {
  std::vector<ChainStep> plan;
  const int L = std::min(k, WG);   // longest chain
  const int nfull = WG / k;
  const int last_len = WG - nfull * k;
  // backward position of w: distance to the end of its chain
  auto pos_bwd = [&](int w) { return std::min((w / k + 1) * k, WG) - 1 - w; };
  // first w >= lo with w mod k == res
  auto first_congruent = [&](int lo, int res) { return lo + (((res - lo) % k) + k) % k; };
  for (int j = 1; j < L; ++j) {
    ChainStep st{};
    st.j = j;
    if (!transpose) {
      // z_w = r_w + M_w z_{w-1} for w mod k == j
      st.recv = (w0 > 0 && w0 % k == j) ? 1 : 0;
      st.send = (w1 < WG && w1 % k == j) ? 1 : 0;
      int wf = first_congruent(w0, j);
      if (wf < w1) {
        st.first[0] = wf - w0; st.stride[0] = k; st.count[0] = (w1 - 1 - wf) / k + 1;
        st.nl = 1;
      }
    } else {
      // z_w = r_w + M_{w+1}^T z_{w+1} for the windows j before their chain end
      st.recv = (w1 < WG && pos_bwd(w1 - 1) == j) ? 1 : 0;
      st.send = (w0 > 0 && pos_bwd(w0 - 1) == j) ? 1 : 0;
      const int hi_full = std::min(w1, nfull * k);
      int wf = first_congruent(w0, k - 1 - j);
      if (wf < hi_full) {
        st.first[st.nl] = wf - w0; st.stride[st.nl] = k;
        st.count[st.nl] = (hi_full - 1 - wf) / k + 1;
        st.nl++;
      }
      const int wr = WG - 1 - j;   // ragged last chain [nfull k, WG)
      if (j < last_len && wr >= std::max(w0, nfull * k) && wr < w1) {
        st.first[st.nl] = wr - w0; st.stride[st.nl] = 1; st.count[st.nl] = 1;
        st.nl++;
      }
    }
    plan.push_back(st);
  }
  return plan;
}

// L_I^{-1} / L_I^{-T}: window prefix / suffix sums, local scan plus,
// across ranks, the sum of the other ranks' window totals (allgather, rank order).
static void li_scan(Ctx &c, bool transpose, double *z) {
  {
    LaunchScope ls(c, K_MODEL, 0, (double)c.s * c.ncol * 16);
    int64_t tot = (int64_t)c.s * c.m;
    k_window_scan<<<(unsigned)((tot + 127) / 128), 128, 0, c.st>>>(z, c.s, c.W, c.m,
                                                                   transpose ? -1 : 1);
    WF_CUDA(cudaGetLastError());
    c.launches++;
  }
  if (!c.comm) return;
  double *mine = transpose ? c.pack_lo : c.pack_hi;
  pack_window(c, mine, z, transpose ? 0 : c.W - 1);
  const size_t cnt = (size_t)c.s * c.m;
  c.comm->allgather(mine, c.gath, cnt, c.st);
  const int rank = c.comm->rank, world = c.comm->world;
  const int qlo = transpose ? rank + 1 : 0, qhi = transpose ? world : rank;
  if (qlo >= qhi) return;
  LaunchScope ls(c, K_MODEL, 0, (double)c.s * c.ncol * 16);
  k_add_totals<<<(unsigned)((cnt + 127) / 128), 128, 0, c.st>>>(z, c.gath, qlo, qhi, c.s, c.W, c.m);
  WF_CUDA(cudaGetLastError());
  c.launches++;
}

void lhat_solve(Ctx &c, bool transpose, double *z) {
  switch (c.pc.lhat) {
    case WF4DVAR_L0:
      return;
    case WF4DVAR_LI:
      li_scan(c, transpose, z);
      return;
    default: break;
  }
  const int k = (c.pc.lhat == WF4DVAR_LEXACT) ? c.WG : c.pc.k;
  if (k <= 1) return;
  const std::vector<ChainStep> plan = chain_plan(c.WG, k, c.w0, c.w0 + c.W, transpose);
  const size_t cnt = (size_t)c.s * c.m;
  for (const ChainStep &st : plan) {
    if (c.comm && (st.recv || st.send)) {
      // chain hand-off across the rank boundary (Lemma 4.2's serial product)
      std::vector<Comm::P2P> ops;
      const int rank = c.comm->rank;
      if (!transpose) {
        if (st.send) {
          pack_window(c, c.pack_hi, z, c.W - 1);
          ops.push_back({c.pack_hi, cnt, rank + 1, true});
        }
        if (st.recv) ops.push_back({c.halo_lo, cnt, rank - 1, false});
      } else {
        if (st.send) {
          pack_window(c, c.pack_lo, z, 0);
          ops.push_back({c.pack_lo, cnt, rank - 1, true});
        }
        if (st.recv) ops.push_back({c.halo_hi, cnt, rank + 1, false});
      }
      c.comm->exchange(ops, c.st);
    }
    if (c.model == WF4DVAR_M_L96 && st.nl == 2) {
      // the full chains' windows and the ragged last chain's window in ONE launch (a
      // one-window Lorenz-96 launch is pure latency: 11 us at configs[2], r02al)
      l96_step2(c, transpose, z, st.first[0], st.stride[0], st.count[0], st.first[1],
                st.count[1]);
      continue;
    }
    for (int l = 0; l < st.nl; ++l)
      model_step(c, transpose, 1.0, z, z, z, st.first[l], st.stride[l], st.count[l]);
  }
}

// --------------------------------------------------------------- setup
// Exact periodic row of M = (I - r Lap)^{-1}:
//   c_d = (rho^d + rho^(s-d)) / ((1 - rho^s) sqrt(1 + 4r)),  d = 0..s-1.
static void heat_row(int s, double r, std::vector<double> &row) {
  const double sq = std::sqrt(1.0 + 4.0 * r);
  const double rho = (1.0 + 2.0 * r - sq) / (2.0 * r);
  const double rs = std::pow(rho, s);
  row.assign(s, 0.0);
  for (int d = 0; d < s; ++d)
    row[d] = (std::pow(rho, d) + std::pow(rho, s - d)) / ((1.0 - rs) * sq);
}

void setup_model(Ctx &c, const wf4dvar_problem &p) {
  const int s = c.s, N = c.N;
  if (c.model == WF4DVAR_M_HEAT) {
    WF_REQUIRE(p.heat_r > 0, WF4DVAR_EINVAL, "heat_r must be > 0");
    std::vector<double> row;
    heat_row(s, p.heat_r, row);
    const double rho = (1.0 + 2.0 * p.heat_r - std::sqrt(1.0 + 4.0 * p.heat_r)) / (2.0 * p.heat_r);
    // smallest D with the dropped tail 2 rho^(D+1)/(1-rho) below 1e-17 * c_0
    int Dneed = 1;
    while (2.0 * std::pow(rho, Dneed + 1) / (1.0 - rho) > 1e-17 * row[0] && Dneed < 1000) ++Dneed;
    int D = Dneed <= 8 ? 8 : Dneed <= 16 ? 16 : Dneed <= 24 ? 24 : Dneed <= 32 ? 32 : 0;
    if (D > 0 && s >= 2 * D + 1) {
      c.heat_D = D;
      c.heat_rho = rho;
      c.heat_gain = rho / p.heat_r;
      if (const char *e = getenv("WF4DVAR_HEAT_STENCIL")) c.heat_iir = atoi(e) == 0;
      for (int d = -D; d <= D; ++d) c.heat_taps[d + D] = row[((d % s) + s) % s];
    } else {
      // small grid or slowly decaying row: materialise the exact circulant M and use
      // the dense (DMMA GEMM) path
      c.heat_D = 0;
      std::vector<double> M((size_t)s * s);
      for (int i = 0; i < s; ++i)
        for (int j = 0; j < s; ++j) M[(size_t)i * s + j] = row[((j - i) % s + s) % s];
      c.Mdense = c.alloc<double>((size_t)N * s * s);
      c.MdenseT = c.alloc<double>((size_t)N * s * s);
      for (int w = 0; w < N; ++w) {
        WF_CUDA(memcpy_sync(c, c.Mdense + (size_t)w * s * s, M.data(), M.size() * 8, cudaMemcpyHostToDevice));
        WF_CUDA(memcpy_sync(c, c.MdenseT + (size_t)w * s * s, M.data(), M.size() * 8, cudaMemcpyHostToDevice));
      }
    }
  } else if (c.model == WF4DVAR_M_HEAT_EXPLICIT) {
    WF_REQUIRE(p.heat_r > 0 && p.heat_r <= 0.5, WF4DVAR_EINVAL,
               "HEAT_EXPLICIT needs 0 < heat_r <= 1/2 (P:L1132 stability)");
    WF_REQUIRE(p.heat_nsteps >= 1 && p.heat_nsteps <= 8, WF4DVAR_EINVAL,
               "HEAT_EXPLICIT needs 1 <= heat_nsteps <= 8");
    WF_REQUIRE(s >= 3, WF4DVAR_EINVAL, "HEAT_EXPLICIT needs s >= 3");
    c.heat_r = p.heat_r;
    c.heat_nsteps = p.heat_nsteps;
  } else if (c.model == WF4DVAR_M_DENSE) {
    WF_REQUIRE(p.M_dense != nullptr, WF4DVAR_EINVAL, "M_dense is NULL");
    c.Mdense = c.alloc<double>((size_t)N * s * s);
    c.MdenseT = c.alloc<double>((size_t)N * s * s);
    std::vector<double> Tm((size_t)s * s);
    for (int w = 0; w < N; ++w) {
      const double *Mw = p.M_dense + (size_t)w * s * s;
      for (int i = 0; i < s; ++i)
        for (int j = 0; j < s; ++j) Tm[(size_t)j * s + i] = Mw[(size_t)i * s + j];
      WF_CUDA(memcpy_sync(c, c.Mdense + (size_t)w * s * s, Mw, (size_t)s * s * 8, cudaMemcpyHostToDevice));
      WF_CUDA(memcpy_sync(c, c.MdenseT + (size_t)w * s * s, Tm.data(), Tm.size() * 8, cudaMemcpyHostToDevice));
    }
  } else if (c.model == WF4DVAR_M_L96) {
    WF_REQUIRE(p.l96_traj != nullptr || N == 0, WF4DVAR_EINVAL, "l96_traj is NULL");
    WF_REQUIRE(s >= 4 && s <= 64, WF4DVAR_EINVAL, "L96 kernel supports 4 <= s <= 64");
    WF_REQUIRE(p.l96_nsub >= 1 && p.l96_nsub <= 8, WF4DVAR_EINVAL, "L96 needs 1 <= nsub <= 8");
    WF_REQUIRE(p.l96_dt > 0, WF4DVAR_EINVAL, "L96 dt must be > 0");
    c.l96_F = p.l96_F; c.l96_dt = p.l96_dt; c.l96_nsub = p.l96_nsub;
    c.traj = c.alloc<double>((size_t)std::max(N, 1) * s * c.m);
    c.l96_sub = c.alloc<double>((size_t)std::max(N, 1) * c.l96_nsub * s * c.m);
    if (N > 0) {
      WF_CUDA(memcpy_sync(c, c.traj, p.l96_traj, (size_t)N * s * c.m * 8, cudaMemcpyHostToDevice));
      l96_substates(c);
    }
  } else {
    throw Error{WF4DVAR_EINVAL, "unknown model kind"};
  }
}

}  // namespace wf
