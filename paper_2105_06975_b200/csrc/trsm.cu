// Cholesky-factor triangular solves for D_hat^{-1} and R_hat^{-1} (P:L647-651,
// "apply ... using the (incomplete) Cholesky factors").
//
// One CTA owns a panel of NB right-hand-side columns and walks the 64-row
// tiles of the triangle in dependency order (down for G, up for U = G^T):
//   T_i = X_i - sum_{j<i} G_ij Y_j      DMMA tile GEMM (dmma.cuh pipeline),
//   Y_i = G_ii^{-1} T_i                 exact substitution in registers, one
//                                       warp per column group, the diagonal
//                                       tile staged transposed in shared memory.
// The off-diagonal work is a true FP64 contraction on the tensor path; the
// diagonal solve is plain forward/backward substitution (backward stable).
// For R_block the factor is block diagonal: tiles left of the row's block are
// known zeros and are skipped (blk > 0).
#include <type_traits>

#include "dmma.cuh"
#include "internal.h"

namespace wf {

constexpr int TB = 64;  // rows per triangle tile

template <int NB>
using TrsmCfg = typename std::conditional<NB == 8, TileCfg<64, 8, 16, 16, 8, 3>,
                                          TileCfg<64, NB, 16, 32, NB / 2, 3>>::type;

struct TrsmLaunch {
  TrsmProb p[2];
  int panels0;
};

template <int NB, bool UPPER, bool V16>
__global__ void __launch_bounds__(128) k_trsm(const TrsmLaunch L) {
  using C = TrsmCfg<NB>;
  extern __shared__ __align__(16) double smem[];
  double *sPipe = smem;                        // C::SMEM_DOUBLES
  double *sT = smem + C::SMEM_DOUBLES;         // [64][NB+1]
  double *sG = sT + TB * (NB + 1);             // [64][65] diagonal tile, transposed

  int panel = blockIdx.x, gi = 0;
  if (panel >= L.panels0) { panel -= L.panels0; gi = 1; }
  const TrsmProb &P = L.p[gi];
  const int c0 = panel * NB;
  const int n = P.n;
  const int ntile = (n + TB - 1) / TB;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / C::WARPS_N, wn = warp % C::WARPS_N;
  const int g = lane >> 2, t = lane & 3;
  const double *__restrict__ G = P.G;
  double *Y = P.Y;
  const double *X = P.X;
  const int ncols = P.ncols;

  for (int it = 0; it < ntile; ++it) {
    const int ti = UPPER ? (ntile - 1 - it) : it;
    const int r0 = ti * TB, r1 = min(n, r0 + TB), nr = r1 - r0;
    // ---- off-diagonal update: acc = G[r0:r1, K] * Y[K, panel]
    int kbeg, kend;
    if (!UPPER) {
      kbeg = P.blk > 0 ? (r0 / P.blk) * P.blk : 0;
      kbeg = (kbeg / 16) * 16;
      kend = r0;
    } else {
      kbeg = r1;
      kend = P.blk > 0 ? min(n, ((r1 - 1) / P.blk + 1) * P.blk) : n;
    }
    double acc[C::FM][C::FN][2];
#pragma unroll
    for (int i = 0; i < C::FM; ++i)
#pragma unroll
      for (int j = 0; j < C::FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    if (kend > kbeg)
      tile_mainloop<C, V16>(sPipe, acc, G + (int64_t)r0 * P.ldg, P.ldg, Y + c0, P.ldy, 0, 0, kbeg,
                            kend, nr, ncols - c0);
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
    // ---- diagonal tile, transposed: sG[c][r] = G[r0 + r][r0 + c]; identity padding
    for (int e = tid; e < TB * TB; e += 128) {
      int r = e / TB, cc = e % TB;
      double v;
      if (r < nr && cc < nr) v = G[(int64_t)(r0 + r) * P.ldg + r0 + cc];
      else v = (r == cc) ? 1.0 : 0.0;
      sG[cc * (TB + 1) + r] = v;
    }
    __syncthreads();
    // ---- substitution: warp w solves columns w, w+4, ...; lane holds rows lane, lane+32
    constexpr int CPW = NB / 4;
    double v0[CPW], v1[CPW];
#pragma unroll
    for (int q = 0; q < CPW; ++q) {
      int cc = warp + 4 * q;
      v0[q] = sT[lane * (NB + 1) + cc];
      v1[q] = sT[(lane + 32) * (NB + 1) + cc];
    }
    if (!UPPER) {
      for (int r = 0; r < TB; ++r) {
        const double diag = sG[r * (TB + 1) + r];
        const double g0 = sG[r * (TB + 1) + lane];        // G[lane][r]
        const double g1 = sG[r * (TB + 1) + lane + 32];   // G[lane+32][r]
        const int src = r & 31;
#pragma unroll
        for (int q = 0; q < CPW; ++q) {
          double mine = (r < 32) ? v0[q] : v1[q];
          double yr = __shfl_sync(0xffffffffu, mine, src) / diag;
          if (lane == src) { if (r < 32) v0[q] = yr; else v1[q] = yr; }
          if (lane > r) v0[q] -= g0 * yr;
          if (lane + 32 > r) v1[q] -= g1 * yr;
        }
      }
    } else {
      for (int r = TB - 1; r >= 0; --r) {
        const double diag = sG[r * (TB + 1) + r];
        const double g0 = sG[r * (TB + 1) + lane];        // U[lane][r]
        const double g1 = sG[r * (TB + 1) + lane + 32];
        const int src = r & 31;
#pragma unroll
        for (int q = 0; q < CPW; ++q) {
          double mine = (r < 32) ? v0[q] : v1[q];
          double yr = __shfl_sync(0xffffffffu, mine, src) / diag;
          if (lane == src) { if (r < 32) v0[q] = yr; else v1[q] = yr; }
          if (lane < r) v0[q] -= g0 * yr;
          if (lane + 32 < r) v1[q] -= g1 * yr;
        }
      }
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
    __threadfence();
    __syncthreads();
  }
}

template <int NB, bool UPPER>
static void run(Ctx &c, const TrsmLaunch &L, int panels, bool v16) {
  using C = TrsmCfg<NB>;
  size_t smem = (C::SMEM_DOUBLES + TB * (NB + 1) + TB * (TB + 1)) * sizeof(double);
  auto kern = v16 ? k_trsm<NB, UPPER, true> : k_trsm<NB, UPPER, false>;
  static bool attr[2] = {false, false};
  if (!attr[v16]) {
    WF_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr[v16] = true;
  }
  kern<<<panels, 128, smem, c.st>>>(L);
  WF_CUDA(cudaGetLastError());
}

void launch_trsm(Ctx &c, const TrsmProb *probs, int nprob, bool upper) {
  TrsmLaunch L{};
  int total_cols = 0, valid = 0;
  double flops = 0, bytes = 0;
  bool v16 = true;
  for (int i = 0; i < nprob; ++i) {
    if (probs[i].ncols <= 0 || probs[i].n <= 0) continue;
    L.p[valid++] = probs[i];
    total_cols += probs[i].ncols;
    double tri = (double)probs[i].n * probs[i].n;
    if (probs[i].blk > 0) tri = (double)probs[i].n * probs[i].blk;
    flops += tri * probs[i].ncols;   // n^2 * ncols multiply-adds / 2 * 2
    bytes += 8.0 * (tri / 2 + 2.0 * probs[i].n * probs[i].ncols);
    v16 = v16 && ((uintptr_t)probs[i].G % 16 == 0) && ((uintptr_t)probs[i].Y % 16 == 0) &&
          (probs[i].ldg % 2 == 0) && (probs[i].ldy % 2 == 0);
  }
  if (!valid) return;
  // panel width: as wide as possible while still giving >= ~1 CTA per SM
  int NB = 64;
  if ((total_cols + 63) / 64 < 148) NB = 32;
  if ((total_cols + 31) / 32 < 148) NB = 16;
  if ((total_cols + 15) / 16 < 148) NB = 8;
  int panels = 0;
  for (int i = 0; i < valid; ++i) {
    int pi = (L.p[i].ncols + NB - 1) / NB;
    if (i == 0) L.panels0 = pi;
    panels += pi;
  }
  if (valid == 1) L.panels0 = panels;
  LaunchScope ls(c, K_TRSM, flops, bytes);
  switch (NB) {
    case 64: upper ? run<64, true>(c, L, panels, v16) : run<64, false>(c, L, panels, v16); break;
    case 32: upper ? run<32, true>(c, L, panels, v16) : run<32, false>(c, L, panels, v16); break;
    case 16: upper ? run<16, true>(c, L, panels, v16) : run<16, false>(c, L, panels, v16); break;
    default: upper ? run<8, true>(c, L, panels, v16) : run<8, false>(c, L, panels, v16); break;
  }
  c.launches++;
}

}  // namespace wf
