// Lorenz-96 tangent-linear model M_w and its adjoint M_w^T (BJ.c2), matrix-free.
//
// dx_i/dt = (x_{i+1} - x_{i-2}) x_{i-1} - x_i + F, periodic,
// RK4; BJ.c2: dt = 0.025, 5 RK4 substeps per window.  M_w is the exact derivative
// of the discrete map (nsub RK4 steps) along the trajectory that starts at
// traj[w-1] ("exact derivative of the discrete RK4 map"); the
// nonlinear stages are recomputed on the fly (no M_w is ever stored: 40x40x50x1024
// doubles would be 655 MB per pass).
//
//   J(x) u : (J u)_i   = (u_{i+1} - u_{i-2}) x_{i-1} + (x_{i+1} - x_{i-2}) u_{i-1} - u_i
//   J^T l  : (J^T l)_j = x_{j-2} l_{j-1} - x_{j+1} l_{j+2} + (x_{j+2} - x_{j-1}) l_{j+1} - l_j
//   RK4 tangent:  d1 = J(x1) v, d2 = J(x2)(v + h/2 d1), d3 = J(x3)(v + h/2 d2),
//                 d4 = J(x4)(v + h d3),  v' = v + h/6 (d1 + 2 d2 + 2 d3 + d4)
//   adjoint (reverse of the above, stages recomputed from the substep start state).
//
// Layout: one CTA = 32 problems (RHS columns, the fastest index -> coalesced) x
// 8 thread rows; thread row ty owns state indices ty, ty+8, ...; periodic
// neighbours are exchanged through shared memory.  FP64 ALU bound.
// The nonlinear stages are recomputed on the fly; only the RK4 substep START states of
// every trajectory window are kept (c.l96_sub, nsub x the trajectory: 82 MB for
// BJ.c2), so the adjoint sweeps its substeps backwards without re-integrating them.
#include "internal.h"

namespace wf {

template <int IPT>
struct L96Thread {
  static constexpr int S_MAX = 8 * IPT;
};

struct L96Args {
  double *out;
  const double *base, *in, *traj, *sub, *add2, *halo;
  const int *row_map;
  double sign, F, dt, h6, h3;   // h6 = dt / 6, h3 = dt / 3 (host-side: no device divisions)
  int s, W, m, nsub, w_first, w_step, nw, dir;
  int w0, WG;   // global index of local window 0; global window count
  int nw0, w_first1;   // blockIdx.y >= nw0: window w_first1 + (blockIdx.y - nw0)
};

// ---- contiguous ownership (s == 8 IPT): lane ty of a problem's 8-lane group owns
// indices [ty IPT, ty IPT + IPT); the periodic neighbours it lacks (two on each side)
// come from the ring neighbours by register shuffles -- no shared memory, no barrier
template <int IPT>
struct Halo2 { double l2, l1, r1, r2; };   // x_{i0-2}, x_{i0-1}, x_{i0+IPT}, x_{i0+IPT+1}

template <int IPT, int LPP = 8>
__device__ __forceinline__ Halo2<IPT> halo2(const double (&x)[IPT], int ty) {
  const int lft = (ty + LPP - 1) % LPP, rgt = (ty + 1) % LPP;
  Halo2<IPT> h;
  h.l2 = __shfl_sync(0xffffffffu, x[IPT - 2], lft, LPP);
  h.l1 = __shfl_sync(0xffffffffu, x[IPT - 1], lft, LPP);
  h.r1 = __shfl_sync(0xffffffffu, x[0], rgt, LPP);
  h.r2 = __shfl_sync(0xffffffffu, x[1], rgt, LPP);
  return h;
}

template <int IPT>
__device__ __forceinline__ double at(const double (&x)[IPT], const Halo2<IPT> &h, int j) {
  // j in [-2, IPT + 1], compile-time after unrolling
  return j == -2 ? h.l2 : j == -1 ? h.l1 : j == IPT ? h.r1 : j == IPT + 1 ? h.r2 : x[j];
}

template <int IPT, int LPP = 8>
__device__ __forceinline__ void l96_rhs_sh(const double (&x)[IPT], double (&f)[IPT], int ty,
                                           double F) {
  const Halo2<IPT> h = halo2<IPT, LPP>(x, ty);
#pragma unroll
  for (int k = 0; k < IPT; ++k)
    f[k] = (at<IPT>(x, h, k + 1) - at<IPT>(x, h, k - 2)) * at<IPT>(x, h, k - 1) - x[k] + F;
}

template <int IPT, int LPP = 8>
__device__ __forceinline__ void l96_jac_sh(const double (&x)[IPT], const double (&u)[IPT],
                                           double (&Ju)[IPT], int ty, bool transpose) {
  const Halo2<IPT> hx = halo2<IPT, LPP>(x, ty), hu = halo2<IPT, LPP>(u, ty);
#pragma unroll
  for (int k = 0; k < IPT; ++k) {
    if (!transpose) {
      Ju[k] = (at<IPT>(u, hu, k + 1) - at<IPT>(u, hu, k - 2)) * at<IPT>(x, hx, k - 1) +
              (at<IPT>(x, hx, k + 1) - at<IPT>(x, hx, k - 2)) * at<IPT>(u, hu, k - 1) - u[k];
    } else {
      Ju[k] = at<IPT>(x, hx, k - 2) * at<IPT>(u, hu, k - 1) -
              at<IPT>(x, hx, k + 1) * at<IPT>(u, hu, k + 2) +
              (at<IPT>(x, hx, k + 2) - at<IPT>(x, hx, k - 1)) * at<IPT>(u, hu, k + 1) - u[k];
    }
  }
}

template <int IPT>
__device__ __forceinline__ void l96_rhs(const double (&x)[IPT], double (&f)[IPT], double *bx,
                                        int s, int ty, int lane, double F) {
  // bx: [S_MAX][32] exchange buffer
#pragma unroll
  for (int k = 0; k < IPT; ++k) {
    int i = ty + 8 * k;
    if (i < s) bx[i * 4 + lane] = x[k];
  }
  __syncwarp();
#pragma unroll
  for (int k = 0; k < IPT; ++k) {
    int i = ty + 8 * k;
    if (i < s) {
      int ip = i + 1 == s ? 0 : i + 1, im1 = i == 0 ? s - 1 : i - 1, im2 = i >= 2 ? i - 2 : i - 2 + s;
      f[k] = (bx[ip * 4 + lane] - bx[im2 * 4 + lane]) * bx[im1 * 4 + lane] - x[k] + F;
    }
  }
  __syncwarp();
}

// Ju = J(x) u, with x already resident in bx (written by l96_rhs of the same stage is
// not reused: x is re-exchanged together with u for clarity)
template <int IPT>
__device__ __forceinline__ void l96_jac(const double (&x)[IPT], const double (&u)[IPT],
                                        double (&Ju)[IPT], double *bx, double *bu, int s, int ty,
                                        int lane, bool transpose) {
#pragma unroll
  for (int k = 0; k < IPT; ++k) {
    int i = ty + 8 * k;
    if (i < s) { bx[i * 4 + lane] = x[k]; bu[i * 4 + lane] = u[k]; }
  }
  __syncwarp();
#pragma unroll
  for (int k = 0; k < IPT; ++k) {
    int i = ty + 8 * k;
    if (i < s) {
      int ip1 = i + 1 == s ? 0 : i + 1, ip2 = i + 2 >= s ? i + 2 - s : i + 2;
      int im1 = i == 0 ? s - 1 : i - 1, im2 = i >= 2 ? i - 2 : i - 2 + s;
      if (!transpose) {
        Ju[k] = (bu[ip1 * 4 + lane] - bu[im2 * 4 + lane]) * bx[im1 * 4 + lane] +
                (bx[ip1 * 4 + lane] - bx[im2 * 4 + lane]) * bu[im1 * 4 + lane] - u[k];
      } else {
        Ju[k] = bx[im2 * 4 + lane] * bu[im1 * 4 + lane] - bx[ip1 * 4 + lane] * bu[ip2 * 4 + lane] +
                (bx[ip2 * 4 + lane] - bx[im1 * 4 + lane]) * bu[ip1 * 4 + lane] - u[k];
      }
    }
  }
  __syncwarp();
}

template <int IPT, bool SH, int LPP = 8>
__device__ __forceinline__ void rhs_any(const double (&x)[IPT], double (&f)[IPT], double *bx,
                                        int s, int ty, int lane, double F) {
  if constexpr (SH) l96_rhs_sh<IPT, LPP>(x, f, ty, F);
  else l96_rhs<IPT>(x, f, bx, s, ty, lane, F);
}

template <int IPT, bool SH, int LPP = 8>
__device__ __forceinline__ void jac_any(const double (&x)[IPT], const double (&u)[IPT],
                                        double (&Ju)[IPT], double *bx, double *bu, int s, int ty,
                                        int lane, bool transpose) {
  if constexpr (SH) l96_jac_sh<IPT, LPP>(x, u, Ju, ty, transpose);
  else l96_jac<IPT>(x, u, Ju, bx, bu, s, ty, lane, transpose);
}

// nonlinear stage states of one RK4 step from x (x1 = x)
template <int IPT, bool SH>
__device__ __forceinline__ void rk4_stages(const double (&x)[IPT], double (&x2)[IPT],
                                           double (&x3)[IPT], double (&x4)[IPT],
                                           double (&xn)[IPT], double *bx, int s, int ty, int lane,
                                           double F, double h) {
  double k1[IPT], k2[IPT], k3[IPT], k4[IPT];
  rhs_any<IPT, SH>(x, k1, bx, s, ty, lane, F);
#pragma unroll
  for (int k = 0; k < IPT; ++k) x2[k] = x[k] + 0.5 * h * k1[k];
  rhs_any<IPT, SH>(x2, k2, bx, s, ty, lane, F);
#pragma unroll
  for (int k = 0; k < IPT; ++k) x3[k] = x[k] + 0.5 * h * k2[k];
  rhs_any<IPT, SH>(x3, k3, bx, s, ty, lane, F);
#pragma unroll
  for (int k = 0; k < IPT; ++k) x4[k] = x[k] + h * k3[k];
  rhs_any<IPT, SH>(x4, k4, bx, s, ty, lane, F);
#pragma unroll
  for (int k = 0; k < IPT; ++k) xn[k] = x[k] + (h / 6.0) * (k1[k] + 2.0 * k2[k] + 2.0 * k3[k] + k4[k]);
}

// the three inner stage states x2, x3, x4 of one RK4 step from x1 (what the adjoint needs)
template <int IPT, bool SH, int LPP = 8>
__device__ __forceinline__ void rk4_inner_states(const double (&x)[IPT], double (&x2)[IPT],
                                                 double (&x3)[IPT], double (&x4)[IPT], double *bx,
                                                 int s, int ty, int lane, double F, double h) {
  double kk[IPT];
  rhs_any<IPT, SH, LPP>(x, kk, bx, s, ty, lane, F);
#pragma unroll
  for (int k = 0; k < IPT; ++k) x2[k] = x[k] + 0.5 * h * kk[k];
  rhs_any<IPT, SH, LPP>(x2, kk, bx, s, ty, lane, F);
#pragma unroll
  for (int k = 0; k < IPT; ++k) x3[k] = x[k] + 0.5 * h * kk[k];
  rhs_any<IPT, SH, LPP>(x3, kk, bx, s, ty, lane, F);
#pragma unroll
  for (int k = 0; k < IPT; ++k) x4[k] = x[k] + h * kk[k];
}

// one stage of the forward tangent fused with its nonlinear stage: f = f(xs) and
// d = J(xs) us from ONE neighbour exchange of xs (round 1 exchanged every stage state
// twice: once for the tendency, once for the Jacobian product)
template <int IPT, int LPP = 8>
__device__ __forceinline__ void l96_fused_sh(const double (&x)[IPT], const double (&u)[IPT],
                                             double (&f)[IPT], double (&Ju)[IPT], int ty, double F) {
  const Halo2<IPT> hx = halo2<IPT, LPP>(x, ty), hu = halo2<IPT, LPP>(u, ty);
#pragma unroll
  for (int k = 0; k < IPT; ++k) {
    const double xm2 = at<IPT>(x, hx, k - 2), xm1 = at<IPT>(x, hx, k - 1), xp1 = at<IPT>(x, hx, k + 1);
    f[k] = (xp1 - xm2) * xm1 - x[k] + F;
    Ju[k] = (at<IPT>(u, hu, k + 1) - at<IPT>(u, hu, k - 2)) * xm1 + (xp1 - xm2) * at<IPT>(u, hu, k - 1) - u[k];
  }
}

template <int IPT>
__device__ __forceinline__ void l96_fused(const double (&x)[IPT], const double (&u)[IPT],
                                          double (&f)[IPT], double (&Ju)[IPT], double *bx, double *bu,
                                          int s, int ty, int lane, double F) {
#pragma unroll
  for (int k = 0; k < IPT; ++k) {
    int i = ty + 8 * k;
    if (i < s) { bx[i * 4 + lane] = x[k]; bu[i * 4 + lane] = u[k]; }
  }
  __syncwarp();
#pragma unroll
  for (int k = 0; k < IPT; ++k) {
    int i = ty + 8 * k;
    if (i < s) {
      int ip1 = i + 1 == s ? 0 : i + 1, im1 = i == 0 ? s - 1 : i - 1, im2 = i >= 2 ? i - 2 : i - 2 + s;
      const double xm2 = bx[im2 * 4 + lane], xm1 = bx[im1 * 4 + lane], xp1 = bx[ip1 * 4 + lane];
      f[k] = (xp1 - xm2) * xm1 - x[k] + F;
      Ju[k] = (bu[ip1 * 4 + lane] - bu[im2 * 4 + lane]) * xm1 + (xp1 - xm2) * bu[im1 * 4 + lane] - u[k];
    }
  }
  __syncwarp();
}

template <int IPT, bool SH, int LPP = 8>
__device__ __forceinline__ void fused_any(const double (&x)[IPT], const double (&u)[IPT],
                                          double (&f)[IPT], double (&Ju)[IPT], double *bx, double *bu,
                                          int s, int ty, int lane, double F) {
  if constexpr (SH) l96_fused_sh<IPT, LPP>(x, u, f, Ju, ty, F);
  else l96_fused<IPT>(x, u, f, Ju, bx, bu, s, ty, lane, F);
}

// The adjoint reads the substep start states of its window from c.l96_sub (written once
// per trajectory by k_l96_substates, round 2) instead of re-integrating them from the
// window start in every apply (round 1: nsub - 1 extra nonlinear RK4 steps per
// adjoint window and a [NSUB_MAX IPT][256] shared-memory stash); forward and adjoint
// are separate instantiations so each gets its own register allocation, and the
// IPT = 5 (s <= 40) variants are held to 2 CTAs per SM (IPT = 8 would spill).
template <int IPT, bool SH, bool ADJ, int LPP = 8>
#ifndef L96_MINB_F
#define L96_MINB_F 3   // r02w (round-1 kernel, configs[2] step): 2 CTAs per SM (96 registers)
                       // 0.519 ms, 3 (80 registers, 48-byte spill) 0.522, 4 (64, 232-byte
                       // spill) 0.595; the fused-stage kernel (r02ak) fits 3 in 80, no spill
#endif
#ifndef L96_MINB_A
#define L96_MINB_A 2
#endif
#ifndef L96_ADJ_STASH
#define L96_ADJ_STASH 0
#endif
// four lanes per problem (s = 40: 10 states per thread, 128-thread CTAs): half the
// neighbour shuffles per flop of the 8-lane mapping, twice the independent chains per
// thread, fewer warps (r02am experiment, WF4DVAR_L96_LPP=4)
#ifndef L96_MINB_F4
#define L96_MINB_F4 3
#endif
#ifndef L96_MINB_A4
#define L96_MINB_A4 2
#endif
__global__ void __launch_bounds__(LPP == 8 ? 256 : 128,
                                  LPP == 4 ? (ADJ ? L96_MINB_A4 : L96_MINB_F4)
                                  : IPT <= 5 ? (ADJ ? L96_MINB_A : SH ? L96_MINB_F : 2) : 1)
k_l96_step(const L96Args a) {
  extern __shared__ double stash[];   // adjoint with L96_ADJ_STASH: [2 IPT][256]
  __shared__ double bx[SH ? 1 : L96Thread<IPT>::S_MAX * 32];
  __shared__ double bu[SH ? 1 : L96Thread<IPT>::S_MAX * 32];
  // 4 problems per warp, 8 lanes per problem (lane = 8 p + ty): the periodic
  // neighbour exchange stays inside the warp (warp-private shared memory, __syncwarp
  // instead of __syncthreads; layout [i][4] -> every access is 32 consecutive doubles)
  constexpr int NT = LPP == 8 ? 256 : 128, PPW = 32 / LPP;   // 32 problems per CTA
  const int tid = threadIdx.y * 32 + threadIdx.x;
  const int wp = tid >> 5, lw = tid & 31;
  const int lane = lw / LPP, ty = lw % LPP;    // lane = problem within the warp
  const int r = blockIdx.x * 32 + wp * PPW + lane;
  double *const bxw = bx + wp * (L96Thread<IPT>::S_MAX * 4);
  double *const buw = bu + wp * (L96Thread<IPT>::S_MAX * 4);
  const int t = blockIdx.y;
  const int w = t < a.nw0 ? a.w_first + t * a.w_step : a.w_first1 + (t - a.nw0);
  const int ws = w + a.dir;                       // local source window
  const bool has = a.w0 + ws >= 0 && a.w0 + ws < a.WG;   // global source exists
  const bool from_halo = ws < 0 || ws >= a.W;      // owned by the neighbour rank
  const bool live = r < a.m;
  const int64_t ld = (int64_t)a.W * a.m;
  const int s = a.s;
  const double h = a.dt, h6 = a.h6, h3 = a.h3;
  double v[IPT];
  if (has) {
    // trajectory start state of the window pair: M_w uses traj[w-1], M_{w+1}^T uses traj[w]
    const int tw = a.w0 + (a.dir < 0 ? w - 1 : w);
#pragma unroll
    for (int k = 0; k < IPT; ++k) {
      int i = SH ? ty * IPT + k : ty + 8 * k;
      v[k] = (live && i < s) ? (from_halo ? a.halo[(int64_t)i * a.m + r]
                                          : a.in[i * ld + (int64_t)ws * a.m + r])
                             : 0.0;
    }
    if constexpr (!ADJ) {
      // forward tangent: nsub RK4 steps, each stage's tendency and Jacobian product
      // from one exchange of the stage state
      double x[IPT];
#pragma unroll
      for (int k = 0; k < IPT; ++k) {
        int i = SH ? ty * IPT + k : ty + 8 * k;
        x[k] = (live && i < s) ? a.traj[((int64_t)tw * s + i) * a.m + r] : 0.0;
      }
      for (int st = 0; st < a.nsub; ++st) {
        double xs[IPT], us[IPT], ks[IPT], ds[IPT], f[IPT], d[IPT];
        fused_any<IPT, SH, LPP>(x, v, f, d, bxw, buw, s, ty, lane, a.F);
#pragma unroll
        for (int k = 0; k < IPT; ++k) {
          ks[k] = f[k]; ds[k] = d[k];
          xs[k] = x[k] + 0.5 * h * f[k]; us[k] = v[k] + 0.5 * h * d[k];
        }
        fused_any<IPT, SH, LPP>(xs, us, f, d, bxw, buw, s, ty, lane, a.F);
#pragma unroll
        for (int k = 0; k < IPT; ++k) {
          ks[k] += 2.0 * f[k]; ds[k] += 2.0 * d[k];
          xs[k] = x[k] + 0.5 * h * f[k]; us[k] = v[k] + 0.5 * h * d[k];
        }
        fused_any<IPT, SH, LPP>(xs, us, f, d, bxw, buw, s, ty, lane, a.F);
#pragma unroll
        for (int k = 0; k < IPT; ++k) {
          ks[k] += 2.0 * f[k]; ds[k] += 2.0 * d[k];
          xs[k] = x[k] + h * f[k]; us[k] = v[k] + h * d[k];
        }
        fused_any<IPT, SH, LPP>(xs, us, f, d, bxw, buw, s, ty, lane, a.F);
#pragma unroll
        for (int k = 0; k < IPT; ++k) {
          x[k] = x[k] + h6 * (ks[k] + f[k]);
          v[k] = v[k] + h6 * (ds[k] + d[k]);
        }
      }
    } else {
      // adjoint: sweep the substeps backwards from their stored start states
      const double *sub = a.sub + (int64_t)tw * a.nsub * s * a.m;
      // the next (earlier) substep's start state is loaded one substep ahead, so its
      // global-memory latency hides under the current substep's arithmetic
      double xnext[IPT];
#pragma unroll
      for (int k = 0; k < IPT; ++k) {
        int i = SH ? ty * IPT + k : ty + 8 * k;
        xnext[k] = (live && i < s) ? sub[((int64_t)(a.nsub - 1) * s + i) * a.m + r] : 0.0;
      }
      for (int st = a.nsub - 1; st >= 0; --st) {
        double x1[IPT], xt[IPT], lu[IPT], ld1[IPT], ld2[IPT], ld3[IPT];
#pragma unroll
        for (int k = 0; k < IPT; ++k) {
          int i = SH ? ty * IPT + k : ty + 8 * k;
          x1[k] = xnext[k];
          if (st > 0) xnext[k] = (live && i < s) ? sub[((int64_t)(st - 1) * s + i) * a.m + r] : 0.0;
        }
#if L96_ADJ_STASH
        // inner stage states x2..x4 parked in this thread's shared-memory slots
        // ([3 IPT][256], consecutive threads -> consecutive words) instead of registers
        {
          double kk[IPT];
          rhs_any<IPT, SH, LPP>(x1, kk, bxw, s, ty, lane, a.F);
#pragma unroll
          for (int k = 0; k < IPT; ++k) { xt[k] = x1[k] + 0.5 * h * kk[k]; stash[k * NT + tid] = xt[k]; }
          rhs_any<IPT, SH, LPP>(xt, kk, bxw, s, ty, lane, a.F);
#pragma unroll
          for (int k = 0; k < IPT; ++k) { xt[k] = x1[k] + 0.5 * h * kk[k]; stash[(IPT + k) * NT + tid] = xt[k]; }
          rhs_any<IPT, SH, LPP>(xt, kk, bxw, s, ty, lane, a.F);
#pragma unroll
          for (int k = 0; k < IPT; ++k) xt[k] = x1[k] + h * kk[k];   // x4 stays in xt
        }
#define WF_STAGE(j) _Pragma("unroll") for (int k = 0; k < IPT; ++k) xt[k] = stash[((j) * IPT + k) * NT + tid];
#else
        double x2[IPT], x3[IPT];
        rk4_inner_states<IPT, SH, LPP>(x1, x2, x3, xt, bxw, s, ty, lane, a.F, h);
#endif
        // lambda_d4 = h/6 l ; lambda_u4 = J4^T lambda_d4
        double lv[IPT], tmp[IPT];
#pragma unroll
        for (int k = 0; k < IPT; ++k) { lv[k] = v[k]; tmp[k] = h6 * v[k]; }
        jac_any<IPT, SH, LPP>(xt, tmp, lu, bxw, buw, s, ty, lane, true);
#pragma unroll
        for (int k = 0; k < IPT; ++k) { lv[k] += lu[k]; ld3[k] = h3 * v[k] + h * lu[k]; }
#if L96_ADJ_STASH
        WF_STAGE(1)
        jac_any<IPT, SH, LPP>(xt, ld3, lu, bxw, buw, s, ty, lane, true);
#else
        jac_any<IPT, SH, LPP>(x3, ld3, lu, bxw, buw, s, ty, lane, true);
#endif
#pragma unroll
        for (int k = 0; k < IPT; ++k) { lv[k] += lu[k]; ld2[k] = h3 * v[k] + 0.5 * h * lu[k]; }
#if L96_ADJ_STASH
        WF_STAGE(0)
        jac_any<IPT, SH, LPP>(xt, ld2, lu, bxw, buw, s, ty, lane, true);
#undef WF_STAGE
#else
        jac_any<IPT, SH, LPP>(x2, ld2, lu, bxw, buw, s, ty, lane, true);
#endif
#pragma unroll
        for (int k = 0; k < IPT; ++k) { lv[k] += lu[k]; ld1[k] = h6 * v[k] + 0.5 * h * lu[k]; }
        jac_any<IPT, SH, LPP>(x1, ld1, lu, bxw, buw, s, ty, lane, true);
#pragma unroll
        for (int k = 0; k < IPT; ++k) v[k] = lv[k] + lu[k];
      }
    }
  }
  if (!live) return;
  // epilogue: every load (base, add2) issued before the first store -- out may alias
  // base, so the compiler cannot hoist the loads itself, and the load -> FMA -> store
  // chain per element was the kernel's top stall (ncu r02an: 20% of the samples)
  double bv[IPT], av[IPT];
#pragma unroll
  for (int k = 0; k < IPT; ++k) {
    const int i = SH ? ty * IPT + k : ty + 8 * k;
    bv[k] = 0.0; av[k] = 0.0;
    if (i < s) {
      const int64_t o = i * ld + (int64_t)w * a.m + r;
      bv[k] = a.base[o];
      if (a.add2) {
        const int j = a.row_map[i];
        if (j >= 0) av[k] = a.add2[(int64_t)j * ld + (int64_t)w * a.m + r];
      }
    }
  }
#pragma unroll
  for (int k = 0; k < IPT; ++k) {
    const int i = SH ? ty * IPT + k : ty + 8 * k;
    if (i < s) {
      double val = bv[k];
      if (has) val = fma(a.sign, v[k], val);
      if (a.add2) val += av[k];
      a.out[i * ld + (int64_t)w * a.m + r] = val;
    }
  }
}

// substep start states along the trajectory: sub[g][st] = state after st nonlinear RK4
// substeps from traj[g] (st = 0: traj[g] itself), for the trajectory windows
// g in [g_lo, g_lo + gridDim.y) -- the ones this rank's adjoint windows start from
template <int IPT, bool SH>
__global__ void __launch_bounds__(256) k_l96_substates(double *sub, const double *traj, double F,
                                                       double h, int s, int m, int nsub, int g_lo) {
  __shared__ double bx[SH ? 1 : L96Thread<IPT>::S_MAX * 32];
  const int tid = threadIdx.y * 32 + threadIdx.x;
  const int wp = tid >> 5, lw = tid & 31;
  const int lane = lw >> 3, ty = lw & 7;
  const int r = blockIdx.x * 32 + wp * 4 + lane;
  double *const bxw = bx + wp * (L96Thread<IPT>::S_MAX * 4);
  const int g = g_lo + blockIdx.y;
  const bool live = r < m;
  double xs[IPT];
#pragma unroll
  for (int k = 0; k < IPT; ++k) {
    const int i = SH ? ty * IPT + k : ty + 8 * k;
    xs[k] = (live && i < s) ? traj[((int64_t)g * s + i) * m + r] : 0.0;
  }
  double *o = sub + (int64_t)g * nsub * s * m;
  for (int st = 0; st < nsub; ++st) {
#pragma unroll
    for (int k = 0; k < IPT; ++k) {
      const int i = SH ? ty * IPT + k : ty + 8 * k;
      if (live && i < s) o[((int64_t)st * s + i) * m + r] = xs[k];
    }
    if (st + 1 == nsub) break;
    double x2[IPT], x3[IPT], x4[IPT], xn[IPT];
    rk4_stages<IPT, SH>(xs, x2, x3, x4, xn, bxw, s, ty, lane, F, h);
#pragma unroll
    for (int k = 0; k < IPT; ++k) xs[k] = xn[k];
  }
}

void l96_substates(Ctx &c) {
  // adjoint windows w read traj[w0 + w] for local w in [0, W) (M_{w+1}^T); the forward
  // tangent reads traj directly
  const int g_lo = std::max(c.w0, 0), g_hi = std::min(c.w0 + c.W, c.N);
  if (g_hi <= g_lo) return;
  dim3 grid((c.m + 31) / 32, g_hi - g_lo), block(32, 8);
  LaunchScope ls(c, K_MODEL, (double)(g_hi - g_lo) * c.m * c.s * 29.0 * (c.l96_nsub - 1),
                 (double)(g_hi - g_lo) * c.m * c.s * 8 * (1 + c.l96_nsub));
#define WF_SUBST(I, S) k_l96_substates<I, S><<<grid, block, 0, c.st>>>(c.l96_sub, c.traj, c.l96_F, c.l96_dt, c.s, c.m, c.l96_nsub, g_lo)
  if (c.s == 40) WF_SUBST(5, true);
  else if (c.s == 64) WF_SUBST(8, true);
  else if (c.s <= 40) WF_SUBST(5, false);
  else WF_SUBST(8, false);
#undef WF_SUBST
  WF_CUDA(cudaGetLastError());
  c.launches++;
}

template <int IPT, bool SH, int LPP = 8>
static void launch_step(Ctx &c, const L96Args &a, dim3 grid, bool transpose) {
  constexpr int NT = LPP == 8 ? 256 : 128;
  const dim3 block(32, NT / 32);
  if (!transpose) k_l96_step<IPT, SH, false, LPP><<<grid, block, 0, c.st>>>(a);
  else {
    const int smem = L96_ADJ_STASH ? 2 * IPT * NT * (int)sizeof(double) : 0;
    if (smem > 48 * 1024) {
      static const cudaError_t attr = cudaFuncSetAttribute(
          k_l96_step<IPT, SH, true, LPP>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      WF_CUDA(attr);
    }
    k_l96_step<IPT, SH, true, LPP><<<grid, block, smem, c.st>>>(a);
  }
}

static void l96_launch(Ctx &c, bool transpose, double sign, const double *in, const double *base,
                       double *out, int w_first, int w_step, int nw, int w_first1, int nw1,
                       const double *add2, const int *row_map);

void l96_step(Ctx &c, bool transpose, double sign, const double *in, const double *base, double *out,
              int w_first, int w_step, int nw, const double *add2, const int *row_map) {
  l96_launch(c, transpose, sign, in, base, out, w_first, w_step, nw, 0, 0, add2, row_map);
}

void l96_step2(Ctx &c, bool transpose, double *z, int f0, int s0, int n0, int f1, int n1) {
  l96_launch(c, transpose, 1.0, z, z, z, f0, s0, n0, f1, n1, nullptr, nullptr);
}

static void l96_launch(Ctx &c, bool transpose, double sign, const double *in, const double *base,
                       double *out, int w_first, int w_step, int nw, int w_first1, int nw1,
                       const double *add2, const int *row_map) {
  L96Args a{};
  a.nw0 = nw; a.w_first1 = w_first1;
  nw += nw1;
  a.out = out; a.base = base; a.in = in; a.traj = c.traj; a.sub = c.l96_sub; a.add2 = add2; a.row_map = row_map;
  a.sign = sign; a.F = c.l96_F; a.dt = c.l96_dt; a.h6 = c.l96_dt / 6.0; a.h3 = c.l96_dt / 3.0; a.s = c.s; a.W = c.W; a.m = c.m;
  a.w0 = c.w0; a.WG = c.WG; a.halo = transpose ? c.halo_hi : c.halo_lo;
  a.nsub = c.l96_nsub; a.w_first = w_first; a.w_step = w_step; a.nw = nw;
  a.dir = transpose ? 1 : -1;
  dim3 grid((c.m + 31) / 32, nw);
  // flops per state element and RK4 substep, counted from the kernel's arithmetic:
  //   nonlinear stages: 4 tendencies x 4 + stage states 3 x 2 + update 7      = 29
  //   tangent:  4 Jacobian products x 6 + stage tangents 3 x 2 + update 7      = 37
  //   adjoint:  4 transposed products x 7 + adjoint stage combinations 14      = 42,
  //             plus the inner stage states x2..x4 recomputed from the stored substep
  //             start state: 3 tendencies x 4 + 3 stage states x 2              = 18
  //             (round 1 re-integrated the start states too: 29 (2 nsub - 1) + 42 nsub)
  const double nl = 29.0, tl = 37.0, ad = 42.0, ns = c.l96_nsub;
  const double per = transpose ? (18.0 + ad) * ns : (nl + tl) * ns;
  double flops = (double)nw * c.m * c.s * per;
  LaunchScope ls(c, K_MODEL, flops, (double)nw * c.m * c.s * 8 * (4 + (transpose ? ns : 0)));
  // contiguous ownership with shuffled neighbours when s == 8 IPT (c2: s = 40)
  static const int lpp = env_int("WF4DVAR_L96_LPP", 8);
  if (c.s == 40 && lpp == 4) launch_step<10, true, 4>(c, a, grid, transpose);
  else if (c.s == 40) launch_step<5, true>(c, a, grid, transpose);
  else if (c.s == 64) launch_step<8, true>(c, a, grid, transpose);
  else if (c.s <= 40) launch_step<5, false>(c, a, grid, transpose);
  else launch_step<8, false>(c, a, grid, transpose);
  WF_CUDA(cudaGetLastError());
  c.launches++;
}

// Nonlinear forecast for the Gauss-Newton outer loop: for every local
// window w with a global predecessor, out_w = M_w(x_{w-1}) = nsub nonlinear RK4 steps
// of Lorenz-96 from the state of window w-1 (local, or the low halo on a rank
// boundary).  Same thread mapping as k_l96_step.
template <int IPT, bool SH>
__global__ void __launch_bounds__(256) k_l96_forecast(double *out, const double *x,
                                                      const double *halo, double F, double h,
                                                      int s, int W, int m, int nsub, int w0) {
  __shared__ double bx[L96Thread<IPT>::S_MAX * 32];
  const int tid = threadIdx.y * 32 + threadIdx.x;
  const int wp = tid >> 5, lw = tid & 31;
  const int lane = lw >> 3, ty = lw & 7;
  const int r = blockIdx.x * 32 + wp * 4 + lane;
  double *const bxw = bx + wp * (L96Thread<IPT>::S_MAX * 4);
  const int w = blockIdx.y;                    // local window
  if (w0 + w < 1) return;                      // global window 0 has no forecast
  const bool live = r < m;
  const int64_t ld = (int64_t)W * m;
  double xs[IPT];
#pragma unroll
  for (int k = 0; k < IPT; ++k) {
    const int i = SH ? ty * IPT + k : ty + 8 * k;
    xs[k] = (live && i < s) ? (w == 0 ? halo[(int64_t)i * m + r] : x[i * ld + (int64_t)(w - 1) * m + r])
                            : 0.0;
  }
  for (int st = 0; st < nsub; ++st) {
    double x2[IPT], x3[IPT], x4[IPT], xn[IPT];
    rk4_stages<IPT, SH>(xs, x2, x3, x4, xn, bxw, s, ty, lane, F, h);
#pragma unroll
    for (int k = 0; k < IPT; ++k) xs[k] = xn[k];
  }
  if (!live) return;
#pragma unroll
  for (int k = 0; k < IPT; ++k) {
    const int i = SH ? ty * IPT + k : ty + 8 * k;
    if (i < s) out[i * ld + (int64_t)w * m + r] = xs[k];
  }
}

void l96_forecast(Ctx &c, const double *x, double *out) {
  dim3 grid((c.m + 31) / 32, c.W), block(32, 8);
  LaunchScope ls(c, K_MODEL, (double)c.W * c.m * c.s * 29.0 * c.l96_nsub,
                 (double)c.W * c.m * c.s * 16);
  if (c.s == 40) k_l96_forecast<5, true><<<grid, block, 0, c.st>>>(out, x, c.halo_lo, c.l96_F, c.l96_dt, c.s, c.W, c.m, c.l96_nsub, c.w0);
  else if (c.s == 64) k_l96_forecast<8, true><<<grid, block, 0, c.st>>>(out, x, c.halo_lo, c.l96_F, c.l96_dt, c.s, c.W, c.m, c.l96_nsub, c.w0);
  else if (c.s <= 40) k_l96_forecast<5, false><<<grid, block, 0, c.st>>>(out, x, c.halo_lo, c.l96_F, c.l96_dt, c.s, c.W, c.m, c.l96_nsub, c.w0);
  else k_l96_forecast<8, false><<<grid, block, 0, c.st>>>(out, x, c.halo_lo, c.l96_F, c.l96_dt, c.s, c.W, c.m, c.l96_nsub, c.w0);
  WF_CUDA(cudaGetLastError());
  c.launches++;
}

}  // namespace wf
