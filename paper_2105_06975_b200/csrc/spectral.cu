// GPU spectral suite: extreme eigenvalues by Lanczos, batched
// over the m right-hand-side columns, for the two operators the paper's theory is
// about:
//   WF4DVAR_OP_PA    P_D^{-1} A   -- Theorem 3.1, eigenvalue intervals of
//                    the block-diagonally preconditioned saddle matrix.  P_D^{-1} A is
//                    self-adjoint in the P_D inner product: preconditioned Lanczos
//                    (the recurrence MINRES runs) gives the tridiagonal T with
//                    diagonal delta_j = (A z_j)^T z_j and off-diagonal gamma_{j+1}.
//   WF4DVAR_OP_LHAT  L_hat^{-T} L^T L L_hat^{-1}  -- Section 4 (Prop. 4.4/4.5, Supp.
//                    Tables S2/S3), on the state segment [s][W][m]; plain Lanczos.
// No reorthogonalisation: the extreme Ritz values converge first (lost orthogonality
// only duplicates converged values).  The tridiagonals are copied to the host and
// their extreme eigenvalues found by Sturm-sequence bisection.
#include <algorithm>
#include <cmath>
#include <vector>

#include "internal.h"

namespace wf {

// y[f] = a[r] x1[f] + b[r] x2[f] + c[r] x3[f]   (r = f % m; x2 / x3 may be NULL)
__global__ void k_lz_lin3(double *y, const double *x1, const double *a, const double *x2,
                          const double *b, const double *x3, const double *cc, int64_t n, int m) {
  int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= n) return;
  int r = (int)(f % m);
  double v = a[r] * x1[f];
  if (x2) v = fma(b[r], x2[f], v);
  if (x3) v = fma(cc[r], x3[f], v);
  y[f] = v;
}

// per-RHS scalars of one Lanczos step
//   mode 0 (normalise):  inv = 1/sqrt(d0)  (d0 = ||v||^2 or z^T v);  gam = sqrt(d0)
//   mode 1 (after T v / A z):  alpha_j = d0;  coefficients of w - alpha v - beta_prev v_prev
__global__ void k_lz_scalars(const double *dots, double *inv, double *gam, double *alpha,
                             double *beta_prev, double *c1, double *c2, double *c3, int m,
                             int mode, double *rec_alpha, double *rec_beta, int j) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= m) return;
  const double d0 = dots[r];
  if (mode == 0) {
    const double g = d0 > 0.0 ? sqrt(d0) : 0.0;
    inv[r] = g > 0.0 ? 1.0 / g : 0.0;
    gam[r] = g;
    if (rec_beta && j >= 0) rec_beta[(int64_t)j * m + r] = g;
  } else {
    alpha[r] = d0;
    if (rec_alpha) rec_alpha[(int64_t)j * m + r] = d0;
    c1[r] = 1.0;
    c2[r] = -d0;
    c3[r] = -beta_prev[r];
  }
}

static unsigned nb(int64_t n, int b) { return (unsigned)((n + b - 1) / b); }

// smallest / largest eigenvalue of the symmetric tridiagonal (a[0..k), b[0..k-1))
static int sturm_count(const std::vector<double> &a, const std::vector<double> &b, int k, double x) {
  int cnt = 0;
  double d = 1.0;
  for (int i = 0; i < k; ++i) {
    const double bb = i ? b[i - 1] * b[i - 1] : 0.0;
    d = (a[i] - x) - (i ? bb / d : 0.0);
    if (d == 0.0) d = -1e-300;
    if (d < 0.0) ++cnt;
  }
  return cnt;
}

static void tri_extremes(const std::vector<double> &a, const std::vector<double> &b, int k,
                         double &emin, double &emax) {
  double lo = 1e300, hi = -1e300;
  for (int i = 0; i < k; ++i) {
    const double rad = (i ? std::fabs(b[i - 1]) : 0.0) + (i + 1 < k ? std::fabs(b[i]) : 0.0);
    lo = std::min(lo, a[i] - rad);
    hi = std::max(hi, a[i] + rad);
  }
  auto bis = [&](int target) {   // smallest x with count(x) >= target
    double l = lo - 1e-12 * (std::fabs(lo) + 1), h = hi + 1e-12 * (std::fabs(hi) + 1);
    for (int it = 0; it < 200; ++it) {
      const double mid = 0.5 * (l + h);
      if (mid == l || mid == h) break;
      if (sturm_count(a, b, k, mid) >= target) h = mid; else l = mid;
    }
    return 0.5 * (l + h);
  };
  emin = bis(1);
  emax = bis(k);
}

// ---- halo exchange for a stand-alone L / L^T application (apply_A does its own)
static void halo_for(Ctx &c, const double *seg, bool transpose) {
  if (!c.comm) return;
  const int rank = c.comm->rank, world = c.comm->world;
  const size_t cnt = (size_t)c.s * c.m;
  std::vector<Comm::P2P> ops;
  if (!transpose) {   // L needs window w0-1 from rank-1
    if (rank + 1 < world) {
      pack_window(c, c.pack_hi, seg, c.W - 1);
      ops.push_back({c.pack_hi, cnt, rank + 1, true});
    }
    if (rank > 0) ops.push_back({c.halo_lo, cnt, rank - 1, false});
  } else {            // L^T needs window w0+W from rank+1
    if (rank > 0) {
      pack_window(c, c.pack_lo, seg, 0);
      ops.push_back({c.pack_lo, cnt, rank - 1, true});
    }
    if (rank + 1 < world) ops.push_back({c.halo_hi, cnt, rank + 1, false});
  }
  c.comm->exchange(ops, c.st);
}

void lanczos(Ctx &c, int op, const double *v0, int steps, double *ritz_min, double *ritz_max,
             double *alpha_out, double *beta_out) {
  WF_REQUIRE(steps >= 1, WF4DVAR_EINVAL, "lanczos: steps >= 1");
  WF_REQUIRE(op == WF4DVAR_OP_PA || op == WF4DVAR_OP_LHAT, WF4DVAR_EINVAL, "lanczos: bad op");
  if (op == WF4DVAR_OP_PA)
    WF_REQUIRE(c.pc.shape == WF4DVAR_PD, WF4DVAR_EINVAL, "lanczos PA needs P_D (SPD)");
  const int m = c.m;
  const int64_t seg = (int64_t)c.s * c.ncol;
  const int64_t n = (op == WF4DVAR_OP_PA) ? c.n : seg;
  const int64_t vb = ((n * 8 + 255) / 256) * 256;
  c.kws_reset(6 * vb + 16 * (size_t)m * 8 + 2 * (size_t)steps * m * 8 + 4096);
  double *v = c.kws_take<double>(n), *vp = c.kws_take<double>(n), *w = c.kws_take<double>(n),
         *z = c.kws_take<double>(n), *t1 = c.kws_take<double>(n), *t2 = c.kws_take<double>(n);
  double *S = c.kws_take<double>(16 * (size_t)m);
  double *dots_d = S, *inv = S + m, *gam = S + 2 * m, *alpha = S + 3 * m, *bprev = S + 4 * m,
         *c1 = S + 5 * m, *c2 = S + 6 * m, *c3 = S + 7 * m;
  double *rec_a = c.kws_take<double>((size_t)steps * m);
  double *rec_b = c.kws_take<double>((size_t)steps * m);
  WF_CUDA(cudaMemsetAsync(S, 0, 16 * (size_t)m * 8, c.st));
  WF_CUDA(cudaMemsetAsync(vp, 0, n * 8, c.st));
  // operator T x (LHAT) on the state segment
  auto apply_T = [&](const double *x, double *y) {
    copy(c, t1, x, seg);
    lhat_solve(c, false, t1);                                  // L_hat^{-1}
    halo_for(c, t1, false);
    model_step(c, false, -1.0, t1, t1, t2, 0, 1, c.W);         // L
    halo_for(c, t2, true);
    model_step(c, true, -1.0, t2, t2, y, 0, 1, c.W);           // L^T
    lhat_solve(c, true, y);                                    // L_hat^{-T}
  };
  const double *v0s = (op == WF4DVAR_OP_PA) ? v0 : v0 + (int64_t)(c.s + c.p) * c.ncol;
  copy(c, v, v0s, n);
  if (op == WF4DVAR_OP_PA) {
    apply_P(c, v, z);                                          // z_1 = P^{-1} v_1
    const double *a[1] = {z}, *bb[1] = {v};
    dots(c, 1, a, bb, n, dots_d);
  } else {
    const double *a[1] = {v};
    dots(c, 1, a, a, n, dots_d);
  }
  k_lz_scalars<<<nb(m, 128), 128, 0, c.st>>>(dots_d, inv, gam, alpha, bprev, c1, c2, c3, m, 0,
                                             nullptr, nullptr, -1);
  c.launches++;
  int k_done = 0;
  for (int j = 0; j < steps; ++j) {
    // normalise: v <- v / gamma (and z for PA);  bprev holds gamma_j for the 3-term update
    k_lz_lin3<<<nb(n, 256), 256, 0, c.st>>>(v, v, inv, nullptr, nullptr, nullptr, nullptr, n, m);
    c.launches++;
    if (op == WF4DVAR_OP_PA) {
      k_lz_lin3<<<nb(n, 256), 256, 0, c.st>>>(z, z, inv, nullptr, nullptr, nullptr, nullptr, n, m);
      c.launches++;
      apply_A(c, z, w);                                        // q = A z_j
      const double *a[1] = {w}, *bb[1] = {z};
      dots(c, 1, a, bb, n, dots_d);                            // delta_j
    } else {
      apply_T(v, w);
      const double *a[1] = {w}, *bb[1] = {v};
      dots(c, 1, a, bb, n, dots_d);                            // alpha_j
    }
    k_lz_scalars<<<nb(m, 128), 128, 0, c.st>>>(dots_d, inv, gam, alpha, bprev, c1, c2, c3, m, 1,
                                               rec_a, nullptr, j);
    k_lz_lin3<<<nb(n, 256), 256, 0, c.st>>>(w, w, c1, v, c2, vp, c3, n, m);
    c.launches += 2;
    std::swap(vp, v);        // vp <- v_j (normalised)
    std::swap(v, w);         // v  <- unnormalised v_{j+1}
    if (op == WF4DVAR_OP_PA) {
      apply_P(c, v, z);
      const double *a[1] = {z}, *bb[1] = {v};
      dots(c, 1, a, bb, n, dots_d);
    } else {
      const double *a[1] = {v};
      dots(c, 1, a, a, n, dots_d);
    }
    k_lz_scalars<<<nb(m, 128), 128, 0, c.st>>>(dots_d, inv, gam, alpha, bprev, c1, c2, c3, m, 0,
                                               nullptr, rec_b, j);
    c.launches++;
    // the next step's 3-term update uses beta_{j+1} = gamma_{j+1}
    WF_CUDA(cudaMemcpyAsync(bprev, gam, m * 8, cudaMemcpyDeviceToDevice, c.st));
    WF_CUDA(cudaGetLastError());
    ++k_done;
  }
  std::vector<double> ha((size_t)steps * m), hb((size_t)steps * m);
  WF_CUDA(memcpy_sync(c, ha.data(), rec_a, ha.size() * 8, cudaMemcpyDeviceToHost));
  WF_CUDA(memcpy_sync(c, hb.data(), rec_b, hb.size() * 8, cudaMemcpyDeviceToHost));
  for (int r = 0; r < m; ++r) {
    std::vector<double> a(k_done), b(k_done);
    double scale = 0.0;
    for (int j = 0; j < k_done; ++j) {
      a[j] = ha[(size_t)j * m + r];
      b[j] = hb[(size_t)j * m + r];
      scale = std::max(scale, std::fabs(a[j]) + std::fabs(b[j]));
    }
    // an (almost) invariant Krylov subspace ends the tridiagonal
    int k = k_done;
    for (int j = 0; j + 1 < k_done; ++j)
      if (!(std::fabs(b[j]) > 1e-13 * scale)) { k = j + 1; break; }
    double lo = 0, hi = 0;
    tri_extremes(a, b, k, lo, hi);
    if (ritz_min) ritz_min[r] = lo;
    if (ritz_max) ritz_max[r] = hi;
    for (int j = 0; j < k_done; ++j) {
      if (alpha_out) alpha_out[(size_t)j * m + r] = a[j];
      if (beta_out) beta_out[(size_t)j * m + r] = b[j];
    }
  }
}

}  // namespace wf
