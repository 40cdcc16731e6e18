// Gauss-Newton outer loops of incremental weak-constraint 4D-Var (
// "the outer loop is used to update linearisations of model and observation
// operators"; P:L687 for Lorenz-96).  Outer iteration l, from the current iterate
// x^(l) = (x_0 .. x_N):
//   linearise   M_w^(l) = tangent linear of M_w about x_{w-1}^(l) (the trajectory the
//               L96 kernels read), H linear;
//   right-hand side (reading A3)
//               b_0 = x_b - x_0,  b_w = M_w(x_{w-1}) - x_w  (w >= 1),
//               d_w = y_w - H x_w,  third block 0;
//   inner loop  the saddle system A (delta eta, delta nu, delta x) = (b, d, 0) solved by
//               the batched preconditioned MINRES / GMRES of krylov.cu;
//   update      x^(l+1) = x^(l) + delta x.
// Every step is a kernel of this library; the windows may be sharded (halo of
// x_{w0-1} from rank-1 for the forecast and the trajectory).
#include <algorithm>
#include <cmath>
#include <vector>

#include "internal.h"

namespace wf {

void l96_forecast(Ctx &c, const double *x, double *out);

// traj[g] (start state of window g, read by M_{g+1}) for the local windows g <= N-1;
// traj[w0 - 1] from the low halo
__global__ void k_set_traj(double *traj, const double *x, const double *halo, int s, int W, int m,
                           int w0, int N) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t per = (int64_t)s * m;
  if (e >= per * (W + 1)) return;
  const int wl = (int)(e / per) - 1;           // -1 = the halo window
  const int64_t rem = e % per;
  const int i = (int)(rem / m), r = (int)(rem % m);
  const int g = w0 + wl;
  if (g < 0 || g > N - 1) return;
  double v;
  if (wl < 0) {
    if (!halo) return;
    v = halo[(int64_t)i * m + r];
  } else {
    v = x[((int64_t)i * W + wl) * m + r];
  }
  traj[((int64_t)g * s + i) * m + r] = v;
}

// b_w = (global w == 0) ? x_b - x_0 : fc_w - x_w     ([s][W][m]; xb is [s][m])
__global__ void k_outer_b(double *b, const double *fc, const double *x, const double *xb, int s,
                          int W, int m, int w0) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t ld = (int64_t)W * m;
  if (e >= (int64_t)s * ld) return;
  const int64_t i = e / ld, col = e % ld;
  const int wl = (int)(col / m), r = (int)(col % m);
  const double xv = x[e];
  b[e] = (w0 + wl == 0) ? xb[i * m + r] - xv : fc[e] - xv;
}

// d_j = y_j - x[H_idx[j]]   (selection H)
__global__ void k_obs_res(double *d, const double *y, const double *x, const int *H_idx, int p,
                          int64_t ld) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)p * ld) return;
  const int64_t j = e / ld, col = e % ld;
  d[e] = y[e] - x[(int64_t)H_idx[j] * ld + col];
}

// y = a - y (in place), x += dx
__global__ void k_rsub(double *y, const double *a, int64_t n) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n) y[e] = a[e] - y[e];
}
__global__ void k_add_inplace(double *x, const double *dx, int64_t n) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n) x[e] += dx[e];
}

static unsigned nbk(int64_t n) { return (unsigned)((n + 255) / 256); }

static void exchange_lo(Ctx &c, const double *seg) {
  if (!c.comm) return;
  const int rank = c.comm->rank, world = c.comm->world;
  const size_t cnt = (size_t)c.s * c.m;
  std::vector<Comm::P2P> ops;
  if (rank + 1 < world) {
    pack_window(c, c.pack_hi, seg, c.W - 1);
    ops.push_back({c.pack_hi, cnt, rank + 1, true});
  }
  if (rank > 0) ops.push_back({c.halo_lo, cnt, rank - 1, false});
  c.comm->exchange(ops, c.st);
}

void outer_loop(Ctx &c, const double *xb, const double *y, double *x, int n_outer,
                const wf4dvar_solve_opts &inner, int32_t *inner_iters, double *dx_norm2,
                double *res_norm2) {
  WF_REQUIRE(n_outer >= 1, WF4DVAR_EINVAL, "outer loop: n_outer >= 1");
  const int m = c.m;
  const int64_t seg = (int64_t)c.s * c.ncol, oseg = (int64_t)c.p * c.ncol;
  // the outer workspace lives outside the Krylov arena (solve() resets that one)
  if (!c.outer_ws) {
    c.outer_ws = c.alloc<double>((size_t)(2 * c.n + seg + 8 * (size_t)m));
  }
  double *rhs = c.outer_ws, *dx = rhs + c.n, *fc = dx + c.n, *dd = fc + seg;
  for (int l = 0; l < n_outer; ++l) {
    // ---- linearisation trajectory and nonlinear forecast M_w(x_{w-1})
    exchange_lo(c, x);
    if (c.model == WF4DVAR_M_L96) {
      if (c.N > 0) {
        const int64_t tot = (int64_t)c.s * m * (c.W + 1);
        k_set_traj<<<nbk(tot), 256, 0, c.st>>>(c.traj, x, c.w0 > 0 ? c.halo_lo : nullptr, c.s,
                                               c.W, m, c.w0, c.N);
        WF_CUDA(cudaGetLastError());
        c.launches++;
        l96_substates(c);
      }
      l96_forecast(c, x, fc);
    } else {
      // linear models: M_w(x_{w-1}) = M_w x_{w-1}; base = 0
      WF_CUDA(cudaMemsetAsync(fc, 0, seg * 8, c.st));
      model_step(c, false, 1.0, x, fc, fc, 0, 1, c.W);
    }
    // ---- right-hand side (b, d, 0)
    double *b = rhs, *d = rhs + seg, *z3 = rhs + seg + oseg;
    k_outer_b<<<nbk(seg), 256, 0, c.st>>>(b, fc, x, xb, c.s, c.W, m, c.w0);
    if (c.H_general) {
      csr_apply(c, d, x, c.Hrp, c.Hcol, c.Hval, c.p, false);
      k_rsub<<<nbk(oseg), 256, 0, c.st>>>(d, y, oseg);
    } else {
      k_obs_res<<<nbk(oseg), 256, 0, c.st>>>(d, y, x, c.H_idx, c.p, c.ncol);
    }
    WF_CUDA(cudaMemsetAsync(z3, 0, seg * 8, c.st));
    c.launches += 2;
    WF_CUDA(cudaGetLastError());
    if (res_norm2) {   // ||(b, d)||^2 per RHS: the nonlinear residual the outer loop drives
      const double *a[1] = {rhs};
      dots(c, 1, a, a, seg + oseg, dd);
      WF_CUDA(memcpy_sync(c, res_norm2 + (size_t)l * m, dd, m * 8, cudaMemcpyDeviceToHost));
    }
    // ---- inner loop
    std::vector<int32_t> its(m);
    wf4dvar_report rep{};
    rep.iters = its.data();
    try {
      solve(c, rhs, dx, inner, &rep);
    } catch (const Error &e) {
      if (e.st != WF4DVAR_ENOCONV) throw;   // an unconverged inner loop still updates x
    }
    if (inner_iters)
      for (int r = 0; r < m; ++r) inner_iters[(size_t)l * m + r] = its[r];
    // ---- update x += delta x
    const double *dx3 = dx + seg + oseg;
    k_add_inplace<<<nbk(seg), 256, 0, c.st>>>(x, dx3, seg);
    c.launches++;
    if (dx_norm2) {
      const double *a[1] = {dx3};
      dots(c, 1, a, a, seg, dd);
      WF_CUDA(memcpy_sync(c, dx_norm2 + (size_t)l * m, dd, m * 8, cudaMemcpyDeviceToHost));
    }
  }
  WF_CUDA(cudaStreamSynchronize(c.st));
}

}  // namespace wf
