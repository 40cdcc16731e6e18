// Sparse incomplete-Cholesky factors: the paper applies
// D_hat^{-1} and R_hat^{-1} "using the incomplete Cholesky factors computed with the
// Matlab function ichol with zero-fill, i.e. using the same sparsity structure as B
// and Q" (R_i: P:L600).
//
// Setup (host, untimed): IC(0) of the n x n matrix on the pattern of its non-zero
// lower triangle, row by row:  for k in pattern(i), k < i:
//     L_ik = (A_ik - sum_{j in pattern(i) & pattern(k), j < k} L_ij L_kj) / L_kk
//     L_ii = sqrt(A_ii - sum_{j in pattern(i), j < i} L_ij^2)
// stored as CSR of the strictly lower part, its transpose (the upper factor L^T) and
// the reciprocal diagonal.
// Apply (device): y = L^{-T} L^{-1} x as two sparse triangular solves, one thread per
// (window, RHS) column walking the rows in order -- the rows of one column are a true
// recurrence; the W m columns are independent and the reads of the factor row are
// warp-broadcast, the reads/writes of the solution coalesced across the columns.
#include <algorithm>
#include <cmath>
#include <vector>

#include "internal.h"

namespace wf {

// forward (upper = 0): y_i = (x_i - sum_{k<i} L_ik y_k) / L_ii, rows ascending
// backward (upper = 1): y_i = (x_i - sum_{k>i} U_ik y_k) / U_ii, rows descending
// Columns [c0, c0 + ncols) of [n][ld] arrays; x may alias y.
__global__ void k_sptrsv(double *y, const double *x, const int *rowptr, const int *col,
                         const double *val, const double *dinv, int n, int64_t ld, int c0,
                         int ncols, int upper) {
  const int cc = blockIdx.x * blockDim.x + threadIdx.x;
  if (cc >= ncols) return;
  const int64_t c = c0 + cc;
  for (int t = 0; t < n; ++t) {
    const int i = upper ? n - 1 - t : t;
    double acc = x[(int64_t)i * ld + c];
    const int k0 = rowptr[i], k1 = rowptr[i + 1];
    int k = k0;
    // 4 independent partial sums: the loads of one row are not serialised
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    for (; k + 4 <= k1; k += 4) {
      a0 = fma(__ldg(val + k), y[(int64_t)__ldg(col + k) * ld + c], a0);
      a1 = fma(__ldg(val + k + 1), y[(int64_t)__ldg(col + k + 1) * ld + c], a1);
      a2 = fma(__ldg(val + k + 2), y[(int64_t)__ldg(col + k + 2) * ld + c], a2);
      a3 = fma(__ldg(val + k + 3), y[(int64_t)__ldg(col + k + 3) * ld + c], a3);
    }
    for (; k < k1; ++k) a0 = fma(__ldg(val + k), y[(int64_t)__ldg(col + k) * ld + c], a0);
    acc -= (a0 + a1) + (a2 + a3);
    y[(int64_t)i * ld + c] = acc * __ldg(dinv + i);
  }
}

// Same solves with LPC lanes per column: the lanes split the row's non-zeros and
// reduce by shuffles, and the last RB solution values of the column live in a
// shared-memory ring (entries farther back -- the wrap-around corners of a periodic
// band -- are read from global memory).  r01t: the one-thread-per-column version,
// reading the solution back through L2 one latency per non-zero, ran the configs-5
// IC(0) solves at ~1 GB/s.
struct SpTri { const int *rowptr, *col; const double *val, *dinv; };

// columns [c0, c0 + nsplit) use factor f0, [c0 + nsplit, c0 + ncols) factor f1 (B on
// window 0 and Q on the other windows in ONE launch: the serial row recurrence is the
// cost, so two launches would double it)
template <int LPC, int RB, int E>
__global__ void __launch_bounds__(128) k_sptrsv_ring(double *y, const double *x, SpTri f0,
                                                     SpTri f1, int nsplit, int n, int64_t ld,
                                                     int c0, int ncols, int upper) {
  constexpr int CPB = 128 / LPC;                 // columns per block
  __shared__ double ring[RB][CPB];
  const int lc = threadIdx.x / LPC, q = threadIdx.x % LPC;
  const int cc = blockIdx.x * CPB + lc;
  const bool live = cc < ncols;
  const int64_t c = c0 + (live ? cc : 0);
  const SpTri &F = cc < nsplit ? f0 : f1;
  const int *rowptr = F.rowptr, *col = F.col;
  const double *val = F.val, *dinv = F.dinv;
  // software pipeline: the next row's factor entries (up to E per lane, i.e. LPC*E per
  // row -- longer rows take a slow tail loop) and right-hand side are loaded while the
  // current row is reduced, so each row costs one shared-memory round instead of a
  // chain of L2 latencies
  int jn[E];
  double vn[E], xn = 0.0, dn = 0.0;
  int kn0 = 0, kn1 = 0;
  auto fetch = [&](int i) {
    kn0 = __ldg(rowptr + i);
    kn1 = __ldg(rowptr + i + 1);
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int k = kn0 + q + e * LPC;
      jn[e] = k < kn1 ? __ldg(col + k) : -1;
      vn[e] = k < kn1 ? __ldg(val + k) : 0.0;
    }
    xn = live ? x[(int64_t)i * ld + c] : 0.0;
    dn = __ldg(dinv + i);
  };
  fetch(upper ? n - 1 : 0);
  for (int t = 0; t < n; ++t) {
    const int i = upper ? n - 1 - t : t;
    int jj[E];
    double vv[E];
#pragma unroll
    for (int e = 0; e < E; ++e) { jj[e] = jn[e]; vv[e] = vn[e]; }
    const double xi = xn, di = dn;
    const int k0 = kn0, k1 = kn1;
    if (t + 1 < n) fetch(upper ? i - 1 : i + 1);
    double a0 = 0.0, a1 = 0.0;
#pragma unroll
    for (int e = 0; e < E; e += 2) {
      if (jj[e] >= 0) {
        const int d = upper ? jj[e] - i : i - jj[e];
        a0 = fma(vv[e], d <= RB ? ring[jj[e] % RB][lc] : y[(int64_t)jj[e] * ld + c], a0);
      }
      if (e + 1 < E && jj[e + 1] >= 0) {
        const int d = upper ? jj[e + 1] - i : i - jj[e + 1];
        a1 = fma(vv[e + 1], d <= RB ? ring[jj[e + 1] % RB][lc] : y[(int64_t)jj[e + 1] * ld + c], a1);
      }
    }
    for (int k = k0 + q + E * LPC; k < k1; k += LPC) {   // rows longer than LPC * E
      const int j = __ldg(col + k);
      const int d = upper ? j - i : i - j;
      a0 = fma(__ldg(val + k), d <= RB ? ring[j % RB][lc] : y[(int64_t)j * ld + c], a0);
    }
    double acc = a0 + a1;
#pragma unroll
    for (int o = LPC / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o, LPC);
    const double yi = (xi - acc) * di;
    if (q == 0) {
      ring[i % RB][lc] = yi;
      if (live) y[(int64_t)i * ld + c] = yi;
    }
    __syncwarp();
  }
}

// IC(0) of the row-major n x n host matrix A (exact zeros outside the pattern).
static void ichol0_host(const std::vector<double> &A, int n, const char *name,
                        std::vector<int> &lrp, std::vector<int> &lci, std::vector<double> &lv,
                        std::vector<double> &diag) {
  // pattern of the strictly lower triangle, row by row (column indices ascending)
  std::vector<std::vector<int>> pat(n);
  std::vector<std::vector<double>> Lrow(n);
  diag.assign(n, 0.0);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < i; ++j)
      if (A[(size_t)i * n + j] != 0.0) pat[i].push_back(j);
  for (int i = 0; i < n; ++i) {
    Lrow[i].assign(pat[i].size(), 0.0);
    for (size_t a = 0; a < pat[i].size(); ++a) {
      const int k = pat[i][a];
      // sum over j < k in pattern(i) and pattern(k): merge of two sorted lists
      double sum = 0.0;
      size_t p = 0, q = 0;
      while (p < a && q < pat[k].size()) {
        const int jp = pat[i][p], jq = pat[k][q];
        if (jp == jq) { sum += Lrow[i][p] * Lrow[k][q]; ++p; ++q; }
        else if (jp < jq) ++p;
        else ++q;
      }
      Lrow[i][a] = (A[(size_t)i * n + k] - sum) / diag[k];
    }
    double d = A[(size_t)i * n + i];
    for (double v : Lrow[i]) d -= v * v;
    WF_REQUIRE(d > 0.0, WF4DVAR_ENOTSPD,
               std::string("IC(0) breakdown (non-positive pivot) of ") + name + " at row " +
                   std::to_string(i));
    diag[i] = std::sqrt(d);
  }
  lrp.assign(n + 1, 0);
  lci.clear();
  lv.clear();
  for (int i = 0; i < n; ++i) {
    for (size_t a = 0; a < pat[i].size(); ++a) {
      lci.push_back(pat[i][a]);
      lv.push_back(Lrow[i][a]);
    }
    lrp[i + 1] = (int)lci.size();
  }
}

void make_ichol(Ctx &c, const std::vector<double> &A, int n, const char *name, SparseFactor &f) {
  std::vector<int> lrp, lci;
  std::vector<double> lv, diag;
  ichol0_host(A, n, name, lrp, lci, lv, diag);
  const int nnz = (int)lci.size();
  // upper factor L^T as CSR: row k of L^T holds column k of L
  std::vector<int> urp(n + 1, 0), uci(nnz);
  std::vector<double> uv(nnz), dinv(n);
  for (int k = 0; k < nnz; ++k) urp[lci[k] + 1]++;
  for (int i = 0; i < n; ++i) urp[i + 1] += urp[i];
  std::vector<int> fill(urp.begin(), urp.end() - 1);
  for (int i = 0; i < n; ++i)
    for (int k = lrp[i]; k < lrp[i + 1]; ++k) {
      const int dst = fill[lci[k]]++;
      uci[dst] = i;
      uv[dst] = lv[k];
    }
  for (int i = 0; i < n; ++i) dinv[i] = 1.0 / diag[i];
  f.n = n;
  f.nnz = nnz;
  f.lrp = c.alloc<int>(n + 1); f.urp = c.alloc<int>(n + 1);
  f.lci = c.alloc<int>(std::max(nnz, 1)); f.uci = c.alloc<int>(std::max(nnz, 1));
  f.lv = c.alloc<double>(std::max(nnz, 1)); f.uv = c.alloc<double>(std::max(nnz, 1));
  f.dinv = c.alloc<double>(n);
  WF_CUDA(memcpy_sync(c, f.lrp, lrp.data(), (n + 1) * 4, cudaMemcpyHostToDevice));
  WF_CUDA(memcpy_sync(c, f.urp, urp.data(), (n + 1) * 4, cudaMemcpyHostToDevice));
  if (nnz) {
    WF_CUDA(memcpy_sync(c, f.lci, lci.data(), nnz * 4, cudaMemcpyHostToDevice));
    WF_CUDA(memcpy_sync(c, f.uci, uci.data(), nnz * 4, cudaMemcpyHostToDevice));
    WF_CUDA(memcpy_sync(c, f.lv, lv.data(), (size_t)nnz * 8, cudaMemcpyHostToDevice));
    WF_CUDA(memcpy_sync(c, f.uv, uv.data(), (size_t)nnz * 8, cudaMemcpyHostToDevice));
  }
  WF_CUDA(memcpy_sync(c, f.dinv, dinv.data(), (size_t)n * 8, cudaMemcpyHostToDevice));
  static const int dense_env = env_int("WF4DVAR_ICHOL_DENSE_MAX", 4096);   // tuning knob
  if (n <= dense_env) {
    // densified L and L^T for the DMMA TRSM path (the values are the IC(0) factor's)
    std::vector<double> Ld((size_t)n * n, 0.0), Ud((size_t)n * n, 0.0);
    for (int i = 0; i < n; ++i) {
      Ld[(size_t)i * n + i] = Ud[(size_t)i * n + i] = diag[i];
      for (int k = lrp[i]; k < lrp[i + 1]; ++k) {
        Ld[(size_t)i * n + lci[k]] = lv[k];
        Ud[(size_t)lci[k] * n + i] = lv[k];
      }
    }
    f.Gd = c.alloc<double>((size_t)n * n);
    f.Gdt = c.alloc<double>((size_t)n * n);
    WF_CUDA(memcpy_sync(c, f.Gd, Ld.data(), Ld.size() * 8, cudaMemcpyHostToDevice));
    WF_CUDA(memcpy_sync(c, f.Gdt, Ud.data(), Ud.size() * 8, cudaMemcpyHostToDevice));
    f.Pd = make_diag_pack(c, f.Gd, n, false);
    f.Pdt = make_diag_pack(c, f.Gdt, n, true);
  }
}

// y[:, c0:c0+ncols] = (L L^T)^{-1} x[:, c0:c0+ncols] over an [n][ncol] segment; with g
// given, columns from c0 + nsplit on use the factor g (same n) in the same launches
void ichol_solve(Ctx &c, const SparseFactor &f, const double *x, double *y, int c0, int ncols,
                 const SparseFactor *g, int nsplit) {
  if (ncols <= 0) return;
  if (!g) { g = &f; nsplit = ncols; }
  if (f.Gd && g->Gd) {
    // dense DMMA TRSM pair on the densified factors (B / Q groups in one launch each)
    const int64_t ld = c.ncol;
    TrsmProb fw[2], bw[2];
    int np = 0;
    const SparseFactor *fs[2] = {&f, g};
    const int cs[2] = {c0, c0 + nsplit}, nc[2] = {nsplit, ncols - nsplit};
    for (int p = 0; p < 2; ++p) {
      if (nc[p] <= 0) continue;
      fw[np] = TrsmProb{fs[p]->Gd, fs[p]->n, x + cs[p], ld, y + cs[p], ld, fs[p]->n, nc[p], 0};
      bw[np] = TrsmProb{fs[p]->Gdt, fs[p]->n, y + cs[p], ld, y + cs[p], ld, fs[p]->n, nc[p], 0};
      fw[np].dpack = fs[p]->Pd;
      bw[np].dpack = fs[p]->Pdt;
      ++np;
    }
    launch_trsm(c, fw, np, false);
    launch_trsm(c, bw, np, true);
    return;
  }
  const double cols = ncols;
  LaunchScope ls(c, K_TRSM, 2.0 * 2.0 * f.nnz * cols + 2.0 * f.n * cols,
                 8.0 * (2.0 * f.nnz + 4.0 * f.n * cols));
  static const int ring_env = env_int("WF4DVAR_SPTRSV_RING", 1);   // tuning experiments only
  if (ring_env) {
    constexpr int LPC = 8, RB = 256, E = 16, CPB = 128 / LPC;
    const unsigned gb = (unsigned)((ncols + CPB - 1) / CPB);
    const SpTri fl{f.lrp, f.lci, f.lv, f.dinv}, fu{f.urp, f.uci, f.uv, f.dinv};
    const SpTri gl{g->lrp, g->lci, g->lv, g->dinv}, gu{g->urp, g->uci, g->uv, g->dinv};
    k_sptrsv_ring<LPC, RB, E><<<gb, 128, 0, c.st>>>(y, x, fl, gl, nsplit, f.n, c.ncol, c0, ncols,
                                                    0);
    k_sptrsv_ring<LPC, RB, E><<<gb, 128, 0, c.st>>>(y, y, fu, gu, nsplit, f.n, c.ncol, c0, ncols,
                                                    1);
  } else {
    for (int part = 0; part < 2; ++part) {
      const SparseFactor &h = part ? *g : f;
      const int a = part ? c0 + nsplit : c0, nc = part ? ncols - nsplit : nsplit;
      if (nc <= 0) continue;
      const unsigned gb = (unsigned)((nc + 127) / 128);
      k_sptrsv<<<gb, 128, 0, c.st>>>(y, x, h.lrp, h.lci, h.lv, h.dinv, h.n, c.ncol, a, nc, 0);
      k_sptrsv<<<gb, 128, 0, c.st>>>(y, y, h.urp, h.uci, h.uv, h.dinv, h.n, c.ncol, a, nc, 1);
    }
  }
  WF_CUDA(cudaGetLastError());
  c.launches += 2;
}

}  // namespace wf
