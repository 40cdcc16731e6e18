// Vector kernels of the hot path: R_diag scaling, the R_ME Woodbury
// low-rank correction (Alg. 3 applied "as a low-rank update to the Cholesky
// factors via the Woodbury identity"), and the batched per-RHS dot
// products of the Krylov solvers (deterministic two-phase reduction, no atomics).
#include "internal.h"

namespace wf {

void copy(Ctx &c, double *dst, const double *src, int64_t n) {
  if (dst == src || n <= 0) return;
  WF_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(double), cudaMemcpyDeviceToDevice, c.st));
}

__global__ void k_scale_rows(double *y, const double *x, const double *rs, int rows, int64_t ld) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)rows * ld) return;
  y[e] = x[e] * rs[e / ld];
}

void scale_rows(Ctx &c, double *y, const double *x, const double *rs, int rows) {
  int64_t tot = (int64_t)rows * c.ncol;
  LaunchScope ls(c, K_VEC, (double)tot, 16.0 * tot);
  k_scale_rows<<<(unsigned)((tot + 255) / 256), 256, 0, c.st>>>(y, x, rs, rows, c.ncol);
  WF_CUDA(cudaGetLastError());
  c.launches++;
}

// t[j][col] = sum_i U[i][j] x[i][col]   then   s = Kinv t   (r <= 8)
template <int RM>
__global__ void k_lowrank_t(double *s_out, const double *x, const double *U, const double *Kinv,
                            int p, int r, int64_t ld) {
  int64_t col = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= ld) return;
  double t[RM];
#pragma unroll
  for (int j = 0; j < RM; ++j) t[j] = 0.0;
  for (int i = 0; i < p; ++i) {
    double xv = x[(int64_t)i * ld + col];
#pragma unroll
    for (int j = 0; j < RM; ++j)
      if (j < r) t[j] = fma(U[i * r + j], xv, t[j]);
  }
#pragma unroll
  for (int a = 0; a < RM; ++a) {
    if (a >= r) break;
    double v = 0.0;
#pragma unroll
    for (int b = 0; b < RM; ++b)
      if (b < r) v = fma(Kinv[a * r + b], t[b], v);
    s_out[(int64_t)a * ld + col] = v;
  }
}

// y[i][col] -= sum_j U[i][j] s[j][col]
__global__ void k_lowrank_apply(double *y, const double *s_in, const double *U, int p, int r,
                                int64_t ld) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)p * ld) return;
  int64_t i = e / ld, col = e % ld;
  double v = 0.0;
  for (int j = 0; j < r; ++j) v = fma(U[i * r + j], s_in[(int64_t)j * ld + col], v);
  y[e] -= v;
}

void lowrank_correct(Ctx &c, double *y, const double *x) {
  if (c.r_me <= 0) return;
  const int p = c.p, r = c.r_me;
  const int64_t ld = c.ncol;
  {
    LaunchScope ls(c, K_VEC, 2.0 * p * r * (double)ld, 8.0 * p * ld);
    k_lowrank_t<8><<<(unsigned)((ld + 127) / 128), 128, 0, c.st>>>(c.ws_lr, x, c.U_me, c.Kinv_me,
                                                                    p, r, ld);
    WF_CUDA(cudaGetLastError());
    c.launches++;
  }
  {
    int64_t tot = (int64_t)p * ld;
    LaunchScope ls(c, K_VEC, 2.0 * p * r * (double)ld, 16.0 * tot);
    k_lowrank_apply<<<(unsigned)((tot + 255) / 256), 256, 0, c.st>>>(y, c.ws_lr, c.U_me, p, r, ld);
    WF_CUDA(cudaGetLastError());
    c.launches++;
  }
}

// ------------------------------------------------------------------ dots
struct DotArgs { const double *a[4]; const double *b[4]; };

template <int ND>
__global__ void __launch_bounds__(256) k_dots_partial(DotArgs args, int64_t rows, int m, int RB,
                                                      int64_t rpb, double *part) {
  __shared__ double sm[ND][256];
  const int t = threadIdx.x;
  const int rl = t % RB, u = t / RB, U = 256 / RB;
  const int r = blockIdx.x * RB + rl;
  const int64_t row0 = (int64_t)blockIdx.y * rpb;
  const int64_t row1 = min(rows, row0 + rpb);
  double acc[ND];
#pragma unroll
  for (int d = 0; d < ND; ++d) acc[d] = 0.0;
  if (r < m && u < U) {
    // 4 rows in flight per thread (independent partial sums, combined in fixed order)
    double acc2[4][ND];
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int d = 0; d < ND; ++d) acc2[q][d] = 0.0;
    int64_t row = row0 + u;
    for (; row + 3 * U < row1; row += 4 * U) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        int64_t f = (row + q * U) * m + r;
#pragma unroll
        for (int d = 0; d < ND; ++d) acc2[q][d] = fma(args.a[d][f], args.b[d][f], acc2[q][d]);
      }
    }
    for (; row < row1; row += U) {
      int64_t f = row * m + r;
#pragma unroll
      for (int d = 0; d < ND; ++d) acc2[0][d] = fma(args.a[d][f], args.b[d][f], acc2[0][d]);
    }
#pragma unroll
    for (int d = 0; d < ND; ++d) acc[d] = (acc2[0][d] + acc2[1][d]) + (acc2[2][d] + acc2[3][d]);
  }
#pragma unroll
  for (int d = 0; d < ND; ++d) sm[d][t] = acc[d];
  __syncthreads();
  if (u == 0 && r < m) {
#pragma unroll
    for (int d = 0; d < ND; ++d) {
      double v = 0.0;
      for (int uu = 0; uu < U; ++uu) v += sm[d][uu * RB + rl];
      part[((int64_t)blockIdx.y * ND + d) * m + r] = v;
    }
  }
}

// one warp per output: lane-strided partial sums, then a fixed-order shuffle tree
// (deterministic; r01 ncu: the one-thread-per-output version took ~50 us)
__global__ void k_dots_final(const double *part, int nparts, int nd, int m, double *out) {
  const int e = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (e >= nd * m) return;
  const int d = e / m, r = e % m;
  double v = 0.0;
  for (int b = lane; b < nparts; b += 32) v += part[((int64_t)b * nd + d) * m + r];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if (lane == 0) out[e] = v;
}

RedGrid red_grid(const Ctx &c, int64_t n) {
  RedGrid g;
  const int m = c.m;
  g.rows = n / m;
  g.RB = m < 256 ? m : 256;
  g.gx = (m + g.RB - 1) / g.RB;
  // >= ~6 blocks of 256 threads per SM even when rows = n/m is small (configs[2]:
  // m = 1024, rows = 5100: the old rows/256 cap gave 80 blocks, 1.2 TB/s)
  g.gy = (int)std::max<int64_t>(1, std::min<int64_t>((6 * 148 + g.gx - 1) / g.gx, (g.rows + 31) / 32));
  g.rpb = (g.rows + g.gy - 1) / g.gy;
  g.gy = (int)((g.rows + g.rpb - 1) / g.rpb);
  return g;
}

void reduce_final(Ctx &c, const double *part, int nparts, int nd, double *out) {
  LaunchScope ls(c, K_DOT, 0, 8.0 * nparts * nd * c.m);
  k_dots_final<<<(nd * c.m + 7) / 8, 256, 0, c.st>>>(part, nparts, nd, c.m, out);
  WF_CUDA(cudaGetLastError());
  c.launches++;
  allreduce(c, out, (size_t)nd * c.m);
}

// y[i][col] (+)= sum_k val[k] x[col_k][col]: one thread per (row, column), columns
// fastest (coalesced across the W m columns of a segment)
__global__ void k_csr_apply(double *y, const double *x, const int *rowptr, const int *col,
                            const double *val, int nrows, int64_t ld, int accumulate) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)nrows * ld) return;
  const int64_t i = e / ld, cc = e - i * ld;
  double v = accumulate ? y[e] : 0.0;
  for (int k = rowptr[i]; k < rowptr[i + 1]; ++k) v = fma(val[k], x[(int64_t)col[k] * ld + cc], v);
  y[e] = v;
}

void csr_apply(Ctx &c, double *y, const double *x, const int *rowptr, const int *col,
               const double *val, int nrows, bool accumulate) {
  const int64_t tot = (int64_t)nrows * c.ncol;
  if (tot == 0) return;
  LaunchScope ls(c, K_VEC, 0, 8.0 * 2 * tot);
  k_csr_apply<<<(unsigned)((tot + 255) / 256), 256, 0, c.st>>>(y, x, rowptr, col, val, nrows,
                                                               c.ncol, accumulate ? 1 : 0);
  WF_CUDA(cudaGetLastError());
  c.launches++;
}

void allreduce(Ctx &c, double *buf, size_t count) {
  if (c.comm) c.comm->allreduce_sum(buf, count, c.st);
}

void dots(Ctx &c, int nd, const double *const *a, const double *const *b, int64_t n, double *out) {
  const int m = c.m;
  const RedGrid rg = red_grid(c, n);
  const int64_t rows = rg.rows, rpb = rg.rpb;
  const int RB = rg.RB, gx = rg.gx, gy = rg.gy;
  const int need = gy * nd * m;
  WF_REQUIRE(need <= c.dot_part_cap, WF4DVAR_EINVAL, "dot partial buffer too small");
  DotArgs args{};
  for (int d = 0; d < nd; ++d) { args.a[d] = a[d]; args.b[d] = b[d]; }
  {
    LaunchScope ls(c, K_DOT, 2.0 * nd * n, 16.0 * nd * n);
    dim3 grid(gx, gy);
    switch (nd) {
      case 1: k_dots_partial<1><<<grid, 256, 0, c.st>>>(args, rows, m, RB, rpb, c.dot_part); break;
      case 2: k_dots_partial<2><<<grid, 256, 0, c.st>>>(args, rows, m, RB, rpb, c.dot_part); break;
      case 3: k_dots_partial<3><<<grid, 256, 0, c.st>>>(args, rows, m, RB, rpb, c.dot_part); break;
      default: k_dots_partial<4><<<grid, 256, 0, c.st>>>(args, rows, m, RB, rpb, c.dot_part); break;
    }
    WF_CUDA(cudaGetLastError());
    c.launches++;
  }
  reduce_final(c, c.dot_part, gy, nd, out);
}

}  // namespace wf
