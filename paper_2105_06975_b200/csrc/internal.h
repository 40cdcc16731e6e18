// Internal declarations of the wf4dvar CUDA library (not part of the C ABI).
#pragma once
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <stdint.h>
#include <stdlib.h>

#include <string>
#include <vector>

#include "../../include/wf4dvar.h"

namespace wf {

// integer tuning knob from the environment (read once by the callers' static locals)
inline int env_int(const char *name, int dflt) {
  const char *e = getenv(name);
  return e ? atoi(e) : dflt;
}

// ---------------------------------------------------------------- errors
struct Error {
  wf4dvar_status st;
  std::string msg;
};

#define WF_CUDA(call)                                                              \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess)                                                         \
      throw ::wf::Error{WF4DVAR_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)}; \
  } while (0)

#define WF_REQUIRE(cond, code, text)                                               \
  do {                                                                             \
    if (!(cond)) throw ::wf::Error{code, text};                                    \
  } while (0)

// ---------------------------------------------------------------- profiling
// K_GEMM: covariance / dense-model products (a1, a2, a10, a12);  K_TRSM: triangular
// panel solves (a7, a8);  K_TRSM_UPD: the DMMA GEMM coupling of a solved TRSM
// super-block to the remaining rows (same k_gemm kernel, counted with the solve).
enum KClass { K_GEMM = 0, K_TRSM, K_TRSM_UPD, K_MODEL, K_VEC, K_DOT, K_SCALAR, K_NCLASS };
static const char *const kClassName[K_NCLASS] = {"gemm_dmma", "trsm_dmma", "trsm_update_dmma",
                                                 "model_stencil", "vector", "dot_reduce",
                                                 "krylov_scalar"};

struct Prof {
  bool on = false;
  int64_t launches[K_NCLASS] = {0};
  double flops[K_NCLASS] = {0};
  double bytes[K_NCLASS] = {0};
  double ms[K_NCLASS] = {0};
  struct Pending { cudaEvent_t a, b; int cls; };
  std::vector<Pending> pending;
  std::vector<cudaEvent_t> pool;
};

// ---------------------------------------------------------------- tile column ranges
// Non-zero columns of a dense-stored matrix per 64-row tile, as at most two disjoint
// intervals [a0, a1) u [b0, b1) (multiples of 16, b0 == b1 when there is one): the
// compact-support (modified-SOAR) covariances of the paper's workload and
// their Cholesky / IC(0) factors are periodic bands, so a 64-row tile meets the
// diagonal band plus at most one wrap-around block.  The DMMA GEMM and TRSM kernels
// skip the K tiles outside them (the dense storage stays; the zeros are not read).
struct KRange { int a0, a1, b0, b1; };
struct TileRanges {
  const double *base = nullptr;
  int64_t ld = 0;
  int rows = 0, cols = 0;
  double coverage = 1.0;        // covered tile area / (rows x cols)
  KRange *d = nullptr;          // device, one per 64-row tile
  std::vector<KRange> h;        // host copy (flop accounting)
};
struct Ctx;
// scan G on the device and register its ranges if they skip >= 25% of the tiles
void register_tile_ranges(Ctx &c, const double *G, int rows, int cols, int64_t ld);
void unregister_tile_ranges(Ctx &c, const void *G);
// the registered matrix containing A (row offset a multiple of 64), else nullptr
const TileRanges *find_tile_ranges(const Ctx &c, const double *A, int *row0, int *col0);
// sum over the 64-row tiles of rows [r0, r0 + nrows) of rows x covered columns in [k0, k1)
double kr_work(const TileRanges &t, int r0, int nrows, int k0, int k1);

// Column intervals met by rows [r0, r0 + nrows) (kr indexed by 64-row tile from row 0),
// shifted by -c0 and clipped to [kbeg, kend): disjoint, ascending; returns 0..2.
// Cover of several tiles: the union of their first and of their second intervals.
__device__ __forceinline__ int kr_intervals(const KRange *kr, int r0, int nrows, int c0,
                                            int kbeg, int kend, int (&lo)[2], int (&hi)[2]) {
  const int t0 = r0 >> 6, t1 = (r0 + nrows - 1) >> 6;
  int a0 = 1 << 30, a1 = -(1 << 30), b0 = 1 << 30, b1 = -(1 << 30);
  for (int t = t0; t <= t1; ++t) {
    const KRange k = kr[t];
    if (k.a1 > k.a0) { a0 = min(a0, k.a0); a1 = max(a1, k.a1); }
    if (k.b1 > k.b0) { b0 = min(b0, k.b0); b1 = max(b1, k.b1); }
  }
  int n = 0;
  auto add = [&](int x0, int x1) {
    x0 = max(x0 - c0, kbeg);
    x1 = min(x1 - c0, kend);
    if (x1 > x0) { lo[n] = x0; hi[n] = x1; ++n; }
  };
  const bool ha = a1 > a0, hb = b1 > b0;
  if (ha && hb && b0 < a1 && b1 > a0) {
    add(min(a0, b0), max(a1, b1));
  } else if (ha && hb && b0 < a0) {
    add(b0, b1);
    add(a0, a1);
  } else {
    if (ha) add(a0, a1);
    if (hb) add(b0, b1);
  }
  return n;
}

// ---------------------------------------------------------------- GEMM
// Y[b] = alpha * A[b] (M x K, row-major, lda) * X[b] (K x N, row-major, ldx)
//        + beta * Z[b] (rows optionally re-indexed by zrow: Z row zrow[i] feeds Y row i)
// for batch b (pointer strides sA, sX, sY, sZ in elements).
struct GemmProb {
  const double *A; int64_t lda, sA;
  const double *X; int64_t ldx, sX;
  double *Y;       int64_t ldy, sY;
  const double *Z; int64_t ldz, sZ;
  const int *zrow;
  int M, N, K;
  double alpha, beta;
  // optional column ranges of A: kr[t] covers GEMM rows [64 t, 64 t + 64); columns are
  // A's own minus kr_c0 (filled by launch_gemm from the registry)
  const KRange *kr = nullptr;
  int kr_c0 = 0;
};

// Triangular solve with a CTA per column panel:
//   lower (fwd):  G Y = X      (G lower triangular, row-major, ldg)
//   upper (bwd):  U Y = X      (U upper triangular, row-major, ldg)
// jstart_blk > 0 restricts the coupling to a block-diagonal factor of block size
// jstart_blk (R_block): tiles outside a row's block are known zeros and skipped.
struct TrsmProb {
  const double *G; int64_t ldg;
  const double *X; int64_t ldx;
  double *Y;       int64_t ldy;
  int n, ncols;   // triangle order, number of right-hand-side columns
  int blk;        // 0 = dense triangle, else block-diagonal block size
  const std::vector<int> *segs = nullptr;   // else: block-diagonal with these block starts
  const double *dpack = nullptr;            // optional setup pack of the diagonal tiles
  const KRange *kr = nullptr;               // optional column ranges of G (64-row tiles)
};
struct Ctx;
// pack of the 64x64 diagonal tiles of an n x n triangular factor (ld = n), setup time
double *make_diag_pack(Ctx &c, const double *G, int n, bool upper);
void fill_diag_pack(Ctx &c, const double *G, int n, bool upper, double *pack);   // async
size_t diag_pack_doubles(int n);   // size of that pack

struct Ctx;

// ---------------------------------------------------------------- IC(0) factors (sparse.cu)
struct SparseFactor {
  int n = 0, nnz = 0;
  int *lrp = nullptr, *lci = nullptr, *urp = nullptr, *uci = nullptr;
  double *lv = nullptr, *uv = nullptr, *dinv = nullptr;
  // the same factor densified (row-major lower / upper, diagonal-tile packs) for the
  // DMMA TRSM: at n <= 4096 a dense solve of the banded factor beats the sparse one
  double *Gd = nullptr, *Gdt = nullptr, *Pd = nullptr, *Pdt = nullptr;
};

// ---------------------------------------------------------------- transport (comm.cu)
// Stream-ordered collectives of the time-window-sharded path.
struct Comm {
  int rank = 0, world = 1;
  struct P2P { void *buf; size_t count; int peer; bool send; };   // count in doubles
  virtual ~Comm() {}
  virtual void exchange(const std::vector<P2P> &ops, cudaStream_t st) = 0;
  virtual void allreduce_sum(double *buf, size_t count, cudaStream_t st) = 0;
  virtual void allgather(const double *send, double *recv, size_t count, cudaStream_t st) = 0;
};
struct LocalGroup;
Comm *make_comm(const wf4dvar_dist &d);
LocalGroup *local_group_create(int world);
void local_group_destroy(LocalGroup *g);
void nccl_unique_id(void *out128);

// Contiguous balanced partition of W windows over `world` ranks.
void partition(int W, int world, int rank, int *w_begin, int *w_end);

// Schedule of one L_hat^{-1} (transpose = 0) or L_hat^{-T} (transpose = 1)
// chain substitution with chains of length k over the global windows [0, WG),
// restricted to the local windows [w0, w1): step j updates the windows at chain
// position j (forward: w mod k == j; backward: j before the chain end); before the
// step the rank receives the neighbour's boundary window (forward: from rank-1 into
// the low halo; backward: from rank+1 into the high halo) and/or sends its own
// boundary window the other way.  Launches are (local first window, stride, count).
struct ChainStep {
  int j, recv, send, nl;
  int first[2], stride[2], count[2];
};
std::vector<ChainStep> chain_plan(int WG, int k, int w0, int w1, bool transpose);

void launch_gemm(Ctx &c, const GemmProb *probs, int nprob, int batch, double flops_hint = -1);
void launch_trsm(Ctx &c, const TrsmProb *probs, int nprob, bool upper);

// ---------------------------------------------------------------- context
struct Ctx {
  // problem.  W = number of LOCAL windows (the segment layout [len][W][m]); the
  // rank owns global windows [w0, w0 + W) of WG = N + 1.
  int s = 0, p = 0, N = 0, W = 0, m = 0;
  int w0 = 0, WG = 0;
  Comm *comm = nullptr;           // world > 1 only
  double *halo_lo = nullptr;      // [s][m]: state of global window w0 - 1 (from rank - 1)
  double *halo_hi = nullptr;      // [s][m]: state of global window w0 + W (from rank + 1)
  double *pack_lo = nullptr, *pack_hi = nullptr;   // [s][m] send staging
  double *gath = nullptr;         // [world][s][m] L_I scan totals
  int model = 0;
  int64_t ncol = 0;   // W*m columns of every segment
  int64_t n = 0;      // (2s+p)*W*m
  cudaStream_t st = nullptr;
  // fork/join streams: the three independent blocks of A and of P_D run concurrently
  cudaStream_t aux[2] = {nullptr, nullptr};
  cudaStream_t aux2 = nullptr;     // second column half of D_hat^{-1} (see dhat_inv)
  cudaStream_t kside = nullptr;    // MINRES: iteration j-1's update overlapping A z_j
  cudaEvent_t ev_kfork = nullptr, ev_kjoin = nullptr;
  cudaEvent_t ev_split[2] = {nullptr, nullptr};
  cudaEvent_t ev_fork = nullptr, ev_join[2] = {nullptr, nullptr};
  cudaEvent_t ev_halo = nullptr;   // apply_A's halo exchange done (aux[1] -> main)
  cudaStream_t cpy = nullptr;          // host path: block-wise H2D of apply_P's input
  cudaEvent_t ev_in[4] = {nullptr, nullptr, nullptr, nullptr};
  cudaEvent_t ev_chunk[4] = {nullptr, nullptr, nullptr, nullptr};   // host path column chunks
  bool aux_priority = true;       // env WF4DVAR_AUX_PRIORITY=0 disables (experiments)
  bool fork_on = true;            // fork/join concurrency of the operator blocks
  int device = 0;
  // device data
  double *B = nullptr, *Q = nullptr, *R = nullptr;
  int *H_idx = nullptr, *H_inv = nullptr;
  // general CSR H_i and its transpose (H^T as CSR over the s state rows)
  int *Hrp = nullptr, *Hcol = nullptr, *HTrp = nullptr, *HTcol = nullptr;
  double *Hval = nullptr, *HTval = nullptr;
  bool H_general = false;
  int heat_nsteps = 1;
  double heat_r = 0;
  double *Mdense = nullptr;       // [N][s][s]
  double *MdenseT = nullptr;      // [N][s][s] transposes
  double *traj = nullptr;         // [N][s][m]
  double *l96_sub = nullptr;      // [N][nsub][s][m] RK4 substep start states along traj
  double l96_F = 8, l96_dt = 0.025; int l96_nsub = 5;
  // heat stencil
  int heat_D = 0;                 // half width (0 => dense path)
  double heat_taps[65];           // taps[d + D], d in [-D, D]
  double heat_rho = 0, heat_gain = 0;   // recursive-filter form: M = gain * (1-rho S)^-1 (1-rho S^-1)^-1
  bool heat_iir = true;           // recursions (default) or the 2D+1-tap stencil
  // preconditioner
  wf4dvar_precond pc{};
  double *GB = nullptr, *GBt = nullptr, *GQ = nullptr, *GQt = nullptr;  // chol(D_hat) & transposes
  double *GR = nullptr, *GRt = nullptr;                                  // chol(R_hat base)
  double *PB = nullptr, *PBt = nullptr, *PQ = nullptr, *PQt = nullptr;  // diagonal-tile packs
  double *PR = nullptr, *PRt = nullptr;
  // explicit inverses (G G^T)^{-1} of D_hat's blocks and of R_hat (reading A32): the
  // preconditioner's solves become one DMMA GEMM each (nullptr: triangular solves)
  double *IB = nullptr, *IQ = nullptr, *IR = nullptr;
  SparseFactor icB, icQ, icR;     // IC(0) factors (pc.factor == WF4DVAR_FACTOR_ICHOL)
  double *Rdiag_inv = nullptr;                                           // [p]
  std::vector<TileRanges> tranges; // registered column ranges (banded covariances / factors)
  std::vector<int> rblk_starts;   // R_block (Algorithm 1): block starts + p (empty = uniform)
  std::vector<int> pvec_store;    // copy of the caller's pvec (pc.pvec points here)
  double *U_me = nullptr, *Kinv_me = nullptr; int r_me = 0;              // Woodbury
  double gamma_used = 0, T_used = 0;
  // workspaces (n doubles each unless noted)
  double *ws_t = nullptr;         // A+P intermediate / P scratch (segment-sized)
  double *ws_seg = nullptr;       // one s*ncol segment
  double *ws_lr = nullptr;        // low-rank scratch [r][ncol]
  double *outer_ws = nullptr;     // outer loop: rhs, dx, forecast
  double *dot_part = nullptr;     // partial sums
  int dot_part_cap = 0;
  double *hostbuf = nullptr;      // pinned
  double *dev_io_x = nullptr, *dev_io_y = nullptr, *dev_io_t = nullptr;
  // counters (per-window constituent products, Tables 7.2-7.3 / S5-S7)
  int64_t n_R = 0, n_Rhat_inv = 0, n_D = 0, n_Dhat_inv = 0, n_M = 0, n_A = 0, n_P = 0;
  int64_t launches = 0;
  struct Counters {
    int64_t v[8];
    Counters operator-(const Counters &o) const { Counters r; for (int i = 0; i < 8; ++i) r.v[i] = v[i] - o.v[i]; return r; }
    Counters operator+(const Counters &o) const { Counters r; for (int i = 0; i < 8; ++i) r.v[i] = v[i] + o.v[i]; return r; }
  };
  Counters counters() const { return Counters{{n_R, n_Rhat_inv, n_D, n_Dhat_inv, n_M, n_A, n_P, launches}}; }
  void set_counters(const Counters &k) {
    n_R = k.v[0]; n_Rhat_inv = k.v[1]; n_D = k.v[2]; n_Dhat_inv = k.v[3]; n_M = k.v[4];
    n_A = k.v[5]; n_P = k.v[6]; launches = k.v[7];
  }
  // CUDA graphs of the MINRES iteration (launch-bound sizes), cached across solves
  bool use_graphs = false;
  cudaStream_t own_st = nullptr;  // library stream for graph capture when st is the legacy stream
  cudaGraphExec_t mg_exec[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  Counters mg_delta[6];
  const void *mg_key[4] = {nullptr, nullptr, nullptr, nullptr};
  double mg_tol = -1, mg_mark = -1;
  bool mg_warm = false;            // an eager MINRES iteration ran since the last drop
  void drop_graphs() {
    for (auto &e : mg_exec)
      if (e) { cudaGraphExecDestroy(e); e = nullptr; }
    for (auto &k : mg_key) k = nullptr;
    mg_warm = false;
  }
  int gemm_cls = K_GEMM;          // profiling class of the next launch_gemm
  // stream-K GEMM: parked partial tiles and per-CTA publish flags, one set per stream
  struct SkState {
    cudaStream_t stream = nullptr; double *ws = nullptr; unsigned *flags = nullptr; size_t cap = 0;
    double *splitk = nullptr; size_t splitk_cap = 0;   // split-K partial tiles
    // dataflow TRSM (trsm.cu k_trsm_df): per (tile, panel) ready flags and the launch
    // epoch / finished-CTA counter pair
    unsigned *df_flags = nullptr; size_t df_cap = 0; unsigned *df_ep = nullptr;
  };
  std::vector<SkState> sk_states;
  // workspaces replaced by a larger one: captured MINRES graphs may still reference
  // them, so they are freed only with the context (freeing on growth left
  // cached graph execs pointing at freed memory)
  std::vector<void *> retired;
  Prof prof;
  std::string last_error;
  std::vector<void *> allocs;

  // persistent Krylov workspace arena (grown on demand, reused across solves)
  char *kws = nullptr;
  size_t kws_cap = 0, kws_used = 0;
  void kws_reset(size_t need) {
    if (need > kws_cap) {
      if (kws) cudaFree(kws);
      kws = nullptr;
      kws_cap = 0;
      if (cudaMalloc((void **)&kws, need) != cudaSuccess) throw Error{WF4DVAR_ENOMEM, "Krylov workspace"};
      kws_cap = need;
    }
    kws_used = 0;
  }
  template <class T> T *kws_take(size_t count) {
    size_t bytes = ((count * sizeof(T) + 255) / 256) * 256;
    if (kws_used + bytes > kws_cap) throw Error{WF4DVAR_ENOMEM, "Krylov workspace overflow"};
    T *p = (T *)(kws + kws_used);
    kws_used += bytes;
    return p;
  }
  int *hpin = nullptr;   // pinned host flags
  std::vector<cudaEvent_t> iter_events;
  cudaEvent_t ev_init = nullptr;  // end of the solver initialisation (report.seconds_init)
  cudaEvent_t iter_event(size_t i) {
    while (iter_events.size() <= i) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      iter_events.push_back(e);
    }
    return iter_events[i];
  }

  template <class T> T *alloc(size_t count) {
    void *ptr = nullptr;
    if (count == 0) count = 1;
    cudaError_t e = cudaMalloc(&ptr, count * sizeof(T));
    if (e != cudaSuccess) throw Error{WF4DVAR_ENOMEM, "cudaMalloc failed"};
    allocs.push_back(ptr);
    return (T *)ptr;
  }
  void prof_begin(int cls, double flops, double bytes, cudaEvent_t *ev);
  void prof_end(int cls, cudaEvent_t ev);
};

// Setup copies: ordered on the context stream and complete on return.  (A plain
// cudaMemcpy from pageable host memory may return before the DMA lands and is
// ordered only on the legacy default stream, so a later kernel on a non-blocking
// library stream could read a half-written buffer.)
inline cudaError_t memcpy_sync(Ctx &c, void *dst, const void *src, size_t bytes,
                               cudaMemcpyKind kind) {
  cudaError_t e = cudaMemcpyAsync(dst, src, bytes, kind, c.st);
  if (e != cudaSuccess) return e;
  return cudaStreamSynchronize(c.st);
}

// Run the enclosed launches on another stream of the context.
// While profiling, everything stays on the main stream: per-launch event times of
// concurrently running kernels would overlap and misstate each kernel's rate.
struct OnStream {
  Ctx &c; cudaStream_t saved;
  OnStream(Ctx &c_, cudaStream_t s) : c(c_), saved(c_.st) { if (!c.prof.on && c.fork_on) c.st = s; }
  ~OnStream() { c.st = saved; }
};
void fork(Ctx &c);   // aux streams wait for the work enqueued so far on c.st
void join(Ctx &c);   // c.st waits for the aux streams

// RAII helper that brackets one launch with profiling events.
// It also opens an NVTX range named after the kernel class (no-op unless a tool
// such as ncu is attached: `ncu --nvtx --nvtx-include "gemm_dmma/"` then selects
// exactly the launches of one class).
struct LaunchScope {
  Ctx &c; int cls; cudaEvent_t ev = nullptr;
  LaunchScope(Ctx &c_, int cls_, double flops, double bytes) : c(c_), cls(cls_) {
    nvtxRangePushA(kClassName[cls]);
    c.prof_begin(cls, flops, bytes, &ev);
  }
  ~LaunchScope() {
    c.prof_end(cls, ev);
    nvtxRangePop();
  }
};

// ---------------------------------------------------------------- ops
// out_w = base_w + sign * M_w in_{w-1}      (transpose == false)
// out_w = base_w + sign * M_{w+1}^T in_{w+1} (transpose == true)
// for windows w = w_first + t * w_step, t in [0, nw); a window whose source
// w-1 / w+1 is outside [0, W) gets out_w = base_w.  When add2 != nullptr the
// kernel also adds add2[row_map[i]] (row_map[i] < 0: nothing) -- used to fuse
// the H^T scatter of A's third block.  in, base, out are [s][W][m] segments;
// out may alias base (and in, if the window sets do not overlap).
void model_step(Ctx &c, bool transpose, double sign, const double *in, const double *base,
                double *out, int w_first, int w_step, int nw, const double *add2 = nullptr,
                const int *row_map = nullptr);

// Lorenz-96 tangent-linear / adjoint window step (same contract as model_step).
void l96_step(Ctx &c, bool transpose, double sign, const double *in, const double *base,
              double *out, int w_first, int w_step, int nw, const double *add2,
              const int *row_map);

// Lorenz-96 chain step over two window groups in one launch (in place on z, sign +1):
// windows f0 + i s0 (i < n0) and f1 + i (i < n1).
void l96_step2(Ctx &c, bool transpose, double *z, int f0, int s0, int n0, int f1, int n1);

// Lorenz-96: recompute c.l96_sub from c.traj (after every trajectory change).
void l96_substates(Ctx &c);

// L-hat^{-1} (forward chains) / L-hat^{-T} (backward chains) in place on z.
void lhat_solve(Ctx &c, bool transpose, double *z);

// vector kernels
void copy(Ctx &c, double *dst, const double *src, int64_t n);
void scale_rows(Ctx &c, double *y, const double *x, const double *row_scale, int rows);
void lowrank_correct(Ctx &c, double *y, const double *x);
void rhat_inv(Ctx &c, const double *x2, double *y2);
void dhat_inv(Ctx &c, const double *x1, double *y1);

// world > 1: in-place sum of per-RHS partial inner products over the ranks
void allreduce(Ctx &c, double *buf, size_t count);
// pack local window wl of an [s][W][m] segment into a contiguous [s][m] buffer
void pack_window(Ctx &c, double *dst, const double *seg, int wl);

// y[i][c] (+)= sum_k val[k] x[col[k]][c] over rows i < nrows, all ld columns (CSR)
void csr_apply(Ctx &c, double *y, const double *x, const int *rowptr, const int *col,
               const double *val, int nrows, bool accumulate);

// host_y != nullptr: every output block is copied to host_y on its own stream as soon
// as it is computed (the host path, overlapping the D2H with the remaining blocks)
void apply_A(Ctx &c, const double *x, double *y, double *host_y = nullptr);
// host_x != nullptr: x is the library's device staging buffer, filled from host_x block
// by block (D_hat / first block first) on the copy stream; each block's solve starts
// when its own input has landed
void apply_P(Ctx &c, const double *x, double *y, const double *host_x = nullptr);

// Gauss-Newton outer loops (outer.cu)
void outer_loop(Ctx &c, const double *xb, const double *y, double *x, int n_outer,
                const wf4dvar_solve_opts &inner, int32_t *inner_iters, double *dx_norm2,
                double *res_norm2);

// spectral suite (spectral.cu)
void lanczos(Ctx &c, int op, const double *v0, int steps, double *ritz_min, double *ritz_max,
             double *alpha_out, double *beta_out);

// Krylov
void solve(Ctx &c, const double *rhs, double *x, const wf4dvar_solve_opts &o, wf4dvar_report *rep);

// launch geometry of the per-RHS reductions over a [n/m][m] view (see vec.cu)
struct RedGrid { int gx, gy, RB; int64_t rows, rpb; };
RedGrid red_grid(const Ctx &c, int64_t n);
// fixed-order final reduction of per-block partials (part[(b*nd + d)*m + r]) -> out[d*m + r]
void reduce_final(Ctx &c, const double *part, int nparts, int nd, double *out);

// batched dots: out[j*m + r] = sum_{f % m == r} a_j[f] * b_j[f], j < nd (<= 4)
void dots(Ctx &c, int nd, const double *const *a, const double *const *b, int64_t n,
          double *out);

void setup_precond(Ctx &c);
void make_ichol(Ctx &c, const std::vector<double> &A, int n, const char *name, SparseFactor &f);
void ichol_solve(Ctx &c, const SparseFactor &f, const double *x, double *y, int c0, int ncols,
                 const SparseFactor *g = nullptr, int nsplit = 0);
std::vector<int> algorithm1_blocks(const std::vector<double> &R, int p, const std::vector<int> &pvec,
                                   double tol, int maxsize, int numproc);
void free_precond(Ctx &c);
void setup_model(Ctx &c, const wf4dvar_problem &p);

}  // namespace wf
