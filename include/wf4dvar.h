/*
 * wf4dvar.h -- C ABI of the B200-native (sm_100a, FP64) hot path of
 * Tabeart & Pearson, "Saddle point preconditioners for weak-constraint 4D-Var"
 * (arXiv 2105.06975).  Citations "P:Lnnn" are lines of that paper's PAPER.md.
 *
 * What the library computes (one call = the whole batch of m right-hand sides):
 *   apply_A : y = A x, A = [[D, 0, L], [0, R, H], [L^T, H^T, 0]]        Eq. 2.2,
 *             matrix-free as c1 = D x1 + L x3, c2 = R x2 + H x3,
 *             c3 = L^T x1 + H^T x2
 *             D = blkdiag(B, Q_1..Q_N), R = blkdiag(R_0..R_N),
 *             H = blkdiag(H_0..H_N); L unit lower block-bidiagonal
 *             with -M_w on the sub-diagonal (Eq. 2.3).
 *   apply_P : y = P^{-1} x for
 *             P_D = blkdiag(D_hat, R_hat, S_hat), S_hat = L_hat^T D^{-1} L_hat
 *               -> (D_hat^{-1} x1, R_hat^{-1} x2, L_hat^{-1} D L_hat^{-T} x3)
 *             P_I = [[D, 0, L_hat], [0, R_hat, 0], [L_hat^T, 0, 0]]
 *               -> c1 = L_hat^{-T} x3, c2 = R_hat^{-1} x2, c3 = L_hat^{-1}(x1 - D c1)
 *
 *             with L_hat in {L_0, L_I, L_M(k) (Def. 4.1,
 *             P:L255-263), L}, R_hat in {R_diag, R_block (Alg. 1),
 *             R_RR (Alg. 2), R_ME (Alg. 3, applied as a Woodbury low-rank update of
 *             the Cholesky solve), R}, D_hat = D or D + delta I.
 *   solve   : batched preconditioned MINRES (P_D; 2-norm residual criterion,
 *             P:L674) or right-preconditioned restarted GMRES (P_I; relative
 *             2-norm residual) from x0 = 0, independently per RHS.
 *
 * Vector layout (every x, y, rhs): ONE contiguous device buffer of
 *   n_local = (2s+p) * W_local * m doubles, W_local = number of local windows,
 * holding three segments, each [len][W_local][m] row-major (RHS index fastest):
 *   delta_eta [s][W][m] | delta_nu [p][W][m] | delta_x [s][W][m].
 * Covariance products over all windows are therefore single GEMMs
 * C (len x len) * X (len x W*m).
 *
 * Ownership: wf4dvar_create deep-copies every host input (the caller may free
 * them on return).  The context owns device copies, Cholesky factors and
 * workspaces.  x, y, rhs are caller-owned DEVICE buffers (e.g. torch float64
 * CUDA tensors) unless an entry point says HOST; report arrays are caller-owned
 * host memory.  x and y must not alias.
 *
 * Streams: apply_A / apply_P / apply_AP enqueue on dist->stream and return
 * without a host synchronisation; wf4dvar_solve* are synchronous.
 *
 * Errors: every entry point returns wf4dvar_status and never throws.
 *   WF4DVAR_EINVAL   bad shape / enum / pointer (e.g. k outside [1, N+1], H_idx
 *                    not strictly increasing in [0, s), p not divisible by block).
 *   WF4DVAR_ENOTSPD  Cholesky breakdown of D_hat, R_hat (message names the block).
 *   WF4DVAR_EINDEF   MINRES met z^T v < 0 (P^{-1} must be SPD).
 *   WF4DVAR_ENOCONV  maxit reached; x and the report are still valid.
 *   WF4DVAR_ECUDA / WF4DVAR_ENOMEM  CUDA runtime / allocation failure.
 * A failed call leaves the context destroyable; wf4dvar_last_error(ctx) returns a
 * message valid until the next call on that context (NULL ctx: last create error).
 *
 * Determinism: no atomics in any reduction; for a fixed problem and device the
 * outputs are bitwise reproducible run to run.  One context per host thread.
 */
#ifndef WF4DVAR_H
#define WF4DVAR_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct wf4dvar_ctx_s *wf4dvar_ctx;

typedef enum {
  WF4DVAR_OK = 0,
  WF4DVAR_EINVAL = 1,
  WF4DVAR_ENOTSPD = 2,
  WF4DVAR_EINDEF = 3,
  WF4DVAR_ENOCONV = 4,
  WF4DVAR_ECUDA = 5,
  WF4DVAR_ENCCL = 6,
  WF4DVAR_ENOMEM = 7
} wf4dvar_status;

/* Model term M_w (maps window w-1 to w, w = 1..N). */
typedef enum {
  WF4DVAR_M_DENSE = 0, /* M_dense[w-1] given as dense s x s row-major              */
  WF4DVAR_M_HEAT = 1,  /* M = (I - r Lap)^{-1}, Lap = periodic second difference
                          (BJ.c0-c4); applied as its exact circulant stencil        */
  WF4DVAR_M_L96 = 2,   /* tangent linear of l96_nsub RK4 steps of Lorenz-96
                           along l96_traj, recomputed matrix-free
                          (the create call stores the RK4 substep start states
                          on the device: N * l96_nsub * s * m doubles)            */
  WF4DVAR_M_HEAT_EXPLICIT = 3 /* the paper's own heat model: M = M_dt^n,
                          M_dt = forward-Euler Dirichlet step (first/last rows zero,
                          interior (r, 1-2r, r)), n = heat_nsteps <= 8 per window,
                          r = heat_r; applied as n fused 3-point sweeps          */
} wf4dvar_model;

/* B, Q, R (and the triangular factors built from them) are stored densely on the
 * device.  Compact-support matrices (e.g. the modified SOAR of P:L566-570, zero for
 * circular lag >= maxval) are detected at create / set_precond time: the exact-zero
 * 64 x 16 tiles are never read by the covariance products and triangular solves
 * (results bit-identical to the dense loops; env WF4DVAR_BANDED=0 disables it). */
typedef struct {
  int32_t s, p, N, m;      /* state size, obs per window, N (W = N+1 windows), RHS   */
  const double *B;         /* [s*s] host, SPD, row-major                            */
  const double *Q;         /* [s*s] host, SPD, shared by windows 1..N       */
  const double *R;         /* [p*p] host, SPD, shared by windows 0..N       */
  const int32_t *H_idx;    /* [p] host: (H_w x)_j = x[H_idx[j]], strictly increasing */
  int32_t model;           /* wf4dvar_model                                         */
  const double *M_dense;   /* DENSE: [N*s*s] host                                   */
  double heat_r;           /* HEAT: r > 0                                           */
  const double *l96_traj;  /* L96: [N][s][m] host, start state of window w-1 for M_w */
  double l96_F, l96_dt;    /* L96: forcing, RK4 step                                */
  int32_t l96_nsub;        /* L96: RK4 steps per window                             */
  int32_t heat_nsteps;     /* HEAT_EXPLICIT: model steps per window, 1..8            */
  /* General observation operator H_i (e.g. the paper's 5-point smoothed
     observations): CSR p x s, host, same for every window.  When H_rowptr != NULL
     it replaces H_idx (which may then be NULL); column indices in [0, s). */
  const int32_t *H_rowptr; /* [p+1]                                                  */
  const int32_t *H_col;    /* [H_rowptr[p]]                                           */
  const double *H_val;     /* [H_rowptr[p]]                                           */
} wf4dvar_problem;

typedef enum { WF4DVAR_PD = 0, WF4DVAR_PI = 1 } wf4dvar_shape;
typedef enum { WF4DVAR_L0 = 0, WF4DVAR_LI = 1, WF4DVAR_LM = 2, WF4DVAR_LEXACT = 3 } wf4dvar_lhat;
typedef enum {
  WF4DVAR_RDIAG = 0, WF4DVAR_RBLOCK = 1, WF4DVAR_RRR = 2, WF4DVAR_RME = 3, WF4DVAR_REXACT = 4
} wf4dvar_rhat;

typedef struct {
  int32_t shape;      /* wf4dvar_shape                                              */
  int32_t lhat;       /* wf4dvar_lhat                                               */
  int32_t k;          /* L_M(k): 1 <= k <= N+1 (ignored otherwise)                  */
  int32_t rhat;       /* wf4dvar_rhat                                               */
  double gamma;       /* R_RR: gamma < 0 => lambda_min(R)                   */
  double T;           /* R_ME: T < 0 => smallest eigenvalue strictly above lambda_min
                         (relative gap 1e-10; reading A6)                  */
  int32_t block;      /* R_BLOCK: uniform block size (last block ragged), Alg. 1
                         with every cut applied (reading A7)                         */
  double dhat_ridge;  /* 0 => D_hat = D; > 0 => D_hat = D + ridge I         */
  /* R_BLOCK by Algorithm 1 in full, used when pvec != NULL (then
     `block` is ignored): pvec[0..npvec) block sizes summing to p; every first
     super-diagonal block with scaled Frobenius norm normvec(j) < block_tol is cut
     (block_tol = +inf cuts all: uniform blocks); maxsize > 0 splits the largest
     block in two if it is larger; numproc > 0 merges the two smallest adjacent
     blocks if there are more than numproc blocks, or splits the largest if there
     are fewer than numproc - 2 (readings A7, A25).  At most 512 blocks; pvec is
     copied. */
  const int32_t *pvec;
  int32_t npvec;
  double block_tol;
  int32_t maxsize, numproc;
  /* Factors of D_hat and R_hat: WF4DVAR_FACTOR_CHOL (0, default)
     dense Cholesky, applied as DMMA TRSM (reading A4); WF4DVAR_FACTOR_ICHOL (1) the
     paper's incomplete Cholesky with zero fill on the non-zero pattern (Matlab ichol
     'nofill'): the preconditioner blocks become L L^T, applied as
     sparse triangular solves.  For compact-support covariances; not with R_ME. */
  int32_t factor;
  /* How dense D_hat / R_hat blocks (n >= 256, exact Cholesky factors, not banded) are
     applied.  WF4DVAR_APPLY_TRSM (0, default): the two triangular solves with the
     Cholesky factors, backward stable (the per-block parity test
     checks ||C y - x|| / (||C|| ||y||) <= 1e-14).  WF4DVAR_APPLY_INVERSE (1): one GEMM
     with the setup-time explicit inverse (G G^T)^{-1} (reading A32); the
     same flops at GEMM rate, but NOT backward stable (backward error up to ~kappa u on
     smooth vectors), which costs Krylov iterations.  Env WF4DVAR_EXPLICIT_INV=0/1
     overrides this field. */
  int32_t apply_mode;
} wf4dvar_precond;
typedef enum { WF4DVAR_APPLY_TRSM = 0, WF4DVAR_APPLY_INVERSE = 1 } wf4dvar_apply_mode;
typedef enum { WF4DVAR_FACTOR_CHOL = 0, WF4DVAR_FACTOR_ICHOL = 1 } wf4dvar_factor;

/* Time-window sharding ("the model propagations M_i can be
 * run in parallel", P:L253 the parallel-in-time L_M(k)).  With world > 1 rank g
 * owns the contiguous global windows [w_begin, w_end) of wf4dvar_partition, all
 * vectors are rank-local ((2s+p)*(w_end-w_begin)*m doubles, same segment layout),
 * B, Q, R, H and the model data are passed in full on every rank.  Per A apply
 * two one-state halos move ([s][m] doubles: x3 of the last window to rank+1 for L,
 * x1 of the first window to rank-1 for L^T); L_hat chains that cross a rank
 * boundary hand their running state over once per crossing (none when k divides
 * every rank's w_begin); L_I uses an allgather of per-rank window sums; the
 * Krylov inner products are summed over the ranks (allreduce of [nd][m] doubles).
 * Every rank calls create / apply / solve / destroy in the same order. */
typedef enum {
  WF4DVAR_TRANSPORT_NONE = 0,  /* world must be 1                                          */
  WF4DVAR_TRANSPORT_NCCL = 1,  /* one process per GPU; NCCL (libnccl.so.2, dlopen'ed)      */
  WF4DVAR_TRANSPORT_LOCAL = 2  /* world ranks = host threads of one process sharing a
                                  wf4dvar_local_group (single-device driving of the
                                  sharded path; stream-ordered, no kernel waits on another) */
} wf4dvar_transport;

typedef struct {
  int32_t rank, world; /* 0 <= rank < world; world <= N+1                           */
  int32_t device;      /* CUDA device ordinal                                       */
  void *stream;        /* cudaStream_t the library enqueues on (NULL = default)     */
  int32_t transport;   /* wf4dvar_transport (ignored when world == 1)               */
  const void *nccl_id; /* NCCL: the 128-byte ncclUniqueId rank 0 obtained from
                          wf4dvar_nccl_unique_id, broadcast by the caller           */
  void *local_group;   /* LOCAL: from wf4dvar_local_group_create(world)             */
} wf4dvar_dist;

typedef enum { WF4DVAR_MINRES = 0, WF4DVAR_GMRES = 1 } wf4dvar_solver;

typedef struct {
  int32_t solver;      /* wf4dvar_solver                                            */
  double tol;          /* relative 2-norm residual target, per RHS                  */
  int32_t maxit;       /* iteration cap (MINRES iterations / GMRES Arnoldi steps)    */
  int32_t restart;     /* GMRES restart length (<= 0: maxit, i.e. full GMRES)        */
  double mark_tol;     /* report the first time every RHS is <= mark_tol (e.g. 1e-8) */
  int32_t check_every; /* host polls convergence every this many iterations (>= 1)   */
} wf4dvar_solve_opts;

typedef struct {
  int32_t *iters;      /* [m] or NULL: iterations to convergence per RHS             */
  double *relres;      /* [m] or NULL: recurrence relative residual at exit         */
  uint8_t *converged;  /* [m] or NULL                                               */
  double *history;     /* [(maxit+1)*m] or NULL: relres per iteration (row = iter)   */
  double seconds;      /* solve wall time (device events)                           */
  double seconds_to_mark; /* time until every RHS <= mark_tol (-1 if never)          */
  int32_t iters_to_mark;  /* iteration at which that happened (-1 if never)          */
  int64_t n_apply_A, n_apply_P;
  int64_t n_R, n_Rhat_inv, n_D, n_Dhat_inv, n_M; /* per-window constituent products,
                          counted as in Tables 7.2-7.3, S5-S7 (R_diag not counted)  */
  double seconds_init;   /* part of `seconds` spent before the first iteration (MINRES:
                            x = 0, r = b, z_1 = P^{-1} b and the first inner products) */
} wf4dvar_report;

wf4dvar_status wf4dvar_create(const wf4dvar_problem *prob, const wf4dvar_precond *pc,
                              const wf4dvar_dist *dist, wf4dvar_ctx *out);
/* Re-run the preconditioner setup only (factorisations of D_hat / R_hat). */
wf4dvar_status wf4dvar_set_precond(wf4dvar_ctx ctx, const wf4dvar_precond *pc);
wf4dvar_status wf4dvar_destroy(wf4dvar_ctx ctx);
wf4dvar_status wf4dvar_local_windows(wf4dvar_ctx ctx, int32_t *w_begin, int32_t *w_end);
wf4dvar_status wf4dvar_vector_len(wf4dvar_ctx ctx, int64_t *n_local);

/* y = A x (device buffers, x != y). */
wf4dvar_status wf4dvar_apply_A(wf4dvar_ctx ctx, const double *x, double *y);
/* y = P^{-1} x (P_D or P_I per the context's preconditioner; device buffers). */
wf4dvar_status wf4dvar_apply_P(wf4dvar_ctx ctx, const double *x, double *y);
/* One "A+P apply" (the unit of the throughput metric): t = P^{-1} x, y = A t.
   All three are device buffers of n_local doubles and must not alias. */
wf4dvar_status wf4dvar_apply_AP(wf4dvar_ctx ctx, const double *x, double *t, double *y);
/* Same with HOST x_host / y_host (pinned recommended): H2D copy, A+P, D2H copy;
   synchronous. */
wf4dvar_status wf4dvar_apply_AP_host(wf4dvar_ctx ctx, const double *x_host, double *y_host);

/* Batched solve A x = rhs from x0 = 0 (device buffers). Synchronous. */
wf4dvar_status wf4dvar_solve(wf4dvar_ctx ctx, const double *rhs, double *x,
                             const wf4dvar_solve_opts *opts, wf4dvar_report *rep);
/* Same with HOST rhs / x: the copies are inside the call (end-to-end path). */
wf4dvar_status wf4dvar_solve_host(wf4dvar_ctx ctx, const double *rhs_host, double *x_host,
                                  const wf4dvar_solve_opts *opts, wf4dvar_report *rep);

/* Gauss-Newton outer loops of incremental 4D-Var.
   Each of n_outer iterations, from the iterate x = (x_0..x_N): re-linearise (for L96
   the tangent-linear trajectory becomes x itself: M_w about x_{w-1}), form the
   right-hand side b_0 = x_b - x_0, b_w = M_w(x_{w-1}) - x_w (nonlinear forecast),
   d_w = y_w - H x_w, third block 0 (reading A3), solve the saddle system with
   `inner`, and update x += delta x.  Device buffers: xb [s][m] (used by the rank
   owning window 0), y [p][W_local][m], x [s][W_local][m] (in: first guess, out:
   final iterate).  Optional host outputs [n_outer*m] (row = outer iteration):
   inner iteration counts, ||delta x||^2 and ||(b, d)||^2 per RHS.  An unconverged
   inner loop still updates x.  Synchronous. */
wf4dvar_status wf4dvar_outer_loop(wf4dvar_ctx ctx, const double *xb, const double *y, double *x,
                                  int32_t n_outer, const wf4dvar_solve_opts *inner,
                                  int32_t *inner_iters, double *dx_norm2, double *res_norm2);

/* Spectral suite: extreme eigenvalues by batched Lanczos, one
   independent run per RHS column, `steps` steps from the start vector v0 (device,
   full vector layout of n_local doubles; OP_LHAT uses only its delta_x segment).
     OP_PA    eigenvalues of P_D^{-1} A (Theorem 3.1): preconditioned
              Lanczos in the P_D inner product (the recurrence of MINRES);
              the context's preconditioner must be P_D.
     OP_LHAT  eigenvalues of L_hat^{-T} L^T L L_hat^{-1} (Section 4, Prop. 4.4/4.5,
              Supp. Tables S2/S3) on the state segment.
   ritz_min / ritz_max: [m] host (extreme Ritz values: converge to the extreme
   eigenvalues as steps grows); alpha / beta: optional [steps*m] host (row = step)
   tridiagonal entries.  Synchronous.  No reorthogonalisation. */
typedef enum { WF4DVAR_OP_PA = 0, WF4DVAR_OP_LHAT = 1 } wf4dvar_spectral_op;
wf4dvar_status wf4dvar_lanczos(wf4dvar_ctx ctx, int32_t op, const double *v0, int32_t steps,
                               double *ritz_min, double *ritz_max, double *alpha, double *beta);

/* Instrumentation.  When enabled, the library brackets every launch of each
   kernel class with CUDA events on the launching stream; read() returns per
   class: launches, total milliseconds, algorithmic flops and bytes. */
typedef struct {
  char name[32];
  int64_t launches;
  double ms;
  double flops;
  double bytes;
} wf4dvar_kstat;
wf4dvar_status wf4dvar_profile_enable(wf4dvar_ctx ctx, int32_t enable);
wf4dvar_status wf4dvar_profile_read(wf4dvar_ctx ctx, wf4dvar_kstat *out, int32_t max_n,
                                    int32_t *n_out);
/* Total number of kernel launches issued by this context so far. */
int64_t wf4dvar_launch_count(wf4dvar_ctx ctx);

/* ---- sharding helpers (host only; no device, no context needed) ---- */
/* The contiguous balanced partition: rank g of `world` owns global windows
   [w_begin, w_end), sizes differing by at most one (earlier ranks larger). */
wf4dvar_status wf4dvar_partition(int32_t W, int32_t world, int32_t rank, int32_t *w_begin,
                                 int32_t *w_end);
/* Schedule of the L_hat^{-1} (transpose = 0) / L_hat^{-T} (transpose = 1) chain
   substitution (Lemma 4.2) for chains of length k (k = N+1 for the
   exact L) restricted to the windows [w_begin, w_end) of W: entry j (j = 1..)
   updates the windows at chain position j -- forward z_w = r_w + M_w z_{w-1},
   backward z_w = r_w + M_{w+1}^T z_{w+1} -- in nl launches of (first local
   window, stride, count); recv = 1 means the neighbour's boundary state is
   received into the halo first (forward from rank-1, backward from rank+1),
   send = 1 that this rank's boundary window is sent the other way first.
   Writes at most max_steps entries; *n_steps = the full count. */
typedef struct {
  int32_t j, recv, send, nl;
  int32_t first[2], stride[2], count[2];
} wf4dvar_chain_step;
wf4dvar_status wf4dvar_chain_plan(int32_t W, int32_t k, int32_t w_begin, int32_t w_end,
                                  int32_t transpose, wf4dvar_chain_step *out,
                                  int32_t max_steps, int32_t *n_steps);
/* Algorithm 1 block structure of R_block, host only: R [p*p] host
   row-major, pvec / block_tol / maxsize / numproc as in wf4dvar_precond.  Writes
   the block starts followed by p (at most max_out entries) to starts_out and the
   entry count (number of blocks + 1) to *n_out.  This is the setup step
   wf4dvar_create runs for R_BLOCK with pvec != NULL. */
wf4dvar_status wf4dvar_rblock_plan(const double *R, int32_t p, const int32_t *pvec, int32_t npvec,
                                   double block_tol, int32_t maxsize, int32_t numproc,
                                   int32_t *starts_out, int32_t max_out, int32_t *n_out);
/* NCCL: rank 0 fills out[128] with a fresh ncclUniqueId (to broadcast). */
wf4dvar_status wf4dvar_nccl_unique_id(void *out128);
/* LOCAL transport: one group shared by `world` contexts of this process. Destroy
   it after every context that uses it. */
wf4dvar_status wf4dvar_local_group_create(int32_t world, void **out);
wf4dvar_status wf4dvar_local_group_destroy(void *group);

const char *wf4dvar_last_error(wf4dvar_ctx ctx);
/* Library build string (compile arch, version). */
const char *wf4dvar_version(void);

#ifdef __cplusplus
}
#endif
#endif /* WF4DVAR_H */
