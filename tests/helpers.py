"""Shared test helpers: run the CPU oracle column by column in library layout."""
import numpy as np

from oracle.models import model_matrices
from oracle.saddle import Precond, Saddle
from synth.layout import from_paper_order, to_paper_order

PC_KEYS = ("shape", "lhat", "k", "rhat", "gamma", "T", "block", "ridge")


def oracle_precond(pc):
    d = dict(pc)
    return Precond(shape=d.get("shape", "PD"), lhat=d.get("lhat", "LM"), k=d.get("k", 4) or 1,
                   rhat=d.get("rhat", "exact"), gamma=d.get("gamma", -1.0), T=d.get("T", -1.0),
                   block=d.get("block", 0), ridge=d.get("ridge", 0.0),
                   pvec=tuple(d["pvec"]) if d.get("pvec") is not None else None,
                   block_tol=d.get("block_tol", float("inf")), maxsize=d.get("maxsize", 0),
                   numproc=d.get("numproc", 0), factor=d.get("factor", "chol"))


class OracleCols:
    """Per-RHS-column oracle saddles (shared M for heat/dense, per column for L96)."""

    def __init__(self, prob, cols=None):
        self.prob = prob
        self.cols = list(range(prob.m)) if cols is None else list(cols)
        shared = None if prob.model == "l96" else model_matrices(prob, 0)
        self.sad = {c: Saddle(prob, col=c, Ms=shared) for c in self.cols}

    def paper(self, vec):
        return to_paper_order(vec, self.prob.s, self.prob.p, self.prob.W, self.prob.m)

    def apply_A(self, vec):
        P = self.paper(vec)
        return {c: self.sad[c].apply_A(P[c]) for c in self.cols}

    def apply_P(self, pc, vec):
        P = self.paper(vec)
        opc = oracle_precond(pc)
        return {c: self.sad[c].apply_Pinv(opc, P[c]) for c in self.cols}


def rel_err_cols(gpu_vec, oracle_dict, prob):
    P = to_paper_order(gpu_vec, prob.s, prob.p, prob.W, prob.m)
    return {c: np.linalg.norm(P[c] - v) / max(np.linalg.norm(v), 1e-300)
            for c, v in oracle_dict.items()}


def seeded_vec(n, seed):
    return np.random.Generator(np.random.PCG64(seed)).standard_normal(n)


# ---------------------------------------------------------------------------------
# Per-block parity of a preconditioner apply.  P^{-1} x is three
# independently computed blocks:
#   P_D:  (D_hat^{-1} x1 | R_hat^{-1} x2 | S_hat^{-1} x3 = L_hat^{-1} D L_hat^{-T} x3)
#   P_I:  (c1 = L_hat^{-T} x3 | R_hat^{-1} x2 | c3 = L_hat^{-1}(x1 - D c1))
# Product-only blocks (no solve with an SPD block) must match the oracle to
# `prod_tol` (1e-12).  Solve blocks (D_hat^{-1}, R_hat^{-1} other than R_diag) must
# have forward error <= max(1e-12, 10 kappa(C_hat) u) AND backward error
# ||C_hat y - x|| / (||C_hat||_2 ||y||) <= 1e-14 per window -- the backward error is
# independent of the implementation, so it also bites where kappa u is large.  The
# backward residual is formed in extended precision (numpy longdouble, 64-bit
# mantissa), so the check's own rounding (~ n * 5e-20) is far below 1e-14.
U64 = 2.220446049250313e-16
BWD_TOL = 1e-14


def _segments(v, s, p, W):
    a = s * W
    return v[:a].reshape(W, s), v[a:a + p * W].reshape(W, p), v[a + p * W:].reshape(W, s)


def _spd_cond(C, cache, key, prob):
    key = (id(prob),) + key    # the problem object is kept alive in the entry (no id reuse)
    if key not in cache:
        ev = np.linalg.eigvalsh(C)
        cache[key] = (ev[-1] / ev[0], ev[-1], prob)
    return cache[key][:2]


def block_parity(prob, pc, x_lib, y_lib, ora, cols, windows=None, prod_tol=1e-12,
                 cache=None):
    """Per-block errors of y_lib = P^{-1} x_lib (library layout) against the oracle
    on the RHS columns `cols`.  Returns a list of failure strings (empty = pass) and
    a dict of the worst errors per block, for printing."""
    cache = {} if cache is None else cache
    s, p, W, m = prob.s, prob.p, prob.W, prob.m
    opc = oracle_precond(pc)
    X = to_paper_order(x_lib, s, p, W, m)
    Y = to_paper_order(y_lib, s, p, W, m)
    fails, worst = [], {}
    wins = sorted(set(range(W) if windows is None else [w % W for w in windows]))

    def note(name, val):
        worst[name] = max(worst.get(name, 0.0), val)

    for c in cols:
        sad = ora.sad[c]
        ref = sad.apply_Pinv(opc, X[c])
        x1, x2, x3 = _segments(X[c], s, p, W)
        g1, g2, g3 = _segments(Y[c], s, p, W)
        o1, o2, o3 = _segments(ref, s, p, W)
        rel = lambda a, b: np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)
        # --- R_hat^{-1} x2 (both shapes)
        if pc.get("rhat", "exact") == "diag":
            e = rel(g2, o2)
            note("Rhat_inv(diag) fwd", e)
            if e > prod_tol:
                fails.append(f"col {c} R_diag^-1 fwd {e:.2e} > {prod_tol:.0e}")
        else:
            Rh = sad.rhat_matrix(opc)
            kap, lmax = _spd_cond(Rh, cache, ("R",) + tuple(sorted(pc.items())), prob)
            tol = max(1e-12, 10 * kap * U64)
            e = rel(g2, o2)
            note("Rhat_inv fwd", e)
            if e > tol:
                fails.append(f"col {c} R_hat^-1 fwd {e:.2e} > {tol:.2e} (kappa {kap:.2e})")
            Rl = Rh.astype(np.longdouble)
            for w in wins:
                r = Rl @ g2[w].astype(np.longdouble) - x2[w].astype(np.longdouble)
                b = float(np.linalg.norm(r.astype(np.float64))) / (lmax * np.linalg.norm(g2[w]))
                note("Rhat_inv bwd", b)
                if b > BWD_TOL:
                    fails.append(f"col {c} w {w} R_hat^-1 bwd {b:.2e} > {BWD_TOL:.0e}")
        if pc.get("shape", "PD") == "PD":
            # --- D_hat^{-1} x1 (window 0: B_hat, windows >= 1: Q_hat)
            for w0, ws in ((0, [0]), (1, list(range(1, W)))):
                if not ws:
                    continue
                Dh = sad.dhat_matrix(opc, w0)
                kap, lmax = _spd_cond(Dh, cache, ("D", w0, pc.get("ridge", 0.0)), prob)
                tol = max(1e-12, 10 * kap * U64)
                e = rel(g1[ws], o1[ws])
                note("Dhat_inv fwd", e)
                if e > tol:
                    fails.append(f"col {c} D_hat^-1 (w{w0}) fwd {e:.2e} > {tol:.2e} "
                                 f"(kappa {kap:.2e})")
                Dl = Dh.astype(np.longdouble)
                for w in [v for v in wins if v in ws]:
                    r = Dl @ g1[w].astype(np.longdouble) - x1[w].astype(np.longdouble)
                    b = float(np.linalg.norm(r.astype(np.float64))) / (lmax * np.linalg.norm(g1[w]))
                    note("Dhat_inv bwd", b)
                    if b > BWD_TOL:
                        fails.append(f"col {c} w {w} D_hat^-1 bwd {b:.2e} > {BWD_TOL:.0e}")
            # --- S_hat^{-1} x3 = L_hat^{-1} D L_hat^{-T} x3: products only (exact D)
            e = rel(g3, o3)
            note("Shat_inv fwd", e)
            if e > prod_tol:
                fails.append(f"col {c} S_hat^-1 fwd {e:.2e} > {prod_tol:.0e}")
        else:
            e1, e3 = rel(g1, o1), rel(g3, o3)
            note("Lhat^-T x3 fwd", e1)
            note("Lhat^-1 (x1 - D c1) fwd", e3)
            if e1 > prod_tol:
                fails.append(f"col {c} L_hat^-T x3 fwd {e1:.2e} > {prod_tol:.0e}")
            if e3 > prod_tol:
                fails.append(f"col {c} L_hat^-1(x1 - D c1) fwd {e3:.2e} > {prod_tol:.0e}")
    return fails, worst


def smooth_vec(prob, seed, cols=None):
    """A library-layout vector whose first two segments lie in the range of the
    covariances (x1_w = D_w z, x2_w = R z; x3 = z): the form of a Krylov vector's
    blocks (A z puts D z1 + L z3 and R z2 + H z3 there), and the input on which a
    solve that is not backward stable (e.g. a product with a computed inverse) fails
    the backward-error bound.  Input generation only (no method arithmetic beyond
    the covariance products that define the inputs)."""
    s, p, W, m = prob.s, prob.p, prob.W, prob.m
    rng = np.random.Generator(np.random.PCG64(seed))
    z1 = rng.standard_normal((s, W, m))
    z2 = rng.standard_normal((p, W, m))
    z3 = rng.standard_normal((s, W, m))
    cs = list(range(m)) if cols is None else list(cols)
    x1, x2 = z1.copy(), z2.copy()
    for c in cs:   # the other columns stay N(0, 1)
        x1[:, 0, c] = prob.B @ z1[:, 0, c]
        x1[:, 1:, c] = prob.Q @ z1[:, 1:, c]
        x2[:, :, c] = prob.R @ z2[:, :, c]
    return np.concatenate([x1.ravel(), x2.ravel(), z3.ravel()])


def gpu_column_ops(ctx, prob, col=0):
    """(A, P^{-1}) callables on ONE paper-ordered RHS column, computed by the CUDA
    path through the C ABI (the column embedded in an otherwise zero batch: every
    apply is column-wise, so the other columns do not touch it).  Feeding these into
    the oracle's Krylov recurrence (oracle/krylov.py) isolates the recurrence from the
    operators' rounding: the oracle's count with the GPU's applies must equal the
    GPU solver's count to +-1 (reading A33).  The column's library-layout
    positions are scattered / gathered on the device (no full-batch transposes)."""
    import torch
    s, p, W, m = prob.s, prob.p, prob.W, prob.m
    # library index of each paper-order entry of column `col` (pure index permutation:
    # paper order is window-major per segment, the library's [len][W][m])
    segs = []
    off = 0
    for ln in (s, p, s):
        i, w = np.meshgrid(np.arange(ln), np.arange(W), indexing="ij")
        segs.append((off + (i * W + w) * m + col).T.reshape(-1))
        off += ln * W * m
    lib_of = np.concatenate(segs)
    ti = torch.from_numpy(lib_of).cuda()
    xd = torch.zeros(prob.n, dtype=torch.float64, device="cuda")
    yd = torch.empty_like(xd)

    def run(fn, v):
        xd.zero_()
        xd[ti] = torch.from_numpy(np.ascontiguousarray(v)).cuda()
        fn(xd, yd)
        torch.cuda.synchronize()
        return yd[ti].cpu().numpy()
    return (lambda v: run(ctx.apply_A, v)), (lambda v: run(ctx.apply_P, v))


def oracle_solution_spread(solver, A, Pinv, b, x_ref, seeds=4, **kw):
    """The oracle's own rounding sensitivity of a Krylov SOLUTION (DESIGN.md reading
    A35): max over `seeds` runs of ||x_noisy - x_ref|| / ||x_ref||, where x_noisy is the
    same oracle solve with every P^{-1} output perturbed by 1e-15 relative N(0,1) noise
    (rounding-level; the same recipe reading A34 uses for residual histories).  Where this
    exceeds north_star's 1e-9 the GPU solution is held to 2x it instead: two correct
    FP64 solves stopping at relres 1e-10 cannot be asked to agree more closely than the
    reference does with itself."""
    out = 0.0
    for sd in range(seeds):
        rng = np.random.default_rng(1000 + sd)

        def P(v, rng=rng):
            y = Pinv(v)
            return y * (1.0 + 1e-15 * rng.standard_normal(y.shape))
        x1, _ = solver(A, P, b, **kw)
        out = max(out, float(np.linalg.norm(x1 - x_ref) / np.linalg.norm(x_ref)))
    return out
