"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Tolerances:
  apply_A          relative 2-norm error per RHS <= 1e-12 (BJ north_star).
  apply_P          relative error per RHS <= max(1e-12, 50 * kappa * u), kappa the
                   largest condition number among the SPD blocks the
                   preconditioner solves with (forward error of any backward-stable
                   solve is Theta(kappa u)); plus, where P is small enough to
                   assemble, the backward error ||P y - x|| / (||P|| ||y||) <= 1e-14.
  solves           ||x_gpu - x_oracle|| / ||x_oracle|| <= 1e-9 and iteration counts
                   within +-1 (BJ north_star) on short runs.
"""
import itertools

import numpy as np
import pytest

from oracle import krylov as KR
from oracle import rhat as RH
from synth import configs as SC
from synth.layout import from_paper_order, to_paper_order

from .helpers import (OracleCols, block_parity, gpu_column_ops, oracle_precond,
                      oracle_solution_spread, rel_err_cols, seeded_vec, smooth_vec)

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

U = 2.220446049250313e-16


def W4():
    import paper_2105_06975_b200 as W
    return W


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda")


def kappa_bound(prob, pc):
    ks = []
    if pc.get("shape", "PD") == "PD":
        r = pc.get("ridge", 0.0)
        ks += [np.linalg.cond(RH.dhat(prob.B, r)), np.linalg.cond(RH.dhat(prob.Q, r))]
    if pc.get("rhat", "exact") != "diag":
        ks.append(np.linalg.cond(RH.rhat(prob.R, pc.get("rhat", "exact"), pc.get("gamma", -1.0),
                                         pc.get("T", -1.0), pc.get("block", 0))))
    return max(ks) if ks else 1.0


PROBS = {
    # ragged everywhere: s, p not multiples of 64; m odd (8-byte load path); dense M_w
    "dense": lambda: SC.random_dense_problem(s=70, p=37, N=4, m=3, seed=1),
    # heat stencil path (s >= 2D+1), p = s/2, m = 5
    "heat": lambda: SC.custom_problem(s=200, N=6, q=2, m=5, seed0=3),
    # BASELINE.json configs[0]
    "c0": lambda: SC.make_problem(0),
    # blocked TRSM with several ragged super-blocks (s = 600 > SB = 256), m = 7
    "mid": lambda: SC.custom_problem(s=600, N=3, q=2, m=7, seed0=5, Bp=(0.05, 1.0),
                                     Qp=(0.05, 0.1), Rp=(0.03, 0.05)),
    # BASELINE.json configs[1] at full size
    "c1": lambda: SC.make_problem(1),
    # Lorenz-96 TLM (configs[2] recipe), 8 problems, N = 12: per-column M_w
    "l96": lambda: SC.make_problem(2, m=8, N=12),
    # the other L96 kernel variants: shared-memory exchange with 5 and 8 states per
    # thread (s = 24, 56), register shuffles with 8 (s = 64), and nsub != 5
    "l96s24": lambda: SC.custom_problem(s=24, N=6, q=2, m=37, model="l96", F=8.0, dt=0.025,
                                        nsub=3, spinup=200, seed0=7, Rp=(1.5, 0.1)),
    "l96s56": lambda: SC.custom_problem(s=56, N=5, q=2, m=9, model="l96", F=8.0, dt=0.02,
                                        nsub=8, spinup=200, seed0=8, Rp=(1.5, 0.1)),
    "l96s64": lambda: SC.custom_problem(s=64, N=5, q=2, m=33, model="l96", F=8.0, dt=0.025,
                                        nsub=1, spinup=200, seed0=9, Rp=(1.5, 0.1)),
}


def get_sampled(name, cols):
    key = (name, tuple(cols))
    if key not in _cache:
        prob = {"c2": lambda: SC.make_problem(2), "c3": lambda: SC.make_problem(3),
                "c4": lambda: SC.make_problem(4)}[name]()
        _cache[key] = (prob, OracleCols(prob, cols))
    return _cache[key]
_cache = {}


def get(name):
    if name not in _cache:
        prob = PROBS[name]()
        _cache[name] = (prob, OracleCols(prob))
    return _cache[name]


CELLS = [dict(shape=s, lhat=l, k=k, rhat=r, block=b, ridge=rd)
         for s, (l, k), (r, b), rd in itertools.product(
             ("PD", "PI"), (("L0", 1), ("LI", 1), ("LM", 1), ("LM", 2), ("LM", 3), ("LM", 4),
                            ("L", 1)),
             (("diag", 0), ("block", 8), ("rr", 0), ("me", 0), ("exact", 0)), (0.0,))]
CELLS.append(dict(shape="PD", lhat="LM", k=2, rhat="exact", ridge=0.01))


@pytest.mark.parametrize("name", ["dense", "heat", "c0", "mid", "c1", "l96", "l96s24", "l96s56",
                                  "l96s64"])
def test_apply_A(name):
    prob, ora = get(name)
    ctx = W4().Context.from_problem(prob, dict(shape="PD", lhat="LM", k=2, rhat="exact"))
    for x in (seeded_vec(prob.n, 11), smooth_vec(prob, 11)):
        y = torch.empty(prob.n, dtype=torch.float64, device="cuda")
        ctx.apply_A(dev(x), y)
        torch.cuda.synchronize()
        errs = rel_err_cols(y.cpu().numpy(), ora.apply_A(x), prob)
        assert max(errs.values()) <= 1e-12, errs


@pytest.mark.parametrize("name", ["dense", "heat"])
@pytest.mark.parametrize("pc", CELLS, ids=lambda p: f"{p['shape']}-{p['lhat']}{p['k']}-{p['rhat']}-r{p['ridge']}")
def test_apply_P(name, pc):
    prob, ora = get(name)
    ctx = W4().Context.from_problem(prob, pc)
    for x in (seeded_vec(prob.n, 12), smooth_vec(prob, 12)):
        y = torch.empty(prob.n, dtype=torch.float64, device="cuda")
        ctx.apply_P(dev(x), y)
        torch.cuda.synchronize()
        yg = y.cpu().numpy()
        fails, worst = block_parity(prob, pc, x, yg, ora, range(prob.m), cache=_kcache)
        assert not fails, (fails[:8], worst)
    x = seeded_vec(prob.n, 12)
    y = torch.empty(prob.n, dtype=torch.float64, device="cuda")
    ctx.apply_P(dev(x), y)
    torch.cuda.synchronize()
    yg = y.cpu().numpy()
    if name == "dense":   # backward error against the assembled P (column 0)
        sad = ora.sad[0]
        P = sad.assemble_P(oracle_precond(pc))
        yc = to_paper_order(yg, prob.s, prob.p, prob.W, prob.m)[0]
        xc = to_paper_order(x, prob.s, prob.p, prob.W, prob.m)[0]
        bwd = np.linalg.norm(P @ yc - xc) / (np.linalg.norm(P, 2) * np.linalg.norm(yc))
        assert bwd <= 1e-14, bwd


_kcache = {}

LARGE_CELLS = [dict(shape="PD", lhat="LM", k=4, rhat="exact"),
               dict(shape="PI", lhat="LM", k=4, rhat="exact"),
               dict(shape="PD", lhat="LM", k=2, rhat="me"),
               dict(shape="PI", lhat="LM", k=3, rhat="me"),
               dict(shape="PD", lhat="LI", k=1, rhat="block", block=50),
               dict(shape="PI", lhat="L0", k=1, rhat="diag"),
               dict(shape="PD", lhat="L", k=1, rhat="rr", ridge=0.01)]


@pytest.mark.parametrize("name", ["mid", "c1"])
@pytest.mark.parametrize("pc", LARGE_CELLS, ids=lambda p: f"{p['shape']}-{p['lhat']}{p['k']}-{p['rhat']}")
def test_apply_P_large(name, pc):
    """n >= 256: the blocked DMMA TRSM path (64-row tiles, setup-time diagonal-tile
    inverses, GEMM coupling) -- per-block forward and backward error."""
    prob, ora = get(name)
    ctx = W4().Context.from_problem(prob, pc)
    for x in (seeded_vec(prob.n, 21), smooth_vec(prob, 21)):
        y = torch.empty(prob.n, dtype=torch.float64, device="cuda")
        ctx.apply_P(dev(x), y)
        torch.cuda.synchronize()
        fails, worst = block_parity(prob, pc, x, y.cpu().numpy(), ora, range(prob.m),
                                    cache=_kcache)
        print(name, pc, worst)
        assert not fails, (fails[:8], worst)


L96_CELLS = [dict(shape="PD", lhat="LM", k=3, rhat="exact"),
             dict(shape="PI", lhat="LM", k=4, rhat="me"),
             dict(shape="PD", lhat="L", k=1, rhat="rr"),
             dict(shape="PI", lhat="LI", k=1, rhat="diag")]


@pytest.mark.parametrize("name", ["l96", "l96s24", "l96s56", "l96s64"])
@pytest.mark.parametrize("pc", L96_CELLS, ids=lambda p: f"{p['shape']}-{p['lhat']}{p['k']}-{p['rhat']}")
def test_apply_P_l96(name, pc):
    prob, ora = get(name)
    ctx = W4().Context.from_problem(prob, pc)
    # exact L^{-1} chains of the L96 TLM amplify rounding (||L^{-1}|| ~ 3e5 at N=50,
    # SURVEY PROBE-4, 8(c)-D2 "solve parts ... the exact-L chain"): 1e-10 there
    prod_tol = 1e-10 if pc["lhat"] == "L" else 1e-12
    for x in (seeded_vec(prob.n, 31), smooth_vec(prob, 31)):
        y = torch.empty(prob.n, dtype=torch.float64, device="cuda")
        ctx.apply_P(dev(x), y)
        torch.cuda.synchronize()
        fails, worst = block_parity(prob, pc, x, y.cpu().numpy(), ora, range(prob.m),
                                    prod_tol=prod_tol, cache=_kcache)
        assert not fails, (fails[:8], worst)


@pytest.mark.parametrize("name,cols", [("c2", (0, 517, 1023)), ("c3", (37,)), ("c4", (255,))])
def test_full_size_sampled_columns(name, cols):
    """BASELINE.json configs at full size, in the bench's launch configuration;
    the oracle computes the sampled RHS columns one by one."""
    prob, ora = get_sampled(name, cols)
    pc = {"c2": dict(shape="PD", lhat="LM", k=4, rhat="exact"),
          "c3": dict(shape="PD", lhat="LM", k=4, rhat="exact"),
          "c4": dict(shape="PI", lhat="LM", k=4, rhat="exact")}[name]
    ctx = W4().Context.from_problem(prob, pc)
    x = seeded_vec(prob.n, 41)
    xd = dev(x)
    y = torch.empty_like(xd)
    ctx.apply_A(xd, y)
    torch.cuda.synchronize()
    errs = rel_err_cols(y.cpu().numpy(), ora.apply_A(x), prob)
    assert max(errs.values()) <= 1e-12, errs
    W = prob.W
    for xv in (x, smooth_vec(prob, 41, cols=cols)):
        ctx.apply_P(dev(xv), y)
        torch.cuda.synchronize()
        fails, worst = block_parity(prob, pc, xv, y.cpu().numpy(), ora, cols,
                                    windows=[0, 1, W // 2, W - 1], cache=_kcache)
        print(name, worst)
        assert not fails, (fails[:8], worst)


@pytest.mark.parametrize("pc,pinned", [(dict(shape="PI", lhat="LM", k=3, rhat="me"), False),
                                       (dict(shape="PD", lhat="LM", k=3, rhat="exact"), True),
                                       (dict(shape="PI", lhat="L", k=1, rhat="block", block=8), True)])
def test_apply_AP_and_host_path_agree(pc, pinned):
    """The host path copies the blocks of x in and of y out on their own streams,
    overlapped with the other blocks' work; same kernels, so bitwise equal."""
    prob, ora = get("heat")
    ctx = W4().Context.from_problem(prob, pc)
    x = seeded_vec(prob.n, 13)
    t = torch.empty(prob.n, dtype=torch.float64, device="cuda")
    y = torch.empty_like(t)
    ctx.apply_AP(dev(x), t, y)
    if pinned:
        xp = torch.from_numpy(x).pin_memory()
        yp = torch.empty(prob.n, dtype=torch.float64).pin_memory()
        for _ in range(2):   # repeated calls reuse the staging buffers and events
            ctx.apply_AP_host(xp.numpy(), yp.numpy())
        yh = yp.numpy()
    else:
        yh = np.empty(prob.n)
        ctx.apply_AP_host(x, yh)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(y.cpu().numpy(), yh)   # same kernels, bitwise
    # against the oracle: A (P^{-1} x)
    tp = ora.apply_P(pc, x)
    tvec = from_paper_order(np.stack([tp[c] for c in range(prob.m)]), prob.s, prob.p, prob.W)
    ref = ora.apply_A(tvec)
    errs = rel_err_cols(yh, ref, prob)
    assert max(errs.values()) <= max(1e-12, 50 * kappa_bound(prob, pc) * U), errs


def test_determinism_bitwise():
    prob, _ = get("heat")
    ctx = W4().Context.from_problem(prob, dict(shape="PD", lhat="LM", k=3, rhat="exact"))
    x = dev(seeded_vec(prob.n, 14))
    outs = []
    for _ in range(3):
        t = torch.empty_like(x)
        y = torch.empty_like(x)
        ctx.apply_AP(x, t, y)
        outs.append(y.cpu().numpy())
    assert all(np.array_equal(outs[0], o) for o in outs[1:])


def test_counters_match_paper_accounting():
    prob, ora = get("heat")
    pc = dict(shape="PD", lhat="LM", k=3, rhat="block", block=8)
    ctx = W4().Context.from_problem(prob, pc)
    b = dev(prob.rhs)
    x = torch.zeros_like(b)
    rep = ctx.solve(b, x, solver="minres", tol=1e-6, maxit=40)
    W, N = prob.W, prob.N
    it_A, it_P = rep["n_apply_A"], rep["n_apply_P"]
    assert rep["n_R"] == W * it_A
    assert rep["n_D"] == W * (it_A + it_P)
    assert rep["n_Dhat_inv"] == W * it_P and rep["n_Rhat_inv"] == W * it_P
    assert rep["n_M"] == 2 * N * it_A + 2 * (N - N // 3) * it_P


def check_recurrence(ctx, prob, solver, it_gpu, it_ora, bp, col=0, **kw):
    """Counts differ by more than 1 (BJ north_star's +-1): decide whether the Krylov
    recurrence or the operators' rounding is responsible (reading A33).  The
    oracle's recurrence (oracle/krylov.py) is run again with every A and P^{-1} apply
    computed by the CUDA path (tests/helpers.gpu_column_ops).  MINRES: its count must
    equal the GPU solver's to +-1.  GMRES: the CGS2 recurrence is itself rounding
    sensitive at tol 1e-10 (r02h, configs[0]: GPU 60 / oracle 62 / recurrence with the
    GPU's applies 62 for full GMRES with the exact L; 72 / 72 / 74 restarted), so the
    GPU count must lie in that recurrence's own envelope -- its counts with 1e-15
    relative noise on every P^{-1} output (4 seeds), widened by +-1.  The cell is
    printed as flagged with all counts (flag, do not silently widen)."""
    gA, gP = gpu_column_ops(ctx, prob, col)
    fn = KR.minres if solver == "minres" else KR.gmres
    _, info = fn(gA, gP, bp, **kw)
    counts = [info["iters"]]
    if solver == "gmres" and abs(it_gpu - info["iters"]) > 1:
        rng = np.random.default_rng(7)
        for _ in range(4):
            nz = lambda v: v * (1 + 1e-15 * rng.standard_normal(v.size))
            counts.append(fn(gA, lambda v: nz(gP(v)), bp, **kw)[1]["iters"])
    print(f"[flag] iteration counts beyond +-1: gpu {it_gpu} oracle {it_ora} "
          f"oracle-recurrence-with-gpu-applies {counts}")
    if min(counts) - 1 <= it_gpu <= max(counts) + 1:
        return True
    # outside the envelope (r02j: full GMRES, configs[0], P_I with the exact L: GPU 60 vs
    # 62 for the oracle and for its recurrence with the GPU's applies under all 5 noise
    # seeds -- the GPU's CGS2 estimate crossed 1e-10 two steps earlier): the caller
    # checks the GPU's stop against the TRUE residual with the oracle's A instead
    assert solver == "gmres", (it_gpu, it_ora, counts)
    return False


@pytest.mark.parametrize("k,rhat", [(5, "exact"), (3, "me"), (2, "rr")])
def test_minres_c0_matches_oracle(k, rhat):
    prob, ora = get("c0")
    pc = dict(shape="PD", lhat="LM", k=k, rhat=rhat)
    ctx = W4().Context.from_problem(prob, pc)
    b = dev(prob.rhs)
    x = torch.empty_like(b)
    rep = ctx.solve(b, x, solver="minres", tol=1e-10, maxit=5000, history=True)
    sad = ora.sad[0]
    bp = to_paper_order(prob.rhs, prob.s, prob.p, prob.W, 1)[0]
    opc = oracle_precond(pc)
    xo, info = KR.minres(sad.apply_A, lambda v: sad.apply_Pinv(opc, v), bp, tol=1e-10, maxit=5000)
    xg = to_paper_order(x.cpu().numpy(), prob.s, prob.p, prob.W, 1)[0]
    assert rep["converged"][0] and info["converged"]
    if abs(int(rep["iters"][0]) - info["iters"]) > 1:
        check_recurrence(ctx, prob, "minres", int(rep["iters"][0]), info["iters"], bp,
                         tol=1e-10, maxit=5000)
    d = np.linalg.norm(xg - xo) / np.linalg.norm(xo)
    if d > 1e-9:   # reading A35
        spread = oracle_solution_spread(KR.minres, sad.apply_A,
                                        lambda v: sad.apply_Pinv(opc, v), bp, xo, tol=1e-10,
                                        maxit=5000)
        print(f"[flag] |x_gpu - x_oracle| {d:.2e} > 1e-9; oracle self-spread {spread:.2e}")
        assert d <= 2 * spread, (d, spread)
    xstar = np.linalg.solve(sad.assemble_A(), bp)
    assert np.linalg.norm(xg - xstar) / np.linalg.norm(xstar) <= 1e-7


@pytest.mark.parametrize("k,rhat,restart", [(5, "exact", 50), (3, "rr", 50), (1, "exact", 20),
                                            # full (unrestarted) GMRES: c0
                                            # runs both full and restarted at 50
                                            (5, "exact", 0), (3, "me", 0), (2, "diag", 0),
                                            (4, "block", 0)])
def test_gmres_c0_matches_oracle(k, rhat, restart):
    prob, ora = get("c0")
    pc = dict(shape="PI", lhat="LM", k=k, rhat=rhat, block=5 if rhat == "block" else 0)
    ctx = W4().Context.from_problem(prob, pc)
    b = dev(prob.rhs)
    x = torch.empty_like(b)
    rep = ctx.solve(b, x, solver="gmres", tol=1e-10, maxit=5000, restart=restart, history=True)
    sad = ora.sad[0]
    bp = to_paper_order(prob.rhs, prob.s, prob.p, prob.W, 1)[0]
    opc = oracle_precond(pc)
    xo, info = KR.gmres(sad.apply_A, lambda v: sad.apply_Pinv(opc, v), bp, tol=1e-10,
                        restart=restart, maxit=5000)
    xg = to_paper_order(x.cpu().numpy(), prob.s, prob.p, prob.W, 1)[0]
    assert rep["converged"][0] and info["converged"]
    if abs(int(rep["iters"][0]) - info["iters"]) > 1:
        if not check_recurrence(ctx, prob, "gmres", int(rep["iters"][0]), info["iters"], bp,
                                tol=1e-10, restart=restart, maxit=5000):
            true_rel = np.linalg.norm(bp - sad.apply_A(xg)) / np.linalg.norm(bp)
            print(f"[flag] GPU stop at {int(rep['iters'][0])}: true relres {true_rel:.2e}")
            assert true_rel <= 2e-10, true_rel
    d = np.linalg.norm(xg - xo) / np.linalg.norm(xo)
    if d > 1e-9:   # reading A35: the oracle's own solution spread under rounding noise
        spread = oracle_solution_spread(KR.gmres, sad.apply_A,
                                        lambda v: sad.apply_Pinv(opc, v), bp, xo, tol=1e-10,
                                        restart=restart, maxit=5000)
        print(f"[flag] |x_gpu - x_oracle| {d:.2e} > 1e-9; oracle self-spread {spread:.2e}")
        assert d <= 2 * spread, (d, spread)


def test_batched_solve_matches_per_rhs_oracle():
    prob, ora = get("heat")
    pc = dict(shape="PI", lhat="LM", k=2, rhat="exact")
    ctx = W4().Context.from_problem(prob, pc)
    b = dev(prob.rhs)
    x = torch.empty_like(b)
    rep = ctx.solve(b, x, solver="gmres", tol=1e-10, maxit=2000, restart=50)
    xg = to_paper_order(x.cpu().numpy(), prob.s, prob.p, prob.W, prob.m)
    B = to_paper_order(prob.rhs, prob.s, prob.p, prob.W, prob.m)
    opc = oracle_precond(pc)
    for c in range(prob.m):
        sad = ora.sad[c]
        xo, info = KR.gmres(sad.apply_A, lambda v: sad.apply_Pinv(opc, v), B[c], tol=1e-10,
                            restart=50, maxit=2000)
        assert info["converged"] and rep["converged"][c]
        if abs(int(rep["iters"][c]) - info["iters"]) > 1:
            if not check_recurrence(ctx, prob, "gmres", int(rep["iters"][c]), info["iters"], B[c],
                                    col=c, tol=1e-10, restart=50, maxit=2000):
                true_rel = np.linalg.norm(B[c] - sad.apply_A(xg[c])) / np.linalg.norm(B[c])
                assert true_rel <= 2e-10, (c, true_rel)
        assert np.linalg.norm(xg[c] - xo) / np.linalg.norm(xo) <= 1e-9


def test_explicit_inverse_mode_agrees_forward():
    """Reading A32 (opt-in, apply_mode="inverse"): the dense preconditioner blocks
    (n >= 256) applied as one GEMM with setup-time explicit inverses.  It agrees with
    the default triangular solves to the forward tolerance of the blocks' conditioning,
    but it is not backward stable: on covariance-range vectors its backward error
    is far above 1e-14 (printed; this is why the triangular solves are the default,
    DESIGN.md section 6)."""
    prob, ora = get("mid")
    x = dev(smooth_vec(prob, 8))
    kap = max(np.linalg.cond(prob.B), np.linalg.cond(prob.Q), np.linalg.cond(prob.R))
    for pc in (dict(shape="PD", lhat="LM", k=2, rhat="exact"),
               dict(shape="PI", lhat="LM", k=2, rhat="rr"),
               dict(shape="PD", lhat="LM", k=2, rhat="block", block=50)):
        outs = {}
        for mode in ("trsm", "inverse"):
            ctx = W4().Context.from_problem(prob, dict(pc, apply_mode=mode))
            y = torch.empty_like(x)
            ctx.apply_P(x, y)
            torch.cuda.synchronize()
            outs[mode] = y.cpu().numpy()
            ctx.close()
        a, b = outs["inverse"], outs["trsm"]
        assert np.linalg.norm(a - b) / np.linalg.norm(b) <= max(1e-12, 10 * kap * U)
        fails, worst = block_parity(prob, pc, x.cpu().numpy(), a, ora, [0], cache=_kcache)
        print("[A32 inverse mode]", pc, worst)


HOST_CHUNK = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_2105_06975_b200 as W
from synth import configs as SC
prob = SC.custom_problem(s=600, N=3, q=2, m=7, seed0=5, Bp=(0.05, 1.0), Qp=(0.05, 0.1),
                         Rp=(0.03, 0.05))
x = np.random.Generator(np.random.PCG64(8)).standard_normal(prob.n)
outs = []
for pc in (dict(shape="PD", lhat="LM", k=2, rhat="exact"),
           dict(shape="PD", lhat="LM", k=2, rhat="exact", apply_mode="inverse")):
    ctx = W.Context.from_problem(prob, pc)
    xp = torch.from_numpy(x).pin_memory()
    yp = torch.empty(prob.n, dtype=torch.float64).pin_memory()
    for _ in range(2):
        ctx.apply_AP_host(xp.numpy(), yp.numpy())
    t = torch.empty(prob.n, dtype=torch.float64, device="cuda")
    y = torch.empty_like(t)
    ctx.apply_AP(torch.from_numpy(x).cuda(), t, y)
    outs += [yp.numpy().copy(), y.cpu().numpy()]
    ctx.close()
np.save(sys.argv[2], np.stack(outs))
"""


def test_host_path_column_chunks(tmp_path):
    """The host path copies the first block in window-aligned column chunks and solves /
    multiplies each chunk as it lands (forced here on a small problem with
    WF4DVAR_HOST_CHUNK_MB=0): same result as the device path to the blocks' conditioning,
    for the triangular solves (default) and the explicit inverses."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = tmp_path / "hc.npy"
    r = subprocess.run([sys.executable, "-c", HOST_CHUNK, root, str(out)], capture_output=True,
                       text=True, env=dict(os.environ, WF4DVAR_HOST_CHUNK_MB="0"), timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    o = np.load(out)
    prob, _ = get("mid")
    kap = max(np.linalg.cond(prob.B), np.linalg.cond(prob.Q), np.linalg.cond(prob.R))
    for host, devv in ((o[0], o[1]), (o[2], o[3])):
        assert np.linalg.norm(host - devv) / np.linalg.norm(devv) <= max(1e-12, 10 * kap * U)
