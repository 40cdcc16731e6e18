"""configs[3]'s structure with the oracle's solve affordable: 128 windows (N = 127),
stride-4 observations, the c3 SOAR lengths (B, Q: 0.01; R: 0.005), but s = 256 instead of
4096 (the oracle's blockwise MINRES at s = 4096 would take hours per RHS).  P_D + MINRES
to 1e-10 with L_M(4) (the headline cell: chains aligned with every 1/2/4/8-rank shard)
and L_M(3) (chains crossing shard boundaries), against the oracle: iteration counts
within +-1 (or the recurrence check of DESIGN.md reading A33) and the solution to 1e-9,
also against the exact solution of the Fourier-block oracle (every RHS).
Also pins the grid's finding that the exact L (k = N + 1 = 128) needs about twice the
iterations of L_M(4) on this periodic heat problem (oracle: 683 vs 1377)."""
import numpy as np
import pytest

from oracle import fourier as FO
from oracle import krylov as KR
from oracle.saddle import Precond, Saddle
from synth import configs as SC
from synth.layout import to_paper_order

from .helpers import gpu_column_ops

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
_P = {}


def problem():
    if "p" not in _P:
        _P["p"] = SC.custom_problem(s=256, N=127, q=4, m=2, seed0=0, Bp=(0.01, 1.0),
                                    Qp=(0.01, 0.1), Rp=(0.005, 0.05))
        _P["sad"] = Saddle(_P["p"], col=0)
    return _P["p"], _P["sad"]


@pytest.mark.parametrize("k", [4, 3])
def test_c3_shaped_minres_matches_oracle(k):
    import paper_2105_06975_b200 as W
    prob, sad = problem()
    pc = dict(shape="PD", lhat="LM", k=k, rhat="exact")
    ctx = W.Context.from_problem(prob, pc)
    b = torch.from_numpy(prob.rhs).cuda()
    x = torch.empty_like(b)
    rep = ctx.solve(b, x, solver="minres", tol=1e-10, maxit=4000, history=True)
    assert all(rep["converged"])
    bp = to_paper_order(prob.rhs, prob.s, prob.p, prob.W, prob.m)[0]
    xo, info = KR.minres(sad.apply_A, lambda v: sad.apply_Pinv(Precond("PD", "LM", k, "exact"), v),
                         bp, tol=1e-10, maxit=4000)
    assert info["converged"]
    it_g = int(rep["iters"][0])
    print(f"[c3-shape k={k}] iters gpu {rep['iters'].tolist()} oracle(col 0) {info['iters']}")
    if abs(it_g - info["iters"]) > 1:
        gA, gP = gpu_column_ops(ctx, prob, 0)
        _, info_g = KR.minres(gA, gP, bp, tol=1e-10, maxit=4000)
        # finite-precision Lanczos counts of runs over 500 iterations move
        # by up to ~2% under rounding-level changes (PROBE-2: +-30 beyond 1000
        # iterations); its secondary rule |d| <= ceil(0.02 it) applies there (reading A33)
        tol_it = 1 if info_g["iters"] <= 500 else int(np.ceil(0.02 * info_g["iters"]))
        print(f"[flag] gpu {it_g} oracle {info['iters']} oracle-recurrence-with-gpu-applies "
              f"{info_g['iters']} (allowed +-{tol_it})")
        assert abs(it_g - info_g["iters"]) <= tol_it
    X = to_paper_order(x.cpu().numpy(), prob.s, prob.p, prob.W, prob.m)
    d = np.linalg.norm(X[0] - xo) / np.linalg.norm(xo)
    xs = FO.solve_heat(prob, to_paper_order(prob.rhs, prob.s, prob.p, prob.W, prob.m))
    e = [np.linalg.norm(X[c] - xs[c]) / np.linalg.norm(xs[c]) for c in range(prob.m)]
    print(f"[c3-shape k={k}] |x_gpu - x_oracle| / |x_oracle| = {d:.2e}; vs exact {max(e):.2e}")
    assert d <= 1e-9, d
    assert max(e) <= 1e-9, e
    ctx.close()


def test_c3_shaped_exact_L_needs_more_iterations():
    import paper_2105_06975_b200 as W
    prob, _ = problem()
    b = torch.from_numpy(prob.rhs).cuda()
    x = torch.empty_like(b)
    its = {}
    for k in (4, 128):
        ctx = W.Context.from_problem(prob, dict(shape="PD", lhat="LM", k=k, rhat="exact"))
        its[k] = int(ctx.solve(b, x, solver="minres", tol=1e-8, maxit=4000)["iters"][0])
        ctx.close()
    print(f"[c3-shape] MINRES iterations to 1e-8: L_M(4) {its[4]}, exact L {its[128]}")
    assert its[128] > 1.5 * its[4]
