"""GPU Gauss-Newton outer loops (wf4dvar_outer_loop)
against the oracle's exact Gauss-Newton sequence (oracle/outer.py)."""
import numpy as np
import pytest

from oracle import outer as GN
from synth import configs as SC

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def WF():
    import paper_2105_06975_b200 as W
    return W


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def run_gpu(prob, pc, n_outer, solver="gmres", **kw):
    ctx = WF().Context.from_problem(prob, pc, **kw)
    xb, y, x = dev(prob.extra["xb"]), dev(prob.extra["y"]), dev(prob.extra["guess"])
    rep = ctx.outer_loop(xb, y, x, n_outer, solver=solver, tol=1e-12, maxit=3000, restart=0)
    return x.cpu().numpy(), rep


def oracle_cols(prob, n_outer):
    out = []
    for c in range(prob.m):
        g = prob.extra["guess"][:, :, c]
        ys = [prob.extra["y"][:, w, c] for w in range(prob.W)]
        its, info = GN.gauss_newton(prob, prob.extra["xb"][:, c], ys,
                                    [g[:, w] for w in range(prob.W)], n_outer, col=c)
        out.append((its, info))
    return out


@pytest.mark.parametrize("pc,solver", [
    (dict(shape="PI", lhat="L", k=1, rhat="exact"), "gmres"),
    (dict(shape="PD", lhat="LM", k=2, rhat="exact"), "minres"),
])
def test_l96_outer_loop_matches_exact_gauss_newton(pc, solver):
    prob = SC.make_problem(2, m=3, N=5)
    n_outer = 4
    xg, rep = run_gpu(prob, pc, n_outer, solver)
    ora = oracle_cols(prob, n_outer)
    for c, (its, info) in enumerate(ora):
        ref = np.stack(its[-1], axis=1)          # [s][W]
        err = np.linalg.norm(xg[:, :, c] - ref) / np.linalg.norm(ref)
        assert err <= 1e-8, (c, err)
        np.testing.assert_allclose(rep["dx_norm"][:, c], info["dx_norm"], rtol=1e-6, atol=1e-9)
        np.testing.assert_allclose(rep["res_norm"][:, c], info["res_norm"], rtol=1e-9)


def test_linear_heat_outer_loop_converges_in_one_step():
    prob = SC.custom_problem(s=64, N=4, q=2, m=2, seed0=5)
    xg, rep = run_gpu(prob, dict(shape="PI", lhat="LM", k=2, rhat="exact"), 2)
    assert np.all(rep["dx_norm"][1] <= 1e-8 * rep["dx_norm"][0])
    ora = oracle_cols(prob, 1)
    for c, (its, _) in enumerate(ora):
        ref = np.stack(its[-1], axis=1)
        assert np.linalg.norm(xg[:, :, c] - ref) / np.linalg.norm(ref) <= 1e-9


def test_sharded_outer_loop_matches_single_rank():
    from .test_gpu_dist import Sharded, run_ranks
    prob = SC.make_problem(2, m=2, N=7)
    pc = dict(shape="PI", lhat="L", k=1, rhat="exact")
    x1, _ = run_gpu(prob, pc, 3)
    sh = Sharded(prob, pc, 2)
    try:
        W = WF()
        s, p, m = prob.s, prob.p, prob.m
        xs, ys = [], []
        for r, (b, e) in enumerate(sh.bounds):
            xs.append(dev(prob.extra["guess"][:, b:e, :]))
            ys.append(dev(prob.extra["y"][:, b:e, :]))
        xb = dev(prob.extra["xb"])

        def fn(r):
            return sh.ctx[r].outer_loop(xb, ys[r], xs[r], 3, solver="gmres", tol=1e-12,
                                        maxit=3000, restart=0)
        run_ranks(2, fn)
        xg = np.concatenate([x.cpu().numpy() for x in xs], axis=1)
        assert np.linalg.norm(xg - x1) / np.linalg.norm(x1) <= 1e-9
    finally:
        sh.close()
