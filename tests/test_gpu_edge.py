"""GPU edge cases of the hot path against the oracle: a single window (N = 0: L = I,
no model term), a single RHS, every state observed (p = s), the two extremes of
L_M(k) (k = 1: L_0; k = N + 1: exact L), one-row / one-column problems, and apply
with a zero vector."""
import numpy as np
import pytest

from synth import configs as SC

from .helpers import OracleCols, rel_err_cols, seeded_vec

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def WF():
    import paper_2105_06975_b200 as W
    return W


def check(prob, pc, tolP=1e-9):
    ctx = WF().Context.from_problem(prob, pc)
    ora = OracleCols(prob)
    x = seeded_vec(prob.n, 1)
    y = torch.empty(prob.n, dtype=torch.float64, device="cuda")
    ctx.apply_A(torch.from_numpy(x).cuda(), y)
    torch.cuda.synchronize()
    assert max(rel_err_cols(y.cpu().numpy(), ora.apply_A(x), prob).values()) <= 1e-12
    ctx.apply_P(torch.from_numpy(x).cuda(), y)
    torch.cuda.synchronize()
    assert max(rel_err_cols(y.cpu().numpy(), ora.apply_P(pc, x), prob).values()) <= tolP
    return ctx


@pytest.mark.parametrize("pc", [dict(shape="PD", lhat="LM", k=1, rhat="exact"),
                                dict(shape="PI", lhat="L", k=1, rhat="rr"),
                                dict(shape="PD", lhat="LI", k=1, rhat="diag")])
def test_single_window(pc):
    check(SC.custom_problem(s=64, N=0, q=2, m=3, seed0=1), pc)


def test_single_rhs_every_point_observed_and_k_extremes():
    prob = SC.custom_problem(s=96, N=5, q=1, m=1, seed0=2, Rp=(0.05, 0.05))
    for k in (1, 2, 6):
        check(prob, dict(shape="PD", lhat="LM", k=k, rhat="exact"))
        check(prob, dict(shape="PI", lhat="LM", k=k, rhat="block", block=32))


def test_tiny_dense_problem_one_observation():
    prob = SC.random_dense_problem(s=3, p=1, N=2, m=1, seed=4)
    check(prob, dict(shape="PD", lhat="LM", k=2, rhat="exact"))
    check(prob, dict(shape="PI", lhat="L", k=1, rhat="diag"))


def test_zero_vector_and_solve_of_zero_rhs():
    prob = SC.custom_problem(s=64, N=3, q=2, m=2, seed0=3)
    ctx = WF().Context.from_problem(prob, dict(shape="PD", lhat="LM", k=2, rhat="exact"))
    z = torch.zeros(prob.n, dtype=torch.float64, device="cuda")
    y = torch.empty_like(z)
    ctx.apply_A(z, y)
    ctx.apply_P(z, y)
    torch.cuda.synchronize()
    assert torch.count_nonzero(y) == 0
    x = torch.empty_like(z)
    rep = ctx.solve(z, x, solver="minres", tol=1e-10, maxit=10)
    assert torch.count_nonzero(x) == 0 and (rep["iters"] == 0).all()


def test_invalid_arguments_fail_loudly():
    W = WF()
    prob = SC.custom_problem(s=64, N=3, q=2, m=2, seed0=3)
    with pytest.raises(W.WF4DVarError):
        W.Context.from_problem(prob, dict(shape="PD", lhat="LM", k=9, rhat="exact"))  # k > N+1
    with pytest.raises(W.WF4DVarError):
        W.Context.from_problem(prob, dict(shape="PD", lhat="LM", k=2, rhat="block", block=0))
    bad = SC.custom_problem(s=64, N=3, q=2, m=2, seed0=3)
    bad.R = -bad.R
    with pytest.raises(W.WF4DVarError) as e:
        W.Context.from_problem(bad, dict(shape="PD", lhat="LM", k=2, rhat="exact"))
    assert e.value.code == "ENOTSPD"
