"""Pins for oracle/krylov.py: finite termination, exact limits (dense LU), 2-norm rule."""
import numpy as np
import pytest

from oracle import krylov as KR
from oracle.saddle import Precond, Saddle
from synth import configs as SC
from synth.layout import to_paper_order


def test_minres_finite_termination():
    A = np.diag(np.arange(1.0, 11.0))
    b = np.ones(10)
    x, info = KR.minres(lambda v: A @ v, lambda v: v.copy(), b, tol=1e-10, maxit=50)
    assert info["converged"] and info["iters"] <= 10
    np.testing.assert_allclose(x, 1.0 / np.arange(1.0, 11.0), rtol=1e-9)


def test_gmres_identity_one_iteration():
    b = np.arange(1.0, 6.0)
    x, info = KR.gmres(lambda v: v.copy(), lambda v: v.copy(), b, tol=1e-12, restart=50)
    assert info["iters"] == 1 and info["converged"]
    np.testing.assert_allclose(x, b)


def test_gmres_indefinite_small_matches_lu():
    rng = np.random.default_rng(0)
    A = rng.standard_normal((40, 40)) + 10 * np.eye(40)
    b = rng.standard_normal(40)
    for restart in (50, 7):
        for ortho in ("cgs2", "mgs"):
            x, info = KR.gmres(lambda v: A @ v, lambda v: v.copy(), b, tol=1e-12,
                               restart=restart, maxit=2000, ortho=ortho)
            assert info["converged"]
            np.testing.assert_allclose(x, np.linalg.solve(A, b), rtol=1e-9)
            h = np.array(info["history"])
            if restart == 50:
                assert np.all(np.diff(h) <= 1e-12)   # GMRES residual monotone


@pytest.fixture(scope="module")
def c0():
    prob = SC.make_problem(0)
    sad = Saddle(prob)
    b = to_paper_order(prob.rhs, prob.s, prob.p, prob.W, 1)[0]
    xstar = np.linalg.solve(sad.assemble_A(), b)
    return prob, sad, b, xstar


@pytest.mark.parametrize("k,rhat", [(5, "exact"), (3, "exact"), (3, "me")])
def test_minres_PD_c0_reaches_exact_solution(c0, k, rhat):
    prob, sad, b, xstar = c0
    pc = Precond("PD", "LM", k, rhat)
    x, info = KR.minres(sad.apply_A, lambda v: sad.apply_Pinv(pc, v), b, tol=1e-10, maxit=5000)
    assert info["converged"]
    true_rel = np.linalg.norm(b - sad.apply_A(x)) / np.linalg.norm(b)
    # the 2-norm recurrence tracks the true residual (reading A8)
    assert true_rel < 1e-8 and info["relres"] <= 1e-10
    assert np.linalg.norm(x - xstar) / np.linalg.norm(xstar) < 1e-7


@pytest.mark.parametrize("k,rhat", [(5, "exact"), (3, "rr"), (1, "exact")])
def test_gmres_PI_c0_reaches_exact_solution(c0, k, rhat):
    prob, sad, b, xstar = c0
    pc = Precond("PI", "LM", k, rhat)
    res = {}
    for ortho in ("cgs2", "mgs"):
        x, info = KR.gmres(sad.apply_A, lambda v: sad.apply_Pinv(pc, v), b, tol=1e-10,
                           restart=50, maxit=5000, ortho=ortho)
        assert info["converged"]
        assert info["relres"] < 1e-9
        assert np.linalg.norm(x - xstar) / np.linalg.norm(xstar) < 1e-8
        res[ortho] = info["iters"]
    assert abs(res["cgs2"] - res["mgs"]) <= 4     # PROBE-3: +-2 typical
