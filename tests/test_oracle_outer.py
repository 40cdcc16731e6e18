"""Pins for oracle/outer.py (Gauss-Newton outer loops, Eq. 1.1)."""
import numpy as np

from oracle import outer as GN
from oracle.saddle import Saddle, primal_solution
from synth import configs as SC


def _cols(prob, col):
    W = prob.W
    g = prob.extra["guess"][:, :, col]
    ys = [prob.extra["y"][:, w, col] for w in range(W)]
    return prob.extra["xb"][:, col], ys, [g[:, w] for w in range(W)]


def test_linear_model_converges_in_one_outer_iteration():
    # the heat model is linear: one exact Gauss-Newton step reaches the minimiser of
    # J, so the next step is zero and J stops decreasing
    prob = SC.custom_problem(s=30, N=3, q=2, m=1, seed0=1)
    xb, ys, x0 = _cols(prob, 0)
    its, info = GN.gauss_newton(prob, xb, ys, x0, 3)
    assert info["dx_norm"][1] <= 1e-9 * info["dx_norm"][0]
    assert info["J"][1] < info["J"][0]
    assert abs(info["J"][2] - info["J"][1]) <= 1e-9 * info["J"][1]


def test_first_step_equals_primal_normal_equations():
    # the saddle step solves the same linearised problem as the primal form
    prob = SC.custom_problem(s=30, N=3, q=2, m=1, seed0=2)
    xb, ys, x0 = _cols(prob, 0)
    its, _ = GN.gauss_newton(prob, xb, ys, x0, 1)
    sad = Saddle(prob)
    W = prob.W
    b = np.concatenate([xb - x0[0]] + [sad.Ms[w - 1] @ x0[w - 1] - x0[w] for w in range(1, W)])
    d = np.concatenate([ys[w] - sad.Hi @ x0[w] for w in range(W)])
    dx = primal_solution(sad, b, d)[W * (prob.s + prob.p):]
    ref = np.concatenate(x0) + dx
    np.testing.assert_allclose(np.concatenate(its[0]), ref, rtol=1e-9, atol=1e-12)


def test_l96_gauss_newton_reaches_a_stationary_point_of_J():
    """Gauss-Newton (no line search) need not decrease J monotonically, but where it
    converges the limit is a stationary point of Eq. (1.1): the directional
    derivatives of J there, by central differences of the cost function itself,
    vanish relative to those at the first guess."""
    prob = SC.make_problem(2, m=2, N=5)
    rng = np.random.default_rng(0)
    for col in range(2):
        xb, ys, x0 = _cols(prob, col)
        its, info = GN.gauss_newton(prob, xb, ys, x0, 16, col=col)
        # GN converges linearly here (non-zero residual problem): ~10x per iteration
        assert info["dx_norm"][-1] < 1e-5 * info["dx_norm"][0], info["dx_norm"]
        H = Saddle(prob).Hi

        def dJ(xs, u, h=1e-6):
            plus = [x + h * uu for x, uu in zip(xs, u)]
            minus = [x - h * uu for x, uu in zip(xs, u)]
            return (GN.cost(prob, plus, xb, ys, H) - GN.cost(prob, minus, xb, ys, H)) / (2 * h)

        for _ in range(3):
            u = [rng.standard_normal(prob.s) for _ in range(prob.W)]
            g0, g1 = dJ(x0, u), dJ(its[-1], u)
            assert abs(g1) <= 1e-4 * abs(g0), (g0, g1)
