"""Gauss-Newton outer loops of incremental weak-constraint 4D-Var (ORACLE, test
infrastructure only).  SURVEY 8(f) NEXT-4; PAPER.md P:L67-71 (outer loops update the
linearisations, inner loops solve the linearised problem), the cost function of
Eq. (1.1) and the saddle-point inner problem (Eq. 2.1) with the
right-hand side of reading A3:
    b_0 = x_b - x_0,  b_w = M_w(x_{w-1}) - x_w,  d_w = y_w - H x_w,  third block 0.
Each inner problem is solved EXACTLY (dense LU of the assembled saddle matrix): the
oracle iterate is the exact Gauss-Newton sequence.  One RHS column at a time."""
import numpy as np

from . import models as OM
from .saddle import Saddle


def forecast(prob, x_prev, col=0):
    """Nonlinear (or linear) model M_w(x_{w-1})."""
    if prob.model == "l96":
        x = x_prev.copy()
        for _ in range(prob.nsub):
            x = OM.l96_rk4_step(x, prob.dt, prob.F)
        return x
    return OM.model_matrices(prob, col)[0] @ x_prev


def linearisation(prob, xs):
    """[M_1 .. M_N] about the iterate: M_w = TLM of the window map at x_{w-1}."""
    if prob.model == "l96":
        return [OM.l96_tlm(xs[w - 1], prob.dt, prob.nsub, prob.F) for w in range(1, len(xs))]
    return OM.model_matrices(prob, 0)


def cost(prob, xs, xb, ys, H):
    """J(x_0..x_N) of Eq. (1.1)."""
    J = (xs[0] - xb) @ np.linalg.solve(prob.B, xs[0] - xb)
    for w, y in enumerate(ys):
        r = y - H @ xs[w]
        J += r @ np.linalg.solve(prob.R, r)
    for w in range(1, len(xs)):
        e = xs[w] - forecast(prob, xs[w - 1])
        J += e @ np.linalg.solve(prob.Q, e)
    return J


def gauss_newton(prob, xb, ys, x0, n_outer, col=0):
    """Returns the iterates [x^(1) .. x^(n_outer)] (each a list of W states) and the
    per-iteration ||delta x||, ||(b, d)|| and J(x^(l))."""
    xs = [v.copy() for v in x0]
    W = len(xs)
    out, dxn, resn, Js = [], [], [], []
    for _ in range(n_outer):
        Ms = linearisation(prob, xs)
        sad = Saddle(prob, col=col, Ms=Ms)
        H = sad.Hi
        b = [xb - xs[0]] + [forecast(prob, xs[w - 1], col) - xs[w] for w in range(1, W)]
        d = [ys[w] - H @ xs[w] for w in range(W)]
        rhs = np.concatenate(b + d + [np.zeros(prob.s)] * W)
        Js.append(cost(prob, xs, xb, ys, H))
        resn.append(np.linalg.norm(np.concatenate(b + d)))
        sol = np.linalg.solve(sad.assemble_A(), rhs)
        dx = sol[W * (prob.s + prob.p):]
        xs = [xs[w] + dx[w * prob.s:(w + 1) * prob.s] for w in range(W)]
        dxn.append(np.linalg.norm(dx))
        out.append([v.copy() for v in xs])
    return out, dict(dx_norm=dxn, res_norm=resn, J=Js)
