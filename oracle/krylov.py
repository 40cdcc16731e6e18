"""Krylov solvers (ORACLE, test infrastructure only), one right-hand side.

minres  Preconditioned MINRES for P_D ("MINRES ... with a
        residual-based convergence criterion in the two norm").  Recurrence of
        Elman, Silvester & Wathen (preconditioned Lanczos + Givens), with the
        true 2-norm residual carried by the extra recurrence on A w
        (reading A8): stop when ||r_j||_2 <= tol ||b||_2, x0 = 0.
gmres   Right-preconditioned restarted GMRES(m_r) for P_I ("relative
        residual in the two norm"), x0 = 0, classical Gram-Schmidt with one
        full re-orthogonalisation (CGS2) or modified Gram-Schmidt (reading A9).
        Iteration count = number of Arnoldi steps (one A P^{-1} product each).
Both return (x, info) with per-iteration relative residual history.
"""
import math

import numpy as np


class IndefinitePreconditioner(RuntimeError):
    pass


def minres(A, Pinv, b, tol=1e-10, maxit=1000):
    n = b.size
    bnorm = np.linalg.norm(b)
    x = np.zeros(n)
    r = b.copy()
    hist = [1.0]
    if bnorm == 0.0:
        return x, dict(iters=0, converged=True, history=hist, relres=0.0)
    v_prev = np.zeros(n)
    v = b.copy()
    z = Pinv(v)
    zv = float(z @ v)
    if zv <= 0.0:
        raise IndefinitePreconditioner("z^T v <= 0 at start")
    gamma = math.sqrt(zv)
    gamma_prev = 1.0
    eta = gamma
    c_prev = c = 1.0
    s_prev = s = 0.0
    w_prev = np.zeros(n)
    w = np.zeros(n)
    Aw_prev = np.zeros(n)
    Aw = np.zeros(n)
    converged = False
    j = 0
    for j in range(1, maxit + 1):
        z = z / gamma
        q = A(z)
        delta = float(q @ z)
        v_new = q - (delta / gamma) * v - (gamma / gamma_prev) * v_prev
        z_new = Pinv(v_new)
        zv = float(z_new @ v_new)
        if zv < 0.0:
            raise IndefinitePreconditioner(f"z^T v < 0 at iteration {j}")
        gamma_new = math.sqrt(zv)
        a0 = c * delta - c_prev * s * gamma
        a1 = math.hypot(a0, gamma_new)
        a2 = s * delta + c_prev * c * gamma
        a3 = s_prev * gamma
        c_new = a0 / a1
        s_new = gamma_new / a1
        w_new = (z - a3 * w_prev - a2 * w) / a1
        Aw_new = (q - a3 * Aw_prev - a2 * Aw) / a1
        x = x + (c_new * eta) * w_new
        r = r - (c_new * eta) * Aw_new
        eta = -s_new * eta
        v_prev, v = v, v_new
        z = z_new
        gamma_prev, gamma = gamma, gamma_new
        c_prev, c = c, c_new
        s_prev, s = s, s_new
        w_prev, w = w, w_new
        Aw_prev, Aw = Aw, Aw_new
        rel = np.linalg.norm(r) / bnorm
        hist.append(rel)
        if rel <= tol or gamma_new == 0.0:
            converged = True
            break
    return x, dict(iters=j, converged=converged, history=hist, relres=hist[-1])


def _givens(a, b):
    d = math.hypot(a, b)
    if d == 0.0:
        return 1.0, 0.0, 0.0
    return a / d, b / d, d


def gmres(A, Pinv, b, tol=1e-10, restart=50, maxit=1000, ortho="cgs2"):
    n = b.size
    bnorm = np.linalg.norm(b)
    x = np.zeros(n)
    hist = [1.0]
    if bnorm == 0.0:
        return x, dict(iters=0, converged=True, history=hist, relres=0.0, n_A=0, n_P=0)
    it = 0
    nA = nP = 0
    first = True
    converged = False
    while True:
        if first:
            r = b.copy()          # x = 0: no A product
            first = False
        else:
            r = b - A(x)
            nA += 1
        beta = np.linalg.norm(r)
        if beta <= tol * bnorm:
            converged = True
            break
        if it >= maxit:
            break
        mr = restart if restart else maxit
        V = np.zeros((mr + 1, n))
        Hm = np.zeros((mr + 1, mr))
        cs = np.zeros(mr)
        sn = np.zeros(mr)
        g = np.zeros(mr + 1)
        V[0] = r / beta
        g[0] = beta
        jj = 0
        for j in range(mr):
            u = Pinv(V[j])
            w = A(u)
            nP += 1
            nA += 1
            it += 1
            if ortho == "cgs2":
                h = V[:j + 1] @ w
                w = w - V[:j + 1].T @ h
                h2 = V[:j + 1] @ w
                w = w - V[:j + 1].T @ h2
                h = h + h2
            else:
                h = np.zeros(j + 1)
                for i in range(j + 1):
                    h[i] = V[i] @ w
                    w = w - h[i] * V[i]
            hn = np.linalg.norm(w)
            Hm[:j + 1, j] = h
            Hm[j + 1, j] = hn
            if hn > 0.0:
                V[j + 1] = w / hn
            for i in range(j):
                t = cs[i] * Hm[i, j] + sn[i] * Hm[i + 1, j]
                Hm[i + 1, j] = -sn[i] * Hm[i, j] + cs[i] * Hm[i + 1, j]
                Hm[i, j] = t
            cs[j], sn[j], Hm[j, j] = _givens(Hm[j, j], Hm[j + 1, j])
            Hm[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            jj = j + 1
            hist.append(abs(g[j + 1]) / bnorm)
            if abs(g[j + 1]) <= tol * bnorm or hn == 0.0 or it >= maxit:
                break
        y = np.zeros(jj)
        for i in range(jj - 1, -1, -1):
            y[i] = (g[i] - Hm[i, i + 1:jj] @ y[i + 1:jj]) / Hm[i, i]
        x = x + Pinv(V[:jj].T @ y)
        nP += 1
    relres = np.linalg.norm(b - A(x)) / bnorm
    return x, dict(iters=it, converged=converged, history=hist, relres=relres, n_A=nA, n_P=nP)
