"""Model operators M_w (ORACLE, test infrastructure only).

heat_M      BJ.c0: "M_i = one implicit-Euler heat step (I - r*Lap)^-1 with the
            second-difference periodic Laplacian" (reading A12: Lap unscaled,
            circulant(-2; 1, 1)).  Plain definition: dense inverse.
heat_explicit_M  NEXT-1: the paper's own heat model, explicit
            forward-Euler Dirichlet step M_dt raised to the number of
            model steps per window (Supp. P:L1134).
l96_*       dx_i/dt = (x_{i+1}-x_{i-2})x_{i-1} - x_i + F,
            periodic, integrated with RK4 (BJ.c2: dt = 0.025, 5 substeps per
            window).  The tangent linear model is the exact derivative of the
            discrete RK4 map, obtained step by step by the chain
            rule through the four RK4 stages.
"""
import numpy as np


def heat_lap(s):
    Lap = np.zeros((s, s))
    for i in range(s):
        Lap[i, i] = -2.0
        Lap[i, (i + 1) % s] += 1.0
        Lap[i, (i - 1) % s] += 1.0
    return Lap


def heat_M(s, r):
    """M = (I - r Lap)^{-1}, dense (the definition)."""
    return np.linalg.inv(np.eye(s) - r * heat_lap(s))


def heat_dirichlet_step(s, r):
    """M_dt of the explicit Dirichlet heat model (Supp. P:L1119-1131):
    forward Euler + centred second differences, first and last rows zero,
    interior rows (r, 1-2r, r) on columns i-1, i, i+1 (columns 0 and s-1 carry
    coefficient 0, as the printed matrix shows)."""
    M = np.zeros((s, s))
    for i in range(1, s - 1):
        M[i, i] = 1.0 - 2.0 * r
        if i - 1 >= 1:
            M[i, i - 1] = r
        if i + 1 <= s - 2:
            M[i, i + 1] = r
    return M


def heat_explicit_M(s, r, nsteps):
    """M between observation times = M_dt raised to the number of model steps per
    window (Supp. P:L1134: "given by M_dt raised to the appropriate power")."""
    return np.linalg.matrix_power(heat_dirichlet_step(s, r), nsteps)


def l96_rhs(x, F=8.0):
    """Lorenz-96 tendency, written with explicit periodic indices."""
    s = x.shape[0]
    out = np.empty_like(x)
    for i in range(s):
        out[i] = (x[(i + 1) % s] - x[(i - 2) % s]) * x[(i - 1) % s] - x[i] + F
    return out


def l96_jac(x):
    """Jacobian J_ij = d rhs_i / d x_j of the Lorenz-96 tendency."""
    s = x.shape[0]
    J = np.zeros((s, s))
    for i in range(s):
        ip, im2, im1 = (i + 1) % s, (i - 2) % s, (i - 1) % s
        J[i, ip] += x[im1]
        J[i, im2] -= x[im1]
        J[i, im1] += x[ip] - x[im2]
        J[i, i] -= 1.0
    return J


def l96_rk4_step(x, dt, F=8.0):
    k1 = l96_rhs(x, F)
    k2 = l96_rhs(x + 0.5 * dt * k1, F)
    k3 = l96_rhs(x + 0.5 * dt * k2, F)
    k4 = l96_rhs(x + dt * k3, F)
    return x + (dt / 6.0) * (k1 + 2.0 * k2 + 2.0 * k3 + k4)


def l96_rk4_step_jac(x, dt, F=8.0):
    """Exact Jacobian of one RK4 step at x (chain rule through the stages)."""
    s = x.shape[0]
    I = np.eye(s)
    k1 = l96_rhs(x, F)
    K1 = l96_jac(x)
    x2 = x + 0.5 * dt * k1
    k2 = l96_rhs(x2, F)
    K2 = l96_jac(x2) @ (I + 0.5 * dt * K1)
    x3 = x + 0.5 * dt * k2
    k3 = l96_rhs(x3, F)
    K3 = l96_jac(x3) @ (I + 0.5 * dt * K2)
    x4 = x + dt * k3
    K4 = l96_jac(x4) @ (I + dt * K3)
    return I + (dt / 6.0) * (K1 + 2.0 * K2 + 2.0 * K3 + K4)


def l96_tlm(x0, dt, nsub, F=8.0):
    """M_w: tangent linear of `nsub` RK4 steps started at x0 (dense s x s)."""
    s = x0.shape[0]
    M = np.eye(s)
    x = x0.copy()
    for _ in range(nsub):
        M = l96_rk4_step_jac(x, dt, F) @ M
        x = l96_rk4_step(x, dt, F)
    return M


def model_matrices(prob, col=0):
    """Dense [M_1..M_N] for RHS/problem column `col` of a synth.Problem."""
    if prob.model == "heat":
        M = heat_M(prob.s, prob.heat_r)
        return [M] * prob.N
    if prob.model == "heat_explicit":
        M = heat_explicit_M(prob.s, prob.heat_r, prob.heat_nsteps)
        return [M] * prob.N
    if prob.model == "dense":
        return [prob.M_dense[w] for w in range(prob.N)]
    if prob.model == "l96":
        return [l96_tlm(prob.traj[w][:, col], prob.dt, prob.nsub, prob.F)
                for w in range(prob.N)]
    raise ValueError(prob.model)
