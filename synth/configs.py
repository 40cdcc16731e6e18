"""Seeded problem builders for BASELINE.json configs[0..4] (and custom sizes).

Everything here is INPUT DATA. Readings:
  A1  SOAR distance is chordal: d = (C/pi)|sin(pi*(x_i-x_j)/C)|, C = domain
      length (1 for the heat grid on [0,1), s index units for Lorenz-96).
  A2  SOAR(d) = var * (1 + d/L) * exp(-d/L)   (BJ.c0 writes "(1+d/0.2)exp(-d/0.2)").
  A3  RHS by linearising about the background forecast x^(0):
      x^(0)_0 = x_b, x^(0)_w = M_w(x^(0)_{w-1}); b = 0 (b_0 = x_b - x^(0)_0 = 0,
      b_w = M_w(x^(0)_{w-1}) - x^(0)_w = 0), d_w = y_w - H x^(0)_w.
  A14 H_w selects every q-th state point starting at 0 (idx_j = q*j), same for all w.
  A15 numpy Generator(PCG64(seed)); RHS/problem column j uses seed (seed0 + j);
      draw order: x_0^t, model noise w=1..N, observation noise w=0..N, background.
The truth/background model propagation below is workload synthesis (it builds
y and x_b); the operator M_w used by the METHOD is implemented separately by
oracle/ and by the CUDA library.
"""
from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import scipy.linalg as sla

from .layout import pack

# (length, variance) pairs; heat grids live on [0,1) with spacing 1/s.
CONFIGS = {
    0: dict(model="heat", s=50, N=4, q=2, m=1, B=(0.2, 1.0), Q=(0.2, 0.1),
            R=(0.1, 0.05), heat_r=0.25,
            desc="BJ.c0 heat s=50 N=4 p=25 single RHS"),
    1: dict(model="heat", s=1000, N=20, q=2, m=16, B=(0.05, 1.0), Q=(0.05, 0.1),
            R=(0.02, 0.05), heat_r=0.25,
            desc="BJ.c1 heat s=1000 N=20 p=500, 16 RHS"),
    2: dict(model="l96", s=40, N=50, q=2, m=1024, B=(2.0, 1.0), Q=(2.0, 0.1),
            R=(1.0, 0.1), F=8.0, dt=0.025, nsub=5, spinup=1000,
            desc="BJ.c2 Lorenz-96 TLM s=40 N=50 p=20, 1024 problems"),
    3: dict(model="heat", s=4096, N=127, q=4, m=64, B=(0.01, 1.0), Q=(0.01, 0.1),
            R=(0.005, 0.05), heat_r=0.25,
            desc="BJ.c3 heat s=4096 N=127 p=1024, 64 RHS"),
    4: dict(model="heat", s=2048, N=31, q=1, m=256, B=(0.02, 1.0), Q=(0.02, 0.1),
            R=(0.1, 0.01), heat_r=0.25,
            desc="BJ.c4 heat s=2048 N=31 p=2048, 256 RHS"),
    # not a BASELINE.json config: the widened row NEXT-1 -- the paper's own
    # heat workload (explicit Dirichlet model, 5-point smoothed H, compact-support
    # modified SOAR, block-structured R_i) at a size that makes the GPU work visible
    5: dict(model="heat_explicit", s=2048, N=31, m=32, nsteps=2,
            desc="NEXT-1 paper heat s=2048 N=31 p=1024 (explicit Dirichlet, smoothed H, "
                 "compact SOAR, block R), 32 RHS"),
}


@dataclass
class Problem:
    name: str
    model: str              # "heat" | "l96" | "dense"
    s: int
    p: int
    N: int
    m: int
    B: np.ndarray           # [s,s]
    Q: np.ndarray           # [s,s] shared by windows 1..N
    R: np.ndarray           # [p,p] shared by windows 0..N
    H_idx: np.ndarray       # [p] int32, strictly increasing
    heat_r: float = 0.0
    F: float = 8.0
    dt: float = 0.0
    nsub: int = 0
    traj: Optional[np.ndarray] = None     # l96: [N][s][m] start state of window w-1 for M_w
    M_dense: Optional[np.ndarray] = None  # dense model: [N][s][s] (M_w for w=1..N)
    rhs: Optional[np.ndarray] = None      # flat library layout, (2s+p)*W*m
    extra: dict = field(default_factory=dict)
    heat_nsteps: int = 1                  # heat_explicit: model steps per window
    H_csr: Optional[tuple] = None         # (rowptr, col, val): general H_i (replaces H_idx)

    @property
    def W(self):
        return self.N + 1

    @property
    def n(self):
        return (2 * self.s + self.p) * self.W * self.m


def chordal_distance(lag, C):
    """Chordal distance on a circle of circumference C for a lag in the same units."""
    return (C / np.pi) * np.abs(np.sin(np.pi * np.asarray(lag, dtype=np.float64) / C))


def soar(d, L, var):
    d = np.asarray(d, dtype=np.float64)
    return var * (1.0 + d / L) * np.exp(-d / L)


def soar_matrix(positions, C, L, var):
    """Dense SOAR covariance between points at `positions` on a circle of length C."""
    pos = np.asarray(positions, dtype=np.float64)
    lag = pos[:, None] - pos[None, :]
    return soar(chordal_distance(lag, C), L, var)


def heat_lap(s):
    """Periodic second-difference matrix (diag -2, off-diagonals +1), unscaled."""
    Lap = -2.0 * np.eye(s)
    i = np.arange(s)
    Lap[i, (i + 1) % s] += 1.0
    Lap[i, (i - 1) % s] += 1.0
    return Lap


def _l96_rhs(x, F):
    # dx_i/dt = (x_{i+1} - x_{i-2}) x_{i-1} - x_i + F, axis 0 = state
    return (np.roll(x, -1, 0) - np.roll(x, 2, 0)) * np.roll(x, 1, 0) - x + F


def _l96_rk4(x, dt, F):
    k1 = _l96_rhs(x, F)
    k2 = _l96_rhs(x + 0.5 * dt * k1, F)
    k3 = _l96_rhs(x + 0.5 * dt * k2, F)
    k4 = _l96_rhs(x + dt * k3, F)
    return x + dt / 6.0 * (k1 + 2 * k2 + 2 * k3 + k4)


def _gaussian(rng_list, chol, shape_first):
    """Draw one N(0, C) sample per column generator: returns [n, m]."""
    z = np.stack([g.standard_normal(shape_first) for g in rng_list], axis=1)
    return chol @ z


def _build(name, model, s, N, q, m, Bp, Qp, Rp, seed0, heat_r=0.25, F=8.0, dt=0.025,
           nsub=5, spinup=1000, with_rhs=True, domain=None):
    W = N + 1
    H_idx = (np.arange(0, s, q)).astype(np.int32)
    p = H_idx.size
    if model == "heat":
        C = 1.0
        pos_state = np.arange(s) / s
    else:
        C = float(s)
        pos_state = np.arange(s, dtype=np.float64)
    pos_obs = pos_state[H_idx]
    B = soar_matrix(pos_state, C, *Bp)
    Q = soar_matrix(pos_state, C, *Qp)
    R = soar_matrix(pos_obs, C, *Rp)
    prob = Problem(name=name, model=model, s=s, p=p, N=N, m=m, B=B, Q=Q, R=R,
                   H_idx=H_idx, heat_r=heat_r, F=F, dt=dt, nsub=nsub)
    if not with_rhs:
        return prob
    rngs = [np.random.Generator(np.random.PCG64(seed0 + j)) for j in range(m)]
    cB = np.linalg.cholesky(B)
    cQ = np.linalg.cholesky(Q)
    cR = np.linalg.cholesky(R)
    if model == "heat":
        lu = sla.lu_factor(np.eye(s) - heat_r * heat_lap(s))
        step = lambda x: sla.lu_solve(lu, x)  # truth/forecast model (synthesis only)
        x0t = _gaussian(rngs, cB, s)
    else:
        def step(x):
            for _ in range(nsub):
                x = _l96_rk4(x, dt, F)
            return x
        spin = F + 0.01 * np.stack([g.standard_normal(s) for g in rngs], axis=1)
        for _ in range(spinup):
            spin = _l96_rk4(spin, dt, F)
        x0t = spin
    truth = [x0t]
    for w in range(1, W):
        truth.append(step(truth[-1]) + _gaussian(rngs, cQ, s))
    y = [truth[w][H_idx] + _gaussian(rngs, cR, p) for w in range(W)]
    xb = x0t + _gaussian(rngs, cB, s)
    guess = [xb]
    for w in range(1, W):
        guess.append(step(guess[-1]))
    eta = np.zeros((s, W, m))            # b = 0 (reading A3)
    nu = np.stack([y[w] - guess[w][H_idx] for w in range(W)], axis=1)   # [p][W][m]
    xx = np.zeros((s, W, m))
    prob.rhs = pack(eta, nu, xx)
    if model == "l96":
        prob.traj = np.ascontiguousarray(np.stack(guess[:N], axis=0))  # [N][s][m]
    prob.extra = dict(truth=np.stack(truth, 1), xb=xb, guess=np.stack(guess, 1), y=np.stack(y, 1))
    return prob


def make_problem(cfg, seed0=0, m=None, N=None, with_rhs=True):
    """Build BASELINE.json configs[cfg]; optionally override batch width m or N.
    With env WF4DVAR_PROBLEM_CACHE=<dir> the built problem is pickled there, keyed by
    the arguments and this module's source (tools running many processes on one box
    build each config once; the content is a deterministic function of the key)."""
    import os
    cdir = os.environ.get("WF4DVAR_PROBLEM_CACHE")
    if cdir:
        import hashlib
        import pickle
        src = open(__file__, "rb").read()
        key = hashlib.sha1(repr((cfg, seed0, m, N, with_rhs)).encode() + src).hexdigest()[:16]
        fn = os.path.join(cdir, f"c{cfg}_{key}.pkl")
        if os.path.exists(fn):
            with open(fn, "rb") as f:
                return pickle.load(f)
        prob = _make_problem(cfg, seed0, m, N, with_rhs)
        os.makedirs(cdir, exist_ok=True)
        with open(fn + ".tmp", "wb") as f:
            pickle.dump(prob, f, protocol=4)
        os.replace(fn + ".tmp", fn)
        return prob
    return _make_problem(cfg, seed0, m, N, with_rhs)


def _make_problem(cfg, seed0, m, N, with_rhs):
    c = dict(CONFIGS[cfg])
    mm = c["m"] if m is None else m
    NN = c["N"] if N is None else N
    if c["model"] == "heat_explicit":
        return paper_heat_problem(s=c["s"], N=NN, m=mm, nsteps=c["nsteps"], seed0=seed0,
                                  with_rhs=with_rhs)
    kw = {}
    if c["model"] == "l96":
        kw = dict(F=c["F"], dt=c["dt"], nsub=c["nsub"], spinup=c["spinup"])
    else:
        kw = dict(heat_r=c["heat_r"])
    return _build(f"c{cfg}", c["model"], c["s"], NN, c["q"], mm, c["B"], c["Q"], c["R"],
                  seed0, with_rhs=with_rhs, **kw)


def custom_problem(s, N, q, m, model="heat", seed0=0, Bp=(0.1, 1.0), Qp=(0.1, 0.1),
                   Rp=(0.05, 0.05), heat_r=0.25, **kw):
    """Parity-test sizes: same recipe, arbitrary (s, N, q, m)."""
    return _build(f"custom_s{s}_N{N}_q{q}_m{m}", model, s, N, q, m, Bp, Qp, Rp, seed0,
                  heat_r=heat_r, **kw)


def random_dense_problem(s, p, N, m, seed=0):
    """Generic small problem with random dense SPD B,Q,R, random dense M_w and a
    random strictly-increasing selection H (tests the general API paths)."""
    rng = np.random.Generator(np.random.PCG64(seed))

    def spd(n):
        A = rng.standard_normal((n, n))
        return A @ A.T / n + 0.5 * np.eye(n)

    B, Q, R = spd(s), spd(s), spd(p)
    H_idx = np.sort(rng.choice(s, size=p, replace=False)).astype(np.int32)
    M = rng.standard_normal((N, s, s)) / np.sqrt(s)
    W = N + 1
    prob = Problem(name=f"dense_s{s}_p{p}_N{N}_m{m}", model="dense", s=s, p=p, N=N, m=m,
                   B=B, Q=Q, R=R, H_idx=H_idx, M_dense=M)
    prob.rhs = rng.standard_normal((2 * s + p) * W * m)
    return prob


def paper_block_R(pvec, pcorr=None, seed=0, density=0.3, L=0.6, maxval=None, sigma=0.4,
                  min_eig=0.41):
    """The paper's block-structured synthetic R_i, reading A26:
      * diagonal block k (size pvec_k): Hadamard product of a sparse random matrix
        (entries U(0,1), density `density`) and a compact-support SOAR matrix on the
        block's index circle (P:L566-568's modified SOAR with theta = pi / maxval,
        standard SOAR form, reading A2; entries beyond maxval zero);
      * off-diagonal block (k, l), k < l: sparse random entries in (0, pcorr_kl)
        (pcorr_kl = 0: uncorrelated), density `density`;
      * R = (diag blocks + upper off-diagonal blocks) + transpose ("adding the diagonal
        blocks and upper half of the matrix and then symmetrising"; the diagonal
        blocks therefore count twice);
      * if lambda_min(R) < 1 the spectrum is shifted so that lambda_min = 0.41.
    pcorr defaults to U(0, 0.3) per off-diagonal block pair.  Input data only."""
    rng = np.random.Generator(np.random.PCG64(seed))
    pvec = [int(v) for v in pvec]
    p = sum(pvec)
    st = np.concatenate([[0], np.cumsum(pvec)]).astype(int)
    nb = len(pvec)
    if pcorr is None:
        pcorr = rng.uniform(0.0, 0.3, size=nb * (nb - 1) // 2)
    U = np.zeros((p, p))
    for k, n in enumerate(pvec):
        mv = maxval or max(2, n // 2)
        i = np.arange(n)
        lag = np.abs(i[:, None] - i[None, :])
        lag = np.minimum(lag, n - lag)
        d = 2.0 * np.abs(np.sin(lag * (np.pi / mv) / 2.0))
        soar = sigma * (1.0 + d / L) * np.exp(-d / L)
        soar[lag > mv] = 0.0
        rnd = rng.uniform(0.0, 1.0, size=(n, n)) * (rng.uniform(size=(n, n)) < density)
        np.fill_diagonal(rnd, 1.0)
        U[st[k]:st[k + 1], st[k]:st[k + 1]] = rnd * soar
    q = 0
    for k in range(nb):
        for l in range(k + 1, nb):
            blk = rng.uniform(0.0, 1.0, size=(pvec[k], pvec[l])) * pcorr[q]
            blk *= rng.uniform(size=blk.shape) < density
            U[st[k]:st[k + 1], st[l]:st[l + 1]] = blk
            q += 1
    R = U + U.T
    lmin = np.linalg.eigvalsh(R)[0]
    if lmin < 1.0:
        R = R + (min_eig - lmin) * np.eye(p)
    return R


def with_R(prob, R):
    """Copy of a problem with another observation covariance (same H, model, RHS
    recipe except that observation noise keeps the original R draw)."""
    import copy
    q = copy.copy(prob)
    q.R = np.array(R, dtype=np.float64)
    return q


# ---------------------------------------------------------------- NEXT-1 workload
def modified_soar_row(s, L, maxval, sigma):
    """First row of the paper's circulant modified-SOAR matrix (reading
    A2 for the parenthesis): c_i = sigma (1 + d_i/L) exp(-d_i/L),
    d_i = 2|sin(i theta/2)|, theta = pi/maxval, on the circular lag i; entries with
    circular lag >= maxval are zero (reading A29: maxval sets the number of
    non-zeros)."""
    i = np.arange(s)
    lag = np.minimum(i, s - i)
    d = 2.0 * np.abs(np.sin(lag * (np.pi / maxval) / 2.0))
    row = sigma * (1.0 + d / L) * np.exp(-d / L)
    row[lag >= maxval] = 0.0
    return row


def modified_soar_matrix(s, L, maxval, sigma, rng):
    row = modified_soar_row(s, L, maxval, sigma)
    C = np.array([np.roll(row, k) for k in range(s)])
    lmin = np.linalg.eigvalsh(C)[0]
    if lmin < 0:   # delta = |lambda_min| + psi, psi ~ U[0, 0.5]
        C = C + (abs(lmin) + rng.uniform(0.0, 0.5)) * np.eye(s)
    return C


def smoothed_H_csr(s):
    """p = s/2 observations of alternate state variables, each smoothed equally over
    5 adjacent state variables with entries 1/5 (reading A28: observed
    variables 1, 3, 5, ...; the 5-point window is clipped at the boundary)."""
    rowptr, col, val = [0], [], []
    for c in range(1, s, 2):
        for k in range(c - 2, c + 3):
            if 0 <= k < s:
                col.append(k)
                val.append(0.2)
        rowptr.append(len(col))
    return (np.array(rowptr, np.int32), np.array(col, np.int32), np.array(val, np.float64))


def paper_heat_problem(s=200, N=7, m=2, nsteps=1, r=0.4, seed0=0, pvec=None,
                       B=(0.6, 100, 0.4), Q=(0.5, 120, 0.2), with_rhs=True):
    """NEXT-1: the paper's own heat workload -- explicit Dirichlet
    forward-Euler model (r = 0.4), 5-point smoothed observations of
    alternate variables, modified-SOAR B and Q with the delta fix
    ((L, maxval, sigma) = (0.6, 100, 0.4) and (0.5, 120, 0.2)), the
    block-structured R_i (paper_block_R).  Input data only."""
    from .layout import pack as _pack
    rng0 = np.random.Generator(np.random.PCG64(10_000 + seed0))
    Bm = modified_soar_matrix(s, *B, rng0)
    Qm = modified_soar_matrix(s, *Q, rng0)
    Hc = smoothed_H_csr(s)
    p = len(Hc[0]) - 1
    if pvec is None:
        pvec = uniform_blocks(p, max(2, p // 5))
    Rm = paper_block_R(pvec, seed=20_000 + seed0)
    Hd = np.zeros((p, s))
    for j in range(p):
        Hd[j, Hc[1][Hc[0][j]:Hc[0][j + 1]]] = Hc[2][Hc[0][j]:Hc[0][j + 1]]
    Mdt = np.zeros((s, s))
    for i in range(1, s - 1):
        Mdt[i, i] = 1 - 2 * r
        if i > 1:
            Mdt[i, i - 1] = r
        if i < s - 2:
            Mdt[i, i + 1] = r
    Mw = np.linalg.matrix_power(Mdt, nsteps)   # truth/forecast propagation (synthesis)
    prob = Problem(name=f"paper_heat_s{s}_N{N}_m{m}", model="heat_explicit", s=s, p=p, N=N,
                   m=m, B=Bm, Q=Qm, R=Rm, H_idx=np.arange(p, dtype=np.int32), heat_r=r,
                   heat_nsteps=nsteps, H_csr=Hc)
    prob.extra = dict(pvec=list(pvec))
    if not with_rhs:
        return prob
    W = N + 1
    rngs = [np.random.Generator(np.random.PCG64(seed0 + j)) for j in range(m)]
    cB, cQ, cR = np.linalg.cholesky(Bm), np.linalg.cholesky(Qm), np.linalg.cholesky(Rm)
    x0t = _gaussian(rngs, cB, s)
    truth = [x0t]
    for w in range(1, W):
        truth.append(Mw @ truth[-1] + _gaussian(rngs, cQ, s))
    y = [Hd @ truth[w] + _gaussian(rngs, cR, p) for w in range(W)]
    xb = x0t + _gaussian(rngs, cB, s)
    guess = [xb]
    for w in range(1, W):
        guess.append(Mw @ guess[-1])
    eta = np.zeros((s, W, m))
    nu = np.stack([y[w] - Hd @ guess[w] for w in range(W)], axis=1)
    prob.rhs = _pack(eta, nu, np.zeros((s, W, m)))
    return prob


def uniform_blocks(p, b):
    pv = [b] * (p // b)
    if p % b:
        pv.append(p % b)
    return pv
