"""Exact Fourier-block form of the heat configurations (ORACLE, tests only).

For BJ.c0/c1/c3/c4 every block is circulant (B, Q, R: SOAR on a uniform
periodic grid; M = (I - r Lap)^{-1}) and H selects every q-th point starting
at index 0.  With the unitary DFT, observation mode l (0 <= l < p) couples only
to the state modes K_l = {l + t p : t = 0..q-1} with weight 1/sqrt(q):
    (H x)^_l = q^{-1/2} sum_t x^_{l + t p}.
So A = [[D,0,L],[0,R,H],[L^T,H^T,0]] splits into p independent real symmetric
blocks of size (2q+1)W.  Solving every block and transforming back gives the
exact x* = A^{-1} rhs at full size, independent of any Krylov method
(SURVEY 8(c)-C2).  Eigenvalues of a symmetric circulant with first row c are
the real DFT of c; the heat step has mu_k = 1 / (1 + 4 r sin^2(pi k / s)).
"""
import numpy as np


def circ_eigs(first_row):
    return np.real(np.fft.fft(first_row))


def heat_mu(s, r):
    k = np.arange(s)
    return 1.0 / (1.0 + 4.0 * r * np.sin(np.pi * k / s) ** 2)


def _check_uniform(prob):
    s, p = prob.s, prob.p
    q = s // p
    assert q * p == s and np.array_equal(prob.H_idx, np.arange(0, s, q)), "needs uniform H"
    return q


def block_matrix(bk, qk, r_l, mu, W, q):
    """Real symmetric (2q+1)W block for one observation mode.
    bk, qk, mu: length-q arrays over the coupled state modes; r_l scalar."""
    n1 = q * W
    n = 2 * n1 + W
    A = np.zeros((n, n))
    iE = lambda t, w: w * q + t              # eta (state mode t, window w)
    iN = lambda w: n1 + w                    # nu (window w)
    iX = lambda t, w: n1 + W + w * q + t     # x
    h = 1.0 / np.sqrt(q)
    for w in range(W):
        A[iN(w), iN(w)] = r_l
        for t in range(q):
            A[iE(t, w), iE(t, w)] = bk[t] if w == 0 else qk[t]
            # L: identity diagonal, -mu on (w, w-1)
            A[iE(t, w), iX(t, w)] = 1.0
            A[iX(t, w), iE(t, w)] = 1.0
            if w >= 1:
                A[iE(t, w), iX(t, w - 1)] = -mu[t]
                A[iX(t, w - 1), iE(t, w)] = -mu[t]
            A[iN(w), iX(t, w)] = h
            A[iX(t, w), iN(w)] = h
    return A


def solve_heat(prob, rhs_cols):
    """Exact A^{-1} rhs for a heat problem.
    rhs_cols: [m][(2s+p)W] paper-ordered real vectors.  Returns same shape."""
    s, p, N = prob.s, prob.p, prob.N
    W = N + 1
    q = _check_uniform(prob)
    b_hat = circ_eigs(prob.B[0])
    q_hat = circ_eigs(prob.Q[0])
    r_hat = circ_eigs(prob.R[0])
    mu = heat_mu(s, prob.heat_r)
    rhs_cols = np.atleast_2d(rhs_cols)
    m = rhs_cols.shape[0]
    out = np.zeros_like(rhs_cols)
    for col in range(m):
        v = rhs_cols[col]
        eta = v[:s * W].reshape(W, s)
        nu = v[s * W:s * W + p * W].reshape(W, p)
        xx = v[s * W + p * W:].reshape(W, s)
        E = np.fft.fft(eta, axis=1, norm="ortho")
        Nn = np.fft.fft(nu, axis=1, norm="ortho")
        X = np.fft.fft(xx, axis=1, norm="ortho")
        Es = np.zeros_like(E)
        Ns = np.zeros_like(Nn)
        Xs = np.zeros_like(X)
        for l in range(p):
            ks = l + p * np.arange(q)
            A = block_matrix(b_hat[ks], q_hat[ks], r_hat[l], mu[ks], W, q)
            rhs = np.concatenate([E[:, ks].ravel(), Nn[:, l], X[:, ks].ravel()])
            sol = np.linalg.solve(A, rhs)
            n1 = q * W
            Es[:, ks] = sol[:n1].reshape(W, q)
            Ns[:, l] = sol[n1:n1 + W]
            Xs[:, ks] = sol[n1 + W:].reshape(W, q)
        eta_s = np.real(np.fft.ifft(Es, axis=1, norm="ortho"))
        nu_s = np.real(np.fft.ifft(Ns, axis=1, norm="ortho"))
        x_s = np.real(np.fft.ifft(Xs, axis=1, norm="ortho"))
        out[col] = np.concatenate([eta_s.ravel(), nu_s.ravel(), x_s.ravel()])
    return out


def saddle_spectrum(prob):
    """All eigenvalues of A for a heat problem (union over the p blocks)."""
    s, p, N = prob.s, prob.p, prob.N
    W = N + 1
    q = _check_uniform(prob)
    b_hat, q_hat, r_hat = circ_eigs(prob.B[0]), circ_eigs(prob.Q[0]), circ_eigs(prob.R[0])
    mu = heat_mu(s, prob.heat_r)
    ev = []
    for l in range(p):
        ks = l + p * np.arange(q)
        ev.append(np.linalg.eigvalsh(block_matrix(b_hat[ks], q_hat[ks], r_hat[l], mu[ks], W, q)))
    return np.sort(np.concatenate(ev))
