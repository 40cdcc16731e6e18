"""Pins for oracle/saddle.py, oracle/fourier.py: Eq. 2.2/2.4, Thm 3.1."""
import itertools
import json
import math
import os

import numpy as np
import pytest

from oracle import lhat as LH
from oracle import rhat as RH
from oracle import spectra as SP
from oracle.fourier import saddle_spectrum, solve_heat
from oracle.saddle import Precond, Saddle, primal_solution
from synth import configs as SC
from synth.layout import to_paper_order

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def c0():
    prob = SC.make_problem(0)
    return prob, Saddle(prob)


def small_dense():
    prob = SC.random_dense_problem(s=5, p=3, N=3, m=1, seed=7)
    return prob, Saddle(prob)


def cells(N):
    for shape, (lh, k), rh in itertools.product(
            ("PD", "PI"), (("L0", None), ("LI", None), ("LM", 1), ("LM", 2), ("LM", 3), ("L", None)),
            ("diag", "block", "rr", "me", "exact")):
        yield Precond(shape=shape, lhat=lh, k=k or 1, rhat=rh, block=2 if rh == "block" else 0)


def test_A_symmetric_and_dense_vs_blockwise(c0):
    prob, sad = c0
    A = sad.assemble_A()
    assert A.shape == (625, 625)     # BJ.c0: "Saddle system has 625 unknowns"
    np.testing.assert_array_equal(A, A.T)
    rng = np.random.default_rng(0)
    x = rng.standard_normal(625)
    np.testing.assert_allclose(sad.apply_A(x), A @ x, rtol=0, atol=1e-12 * np.linalg.norm(A @ x))


def test_spec_special_case_A():
    # D = R = I, H = 0, L = I  =>  A x = (x1 + x3, x2, x1)
    prob, sad = small_dense()
    s, p, N = sad.s, sad.p, sad.N
    sad.B = np.eye(s); sad.Q = np.eye(s); sad.R = np.eye(p)
    sad.Hi = np.zeros((p, s)); sad.Ms = [np.zeros((s, s))] * N
    x = np.random.default_rng(1).standard_normal((2 * s + p) * (N + 1))
    x1, x2, x3 = sad.split(x)
    want = sad.join([a + b for a, b in zip(x1, x3)], x2, x1)
    np.testing.assert_array_equal(sad.apply_A(x), want)
    np.testing.assert_allclose(sad.assemble_A() @ x, want, atol=1e-15)


def test_spec_special_case_PI():
    # L_hat = I, D = I  =>  P_I^{-1} x = (x3, R_hat^{-1} x2, x1 - x3)
    prob, sad = small_dense()
    s, p, N = sad.s, sad.p, sad.N
    sad.B = np.eye(s); sad.Q = np.eye(s)
    pc = Precond(shape="PI", lhat="L0", rhat="exact")
    x = np.random.default_rng(2).standard_normal((2 * s + p) * (N + 1))
    x1, x2, x3 = sad.split(x)
    want = sad.join(x3, [np.linalg.solve(sad.R, v) for v in x2], [a - b for a, b in zip(x1, x3)])
    np.testing.assert_allclose(sad.apply_Pinv(pc, x), want, atol=1e-13)
    np.testing.assert_allclose(sad.explicit_apply_Pinv(pc, x), want, atol=1e-12)


@pytest.mark.parametrize("pc", list(cells(3)), ids=lambda p: f"{p.shape}-{p.lhat}{p.k}-{p.rhat}")
def test_blockwise_P_equals_dense_solve(pc):
    prob, sad = small_dense()
    x = np.random.default_rng(3).standard_normal((2 * sad.s + sad.p) * sad.W)
    P = sad.assemble_P(pc)
    y = sad.apply_Pinv(pc, x)
    np.testing.assert_allclose(P @ y, x, atol=1e-10 * np.linalg.norm(x))
    np.testing.assert_allclose(y, sad.explicit_apply_Pinv(pc, x), rtol=1e-8,
                               atol=1e-9 * np.linalg.norm(y))
    if pc.shape == "PD":   # P_D SPD (required by preconditioned MINRES)
        np.testing.assert_allclose(P, P.T, atol=1e-12)
        assert np.linalg.eigvalsh((P + P.T) / 2)[0] > 0


def test_c0_blockwise_vs_explicit_all_cells(c0):
    prob, sad = c0
    x = np.random.default_rng(4).standard_normal(625)
    for pc in (Precond("PD", "LM", 3, "exact"), Precond("PI", "LM", 2, "me"),
               Precond("PD", "LI", 1, "block", block=5), Precond("PI", "L", 5, "rr"),
               Precond("PD", "LM", 4, "diag", ridge=0.01)):
        y = sad.apply_Pinv(pc, x)
        P = sad.assemble_P(pc)
        # backward error (P_D is very ill-conditioned here: kappa ~ 1e10)
        bwd = np.linalg.norm(P @ y - x) / (np.linalg.norm(P, 2) * np.linalg.norm(y))
        assert bwd < 1e-14, (pc, bwd)


def test_theorem31_containment_c0(c0):
    # Theorem 3.1 with all lambda terms from dense eigensolves.
    prob, sad = c0
    A = sad.assemble_A()
    D = sad.assemble_D()
    W, s = sad.W, sad.s
    import scipy.linalg as sla
    Rb = sla.block_diag(*([sad.R] * W))
    Hb = sla.block_diag(*([sad.Hi] * W))
    L = LH.assemble("L", sad.Ms, s)
    S = L.T @ np.linalg.solve(D, L) + Hb.T @ np.linalg.solve(Rb, Hb)
    St = L.T @ np.linalg.solve(D, L)
    lamS = SP.gen_eigvals_sym(S, St)
    kD = np.linalg.cond(D)
    for pc in (Precond("PD", "LM", 3, "exact"), Precond("PD", "LM", 2, "rr"),
               Precond("PD", "L0", 1, "me"), Precond("PD", "LM", 5, "diag", ridge=0.01)):
        P = sad.assemble_P(pc)
        ev = np.sort(np.real(sla.eigvals(A, P)))
        Dh = sla.block_diag(RH.dhat(sad.B, pc.ridge), *([RH.dhat(sad.Q, pc.ridge)] * sad.N))
        Rh = sla.block_diag(*([sad.rhat_matrix(pc)] * W))
        lD = SP.gen_eigvals_sym(D, Dh)
        lR = SP.gen_eigvals_sym(Rb, Rh)
        Lh = LH.assemble(pc.lhat, sad.Ms, s, pc.k)
        lL = SP.gen_eigvals_sym(L.T @ L, Lh.T @ Lh)
        iv = SP.theorem31_intervals(lD[0], lD[-1], lR[0], lR[-1], lamS[0], lamS[-1],
                                    lL[0], lL[-1], kD)
        assert np.all(SP.in_intervals(ev, iv, rtol=1e-7)), pc


def test_theorem31_collapse_when_S_hat_exact():
    # D_hat = D, R_hat = R, L_hat = L and H = 0 give S_hat = S, so all
    # eigenvalues of P_D^{-1} A lie in {(1-sqrt5)/2, 1, (1+sqrt5)/2}.
    prob, sad = small_dense()
    sad.Hi = np.zeros((sad.p, sad.s))
    import scipy.linalg as sla
    ev = np.real(sla.eigvals(sad.assemble_A(), sad.assemble_P(Precond("PD", "L", 4, "exact"))))
    targets = np.array([(1 - math.sqrt(5)) / 2, 1.0, (1 + math.sqrt(5)) / 2])
    assert np.all(np.min(np.abs(ev[:, None] - targets[None, :]), axis=1) < 1e-8)


def _attained_case(a, b, c=2.5, s=4, p=3, N=2, seed=3):
    """A saddle system on which every bound of Theorem 3.1 is attained: D = c I
    (kappa(D) = 1), D_hat = D / a and R_hat = R / a (D_hat^{-1} D = R_hat^{-1} R = a I),
    L_hat = L / sqrt(b) ((L_hat^T L_hat)^{-1} L^T L = b I), H = 0 (S = S_tilde).  Then
    P_D^{-1} A has exactly the eigenvalues a and (a -+ sqrt(a^2 + 4 a b)) / 2 (the
    eta/x block: [[a I, a L D^-1 ...]] reduces to lambda^2 - a lambda - a b = 0).
    Returns the dense eigenvalues (computed here, independently of the formula)."""
    import scipy.linalg as sla
    rng = np.random.default_rng(seed)
    W = N + 1
    Ms = [rng.standard_normal((s, s)) * 0.5 for _ in range(N)]
    L = LH.assemble("L", Ms, s)
    D = c * np.eye(s * W)
    G = rng.standard_normal((p, p))
    R1 = G @ G.T + p * np.eye(p)
    R = sla.block_diag(*([R1] * W))
    Z = np.zeros
    A = np.block([[D, Z((s * W, p * W)), L], [Z((p * W, s * W)), R, Z((p * W, s * W))],
                  [L.T, Z((s * W, p * W)), Z((s * W, s * W))]])
    Lh = L / math.sqrt(b)
    P = sla.block_diag(D / a, R / a, Lh.T @ np.linalg.solve(D, Lh))
    return np.sort(np.real(sla.eigvals(A, P)))


@pytest.mark.parametrize("a,b", [(1.0, 1.0), (0.7, 1.9), (2.3, 0.4)])
def test_theorem31_intervals_attained(a, b):
    """theorem31_intervals pinned by value: in the attained case each of the three
    intervals degenerates to a point, and the points are the dense eigenvalues of
    P_D^{-1} A (a = b = 1 is the S:L545 collapse {(1-sqrt5)/2, 1, (1+sqrt5)/2})."""
    ev = _attained_case(a, b)
    iv = SP.theorem31_intervals(a, a, a, a, 1.0, 1.0, b, b, 1.0)
    for lo, hi in iv:
        assert abs(hi - lo) <= 1e-15 * max(1.0, abs(lo))
    pts = np.array([iv[0][0], iv[1][0], iv[2][0]])
    # every eigenvalue is one of the three points, and each point is attained
    d = np.abs(ev[:, None] - pts[None, :])
    assert np.all(d.min(axis=1) < 1e-9 * max(1.0, np.abs(ev).max())), (ev, pts)
    assert np.all(d.min(axis=0) < 1e-9 * max(1.0, np.abs(ev).max())), (ev, pts)
    if a == 1.0 and b == 1.0:
        np.testing.assert_allclose(pts, [(1 - math.sqrt(5)) / 2, 1.0, (1 + math.sqrt(5)) / 2],
                                   rtol=0, atol=1e-15)


def test_saddle_equals_primal_normal_equations(c0):
    # the saddle solution's dx solves the primal normal equations.
    prob, sad = c0
    v = to_paper_order(prob.rhs, prob.s, prob.p, prob.W, 1)[0]
    s, p, W = sad.s, sad.p, sad.W
    b, d = v[:s * W], v[s * W:s * W + p * W]
    xs = np.linalg.solve(sad.assemble_A(), v)
    xp = primal_solution(sad, b, d)
    np.testing.assert_allclose(xs, xp, rtol=0, atol=1e-9 * np.linalg.norm(xp))


def test_first_guess_invariance_heat(c0):
    # Reading A3: for the linear heat model x^(0) + dx does not depend on x^(0).
    prob, sad = c0
    s, p, W = sad.s, sad.p, sad.W
    v = to_paper_order(prob.rhs, s, p, W, 1)[0]
    dx = np.linalg.solve(sad.assemble_A(), v)[(s + p) * W:]
    ex = prob.extra
    b0 = np.concatenate([ex["xb"][:, 0]] + [np.zeros(s)] * (W - 1))
    d0 = np.concatenate([ex["y"][:, w, 0] for w in range(W)])
    dx0 = np.linalg.solve(sad.assemble_A(), np.concatenate([b0, d0, np.zeros(s * W)]))[(s + p) * W:]
    guess = np.concatenate([ex["guess"][:, w, 0] for w in range(W)])
    np.testing.assert_allclose(guess + dx, dx0, atol=1e-8 * np.linalg.norm(dx0))


def test_fourier_blocks_exact(c0):
    prob, sad = c0
    A = sad.assemble_A()
    np.testing.assert_allclose(saddle_spectrum(prob), np.linalg.eigvalsh(A), atol=1e-12 * 40)
    v = to_paper_order(prob.rhs, prob.s, prob.p, prob.W, 1)
    xf = solve_heat(prob, v)[0]
    np.testing.assert_allclose(xf, np.linalg.solve(A, v[0]), atol=1e-9 * np.linalg.norm(xf))


def test_counter_identities_match_paper_tables():
    # D5 / Tables S5-S7 (N = 5): per A: R_i +W, D_i +W, M +2N; per P_D: Dhat^-1 +W,
    # Rhat^-1 +W (not counted for R_diag), D_i +W, M +2(N - floor(N/k)); per P_I: same
    # without Dhat^-1.  Iterations derived as R_i / W reproduce every column.
    rows = json.load(open(os.path.join(GOLD, "matvec_tables_heat_N5.json")))["rows"]
    prob = SC.custom_problem(s=8, N=5, q=2, m=1)
    sad = Saddle(prob)
    W = sad.W
    x = np.random.default_rng(0).standard_normal((2 * sad.s + sad.p) * W)
    for row in rows:
        pc = Precond(shape=row["shape"], lhat="LM", k=row["k"], rhat=row["rhat"], block=2)
        sad.counters = dict(R=0, Rhat_inv=0, D=0, Dhat_inv=0, M=0)
        sad.apply_A(x)
        sad.apply_Pinv(pc, x)
        if pc.rhat == "diag":
            sad.counters["Rhat_inv"] = 0
        it = row["R"] // W
        assert it * W == row["R"]
        c = sad.counters
        assert it * c["R"] == row["R"] and it * c["D"] == row["D"] and it * c["M"] == row["M"], row
        if "Dhat_inv" in row:
            assert it * c["Dhat_inv"] == row["Dhat_inv"]
        else:
            assert c["Dhat_inv"] == 0
        if "Rhat_inv" in row:
            assert it * c["Rhat_inv"] == row["Rhat_inv"]
