"""Pins for oracle/rhat.py: Algorithms 1-3 and Lemmas 5.1/5.2."""
import numpy as np
import pytest

from oracle import rhat as RH
from oracle import spectra as SP
from synth import configs as SC


def spd(n, seed):
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((n, n))
    return A @ A.T / n + 0.1 * np.eye(n)


@pytest.mark.parametrize("R", [spd(30, 1), SC.make_problem(0, with_rhs=False).R])
def test_lemma51_rr_spectral_map(R):
    lam = np.linalg.eigvalsh(R)
    for gamma in (None, 0.3):
        Rrr, g = RH.r_rr(R, gamma)
        got = np.sort(SP.gen_eigvals_sym(R, Rrr))
        np.testing.assert_allclose(got, np.sort(SP.lemma51_map(lam, g)), atol=1e-10)
        assert np.all((got > 0) & (got < 1))


@pytest.mark.parametrize("R", [spd(30, 2), SC.make_problem(0, with_rhs=False).R])
def test_lemma52_me_spectral_map(R):
    lam = np.linalg.eigvalsh(R)
    for T in (None, float(np.median(lam))):
        Rme, TT = RH.r_me(R, T)
        got = np.sort(SP.gen_eigvals_sym(R, Rme))
        np.testing.assert_allclose(got, np.sort(SP.lemma52_map(lam, TT)), atol=1e-10)
        assert abs(got[-1] - 1.0) < 1e-10   # lambda_max(R_ME^{-1} R) = 1


def test_auto_T_changes_only_the_smallest_distinct_eigenvalue():
    # T = second smallest eigenvalue, "only a single eigenvalue is changed".
    R = spd(25, 4)
    Rme, T = RH.r_me(R)
    got = np.sort(SP.gen_eigvals_sym(R, Rme))
    assert np.sum(got < 1 - 1e-10) == 1
    # c0's circulant R (odd p = 25): the smallest eigenvalue is a degenerate pair,
    # so the "single" distinct eigenvalue has multiplicity 2 (reading A6).
    Rc = SC.make_problem(0, with_rhs=False).R
    Rme, T = RH.r_me(Rc)
    got = np.sort(SP.gen_eigvals_sym(Rc, Rme))
    assert np.sum(got < 1 - 1e-10) == 2


def test_algorithm1_block():
    R = spd(12, 5)
    pvec = [3, 3, 3, 3]
    # tol = 0: every norm >= 0 -> no cut -> R_block = R
    Rb, blocks, _ = RH.r_block(R, pvec, tol=0.0)
    np.testing.assert_array_equal(Rb, R)
    # tol = inf: every cut -> block diagonal with blocks pvec
    Rb, blocks, _ = RH.r_block(R, pvec, tol=np.inf)
    assert blocks == [(0, 3), (3, 6), (6, 9), (9, 12)]
    for a, b in blocks:
        np.testing.assert_array_equal(Rb[a:b, a:b], R[a:b, a:b])
    assert np.count_nonzero(Rb) == 4 * 9
    # SPEC S:L362 hand trace: norms (0.5, 0.05, 0.7), tol 0.1 -> one cut after block 2,
    # keeping the (1,2) and (3,4) couplings (incl. nothing across the cut).
    R2 = np.eye(8) * 3.0
    vals = [0.5, 0.05, 0.7]
    for j, v in enumerate(vals):
        a, b = 2 * j, 2 * (j + 1)
        R2[a:a + 2, b:b + 2] = v
        R2[b:b + 2, a:a + 2] = v
    R2[0:2, 6:8] = R2[6:8, 0:2] = 0.01
    Rb, blocks, normvec = RH.r_block(R2, [2, 2, 2, 2], tol=0.1)
    np.testing.assert_allclose(normvec, vals)
    assert blocks == [(0, 4), (4, 8)]
    np.testing.assert_array_equal(Rb[0:4, 0:4], R2[0:4, 0:4])
    np.testing.assert_array_equal(Rb[4:8, 4:8], R2[4:8, 4:8])
    assert not Rb[0:4, 4:8].any() and not Rb[4:8, 0:4].any()


def test_uniform_pvec_and_diag():
    assert RH.uniform_pvec(25, 5) == [5] * 5
    assert RH.uniform_pvec(26, 5) == [5] * 5 + [1]
    R = spd(6, 9)
    np.testing.assert_array_equal(RH.r_diag(R), np.diag(np.diag(R)))
