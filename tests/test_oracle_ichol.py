"""Pins for oracle/ichol.py (IC(0), Matlab ichol 'nofill', P:L572 / P:L600)."""
import numpy as np
import pytest
import scipy.linalg as sla

from oracle import ichol as IC
from synth import configs as SC


def test_defining_property_on_the_pattern_and_dropped_fill():
    # circulant compact-support SOAR (wrap-around corners): fill outside the pattern is dropped
    A = SC.modified_soar_matrix(60, 0.6, 8, 0.4, np.random.default_rng(0)) + 0.1 * np.eye(60)
    L = IC.ichol0(A)
    P = np.tril(A != 0)
    assert np.all(L[~P] == 0.0)                                   # pattern of tril(A)
    LLt = L @ L.T
    np.testing.assert_allclose(LLt[P], A[P], rtol=1e-12, atol=1e-14)   # (LL^T)_ij = A_ij on P
    assert np.abs(LLt - A).max() > 1e-6                           # ... and only there


def test_banded_matrix_without_wrap_is_exact_cholesky():
    # the Cholesky factor of a banded matrix stays inside the band: nothing is dropped
    n, b = 50, 4
    rng = np.random.default_rng(1)
    A = np.zeros((n, n))
    for i in range(n):
        for j in range(max(0, i - b), i + 1):
            A[i, j] = A[j, i] = rng.uniform(-0.2, 0.2)
    A += np.diag(np.abs(A).sum(1) + 1.0)
    np.testing.assert_allclose(IC.ichol0(A), np.linalg.cholesky(A), rtol=1e-12, atol=1e-14)


def test_dense_matrix_is_exact_cholesky_and_hand_example():
    rng = np.random.default_rng(2)
    X = rng.standard_normal((20, 20))
    A = X @ X.T + 20 * np.eye(20)
    np.testing.assert_allclose(IC.ichol0(A), np.linalg.cholesky(A), rtol=1e-12)
    A3 = np.array([[4.0, 2.0, 0.0], [2.0, 5.0, 1.0], [0.0, 1.0, 3.0]])
    L3 = np.array([[2.0, 0.0, 0.0], [1.0, 2.0, 0.0], [0.0, 0.5, np.sqrt(2.75)]])
    np.testing.assert_allclose(IC.ichol0(A3), L3, rtol=1e-15)


def test_nonpositive_pivot_raises():
    with pytest.raises(np.linalg.LinAlgError):
        IC.ichol0(np.array([[1.0, 2.0], [2.0, 1.0]]))
