"""NEXT-1 oracle pins: the paper's own heat workload -- explicit
Dirichlet forward-Euler model (Supp. P:L1119-1134), 5-point smoothed
observations, modified SOAR with the delta fix."""
import numpy as np
import pytest

from oracle import models as OM
from oracle.saddle import Precond, Saddle, csr_matrix, selection_matrix
from synth import configs as SC


@pytest.mark.parametrize("s,r", [(10, 0.4), (57, 0.4), (200, 0.25), (31, 0.5)])
def test_dirichlet_step_spectrum_closed_form(s, r):
    M = OM.heat_dirichlet_step(s, r)
    assert np.array_equal(M, M.T)                       # symmetric (zero boundary rows/cols)
    assert not M[0].any() and not M[-1].any()           # P:L845-852 first/last rows zero
    lam = np.sort(np.linalg.eigvalsh(M))
    j = np.arange(1, s - 1)
    ref = np.sort(np.concatenate([1 - 4 * r * np.sin(j * np.pi / (2 * (s - 1))) ** 2, [0.0, 0.0]]))
    np.testing.assert_allclose(lam, ref, atol=1e-13)
    assert np.max(np.abs(lam)) < 1.0                    # |lambda| < 1 for r <= 1/2


def test_dirichlet_step_is_the_printed_stencil():
    s, r = 6, 0.4
    M = OM.heat_dirichlet_step(s, r)
    ref = np.array([[0, 0, 0, 0, 0, 0],
                    [0, 1 - 2 * r, r, 0, 0, 0],
                    [0, r, 1 - 2 * r, r, 0, 0],
                    [0, 0, r, 1 - 2 * r, r, 0],
                    [0, 0, 0, r, 1 - 2 * r, 0],
                    [0, 0, 0, 0, 0, 0]])
    np.testing.assert_array_equal(M, ref)
    # M between observation times = M_dt^n (Supp. P:L1134)
    np.testing.assert_allclose(OM.heat_explicit_M(s, r, 3), M @ M @ M, rtol=0, atol=1e-15)


def test_smoothed_H():
    s = 20
    rp, col, val = SC.smoothed_H_csr(s)
    H = csr_matrix(rp, col, val, s)
    assert H.shape == (s // 2, s)                       # p = s/2
    assert set(np.unique(H)) <= {0.0, 0.2}              # entries 0 or 1/5
    interior = [j for j in range(s // 2) if 2 <= 2 * j + 1 <= s - 3]
    np.testing.assert_allclose(H[interior].sum(1), 1.0)  # equal 5-point smoothing
    assert all(H[j, 2 * j + 1] == 0.2 for j in range(s // 2))   # alternate variables
    # CSR with unit entries reproduces the selection operator
    idx = np.arange(0, s, 3)
    rp1 = np.arange(len(idx) + 1, dtype=np.int32)
    np.testing.assert_array_equal(csr_matrix(rp1, idx, np.ones(len(idx)), s),
                                  selection_matrix(idx, s))


def test_modified_soar():
    s = 300
    row = SC.modified_soar_row(s, 0.6, 100, 0.4)
    assert row[0] == pytest.approx(0.4)                 # sigma at lag 0
    assert np.count_nonzero(row) == 2 * 100 - 1         # maxval sets the non-zeros
    np.testing.assert_allclose(row[1:], row[1:][::-1])  # symmetric circulant row
    C = SC.modified_soar_matrix(s, 0.6, 100, 0.4, np.random.default_rng(0))
    assert np.linalg.eigvalsh(C)[0] > 0                 # delta fix makes it SPD


def test_paper_heat_saddle_blockwise_equals_explicit():
    prob = SC.paper_heat_problem(s=40, N=4, m=1, nsteps=2)
    sad = Saddle(prob)
    v = np.random.default_rng(3).standard_normal(prob.n)
    np.testing.assert_allclose(sad.apply_A(v), sad.explicit_apply_A(v), rtol=0, atol=1e-12)
    for pc in (Precond("PD", "LM", 2, "block", pvec=tuple(prob.extra["pvec"]), block_tol=0.05),
               Precond("PI", "L", 1, "me")):
        np.testing.assert_allclose(sad.apply_Pinv(pc, v), sad.explicit_apply_Pinv(pc, v),
                                   rtol=1e-9, atol=1e-9)
