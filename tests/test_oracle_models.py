"""Pins for oracle/models.py against the paper's formulas and the mathematics."""
import math

import numpy as np
import pytest

from oracle import models as OM
from synth import configs as SC


def test_l96_rhs_worked_example():
    # dx_i/dt = (x_{i+1}-x_{i-2})x_{i-1} - x_i + 8, periodic.
    # s=4, x=(1,2,3,4): (x_1 - x_{-2}) x_{-1} - x_0 + 8 = (2-3)*4 - 1 + 8 = 3
    assert OM.l96_rhs(np.array([1.0, 2.0, 3.0, 4.0]), 8.0)[0] == 3.0


def test_l96_fixed_point():
    x = np.full(40, 8.0)
    assert np.all(OM.l96_rhs(x, 8.0) == 0.0)
    np.testing.assert_array_equal(OM.l96_rk4_step(x, 0.025, 8.0), x)


def test_l96_rk4_matches_independent_vectorised_rk4():
    rng = np.random.default_rng(3)
    x = 8 + rng.standard_normal(40)
    a = OM.l96_rk4_step(x, 0.025, 8.0)
    b = SC._l96_rk4(x[:, None], 0.025, 8.0)[:, 0]   # synth's vectorised RK4
    np.testing.assert_allclose(a, b, rtol=0, atol=1e-13)


def test_l96_tlm_is_derivative_of_rk4_map():
    # TLM = exact derivative of 5 RK4 substeps (BJ.c2): central FD.
    rng = np.random.default_rng(5)
    x0 = 8 + rng.standard_normal(40)
    for _ in range(200):
        x0 = OM.l96_rk4_step(x0, 0.025)
    M = OM.l96_tlm(x0, 0.025, 5)
    v = rng.standard_normal(40)
    eps = 1e-5

    def flow(x):
        for _ in range(5):
            x = OM.l96_rk4_step(x, 0.025)
        return x

    fd = (flow(x0 + eps * v) - flow(x0 - eps * v)) / (2 * eps)
    assert np.linalg.norm(M @ v - fd) / np.linalg.norm(fd) < 1e-6
    # dt -> 0 consistency: M -> I
    Ms = OM.l96_tlm(x0, 1e-8, 1)
    assert np.abs(Ms - np.eye(40)).max() < 1e-6


def test_heat_M_closed_forms():
    s, r = 50, 0.25
    M = OM.heat_M(s, r)
    # symmetric circulant
    np.testing.assert_allclose(M, M.T, atol=1e-15)
    # M (I - r Lap) = I
    np.testing.assert_allclose(M @ (np.eye(s) - r * OM.heat_lap(s)), np.eye(s), atol=1e-14)
    # eigenvalues 1/(1+4 r sin^2(pi j/s)) in [1/(1+4r), 1]
    ev = np.sort(np.linalg.eigvalsh(M))
    j = np.arange(s)
    ref = np.sort(1.0 / (1.0 + 4 * r * np.sin(np.pi * j / s) ** 2))
    np.testing.assert_allclose(ev, ref, atol=1e-14)
    # first row: periodic sum of the infinite-line Green's function rho^|d|/sqrt(1+4r)
    rho = (1 + 2 * r - math.sqrt(1 + 4 * r)) / (2 * r)
    d = np.arange(s)
    row = (rho ** d + rho ** (s - d)) / ((1 - rho ** s) * math.sqrt(1 + 4 * r))
    np.testing.assert_allclose(M[0], row, atol=1e-15)
    np.testing.assert_allclose(M[0, :3], [0.70711, 0.12132, 0.020815], rtol=1e-4)


def test_soar_chordal_spd_and_circulant_eigs():
    for cfg in (0, 1):
        prob = SC.make_problem(cfg, with_rhs=False)
        for C in (prob.B, prob.Q, prob.R):
            ev = np.linalg.eigvalsh(C)
            assert ev[0] > 0
            # circulant eigenvalues = DFT of the first row
            np.testing.assert_allclose(np.sort(ev), np.sort(np.real(np.fft.fft(C[0]))),
                                       atol=1e-12 * ev[-1])
