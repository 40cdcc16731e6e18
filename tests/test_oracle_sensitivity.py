"""Reading A35: the oracle's own solution spread under rounding-level noise.

configs[0] with P_I, L_M(5), R_hat = R under GMRES(50) to relres 1e-10 is a cell where two
correct FP64 solves differ by more than north_star's 1e-9: the oracle against itself,
with 1e-15 relative noise on every P^{-1} output, already moves the solution by > 1e-9.
A well-conditioned cell (P_I, L_M(1), R_hat = R, GMRES(20)) stays far below 1e-9.  These
pins keep the GPU tests' fallback bound (2x this spread) from being vacuous."""
import numpy as np

from oracle import krylov as KR
from oracle.saddle import Saddle
from synth import configs as SC
from synth.layout import to_paper_order

from .helpers import oracle_precond, oracle_solution_spread


def _cell(k, restart):
    prob = SC.make_problem(0)
    sad = Saddle(prob)
    bp = to_paper_order(prob.rhs, prob.s, prob.p, prob.W, 1)[0]
    opc = oracle_precond(dict(shape="PI", lhat="LM", k=k, rhat="exact"))
    P = lambda v: sad.apply_Pinv(opc, v)
    x0, info = KR.gmres(sad.apply_A, P, bp, tol=1e-10, restart=restart, maxit=5000)
    assert info["converged"]
    return oracle_solution_spread(KR.gmres, sad.apply_A, P, bp, x0, tol=1e-10, restart=restart,
                                  maxit=5000)


def test_spread_exceeds_1e9_on_the_sensitive_cell():
    assert _cell(5, 50) > 1e-9


def test_spread_small_on_a_well_conditioned_cell():
    assert _cell(1, 20) < 1e-11
