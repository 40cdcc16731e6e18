"""Seeded synthetic inputs shared by the CPU oracle (tests) and the CUDA path.

This package builds PROBLEM DATA only: the covariance blocks B, Q, R, the
observation selection H_idx, the model description (heat parameter r, or a
Lorenz-96 linearisation trajectory) and the right-hand sides (b, d, 0).
It contains none of the method's arithmetic (no saddle operator, no
preconditioner, no Krylov step, no tangent-linear model): those live
independently in ``oracle/`` (test infrastructure) and in the CUDA library.

The recipe follows BASELINE.json ``configs`` with the readings recorded in
DESIGN.md ("Input recipe"): chordal SOAR distance (reading A1), the standard
SOAR form var*(1+d/L)exp(-d/L) (A2), the first-guess RHS linearisation (A3),
every-q-th-point selection H (A14), PCG64 seeds per RHS column (A15).
"""
from .configs import CONFIGS, make_problem, custom_problem  # noqa: F401
from .layout import pack, unpack, to_paper_order, from_paper_order  # noqa: F401
