"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct float64 NumPy/SciPy implementation of what the
hot path computes, written from PAPER.md (arXiv 2105.06975, Tabeart & Pearson).
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import it.  The product path
(``paper_2105_06975_b200``) never imports, links or executes anything here, and
this package never imports the product path: the two share no code.  Shared
seeded inputs come from ``synth/`` which holds none of the method's arithmetic.

Modules
  models   heat step M = (I - r Lap)^{-1} (dense), Lorenz-96 rhs/RK4 and the
           exact tangent linear of the discrete RK4 map (dense Jacobian).
  lhat     L, L_0, L_I, L_M(k) assembled densely (Eq. 2.3, Def. 4.1) and the
           chain substitution of Lemma 4.2 written out literally.
  rhat     R_diag, R_block (Alg. 1), R_RR (Alg. 2), R_ME (Alg. 3) as dense
           matrices from their definitions; D_hat (ridge).
  saddle   explicit assembly of A (Eq. 2.2), P_D, P_I (Eq. 2.4) and dense
           applies; blockwise applies following P:L629-667 with counters.
  krylov   preconditioned MINRES (ESW recurrence, 2-norm residual tracking)
           and right-preconditioned restarted GMRES (CGS2 or MGS).
  spectra  Theorem 3.1 intervals, Prop. 4.4 unit count, Prop. 4.5 / Remark
           bounds, Supp. Prop. S5 closed form, Lemma 5.1/5.2 maps.
  fourier  exact Fourier-block decomposition of the heat configs (circulant
           B, Q, R, M and uniform selection H).

Parity status per function is recorded in DESIGN.md ("Oracle pins").
"""
