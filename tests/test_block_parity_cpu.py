"""The per-block parity check (tests/helpers.block_parity) itself:
it must pass the oracle's own output and catch (i) a D_hat^{-1} applied as a product
with a computed explicit inverse (not backward stable, reading A32), (ii) a 1e-10
error in a product-only block, (iii) a dropped R_hat^{-1} window.  CPU only."""
import numpy as np
import scipy.linalg as sla

from synth import configs as SC
from synth.layout import from_paper_order, to_paper_order

from .helpers import OracleCols, block_parity, smooth_vec


def _setup(pc):
    prob = SC.custom_problem(s=300, N=2, q=2, m=2, seed0=4, Bp=(0.05, 1.0), Qp=(0.05, 0.1),
                             Rp=(0.03, 0.05))
    ora = OracleCols(prob)
    x = smooth_vec(prob, 3)
    ref = ora.apply_P(pc, x)
    Y = np.stack([ref[c] for c in range(prob.m)])
    return prob, ora, x, Y


def test_oracle_output_passes():
    for pc in (dict(shape="PD", lhat="LM", k=2, rhat="exact"),
               dict(shape="PI", lhat="LM", k=2, rhat="me"),
               dict(shape="PD", lhat="L", k=1, rhat="diag")):
        prob, ora, x, Y = _setup(pc)
        y = from_paper_order(Y, prob.s, prob.p, prob.W)
        fails, worst = block_parity(prob, pc, x, y, ora, range(prob.m))
        assert not fails, fails
        assert worst["Dhat_inv bwd" if pc["shape"] == "PD" else "Rhat_inv bwd"] < 1e-15


def test_explicit_inverse_fails_backward_error():
    pc = dict(shape="PD", lhat="LM", k=2, rhat="exact")
    prob, ora, x, Y = _setup(pc)
    s, W = prob.s, prob.W
    X = to_paper_order(x, prob.s, prob.p, W, prob.m)
    G = np.linalg.cholesky(prob.Q)
    Gi = sla.solve_triangular(G, np.eye(s), lower=True)
    Qinv = Gi.T @ Gi
    for c in range(prob.m):
        for w in range(1, W):
            Y[c, w * s:(w + 1) * s] = Qinv @ X[c, w * s:(w + 1) * s]
    fails, worst = block_parity(prob, pc, x, from_paper_order(Y, prob.s, prob.p, W), ora,
                                range(prob.m))
    assert any("D_hat^-1 bwd" in f for f in fails), worst
    assert not any("fwd" in f for f in fails), fails   # forward error is kappa u: passes


def test_product_block_error_and_dropped_window_caught():
    pc = dict(shape="PI", lhat="LM", k=2, rhat="exact")
    prob, ora, x, Y = _setup(pc)
    s, p, W = prob.s, prob.p, prob.W
    Y2 = Y.copy()
    Y2[0, :s] *= 1 + 1e-10                    # c1 = L_hat^{-T} x3, window 0
    fails, _ = block_parity(prob, pc, x, from_paper_order(Y2, s, p, W), ora, [0])
    assert any("L_hat^-T" in f for f in fails), fails
    Y3 = Y.copy()
    o = s * W
    Y3[1, o + p:o + 2 * p] = to_paper_order(x, s, p, W, prob.m)[1, o + p:o + 2 * p]
    fails, _ = block_parity(prob, pc, x, from_paper_order(Y3, s, p, W), ora, [1])
    assert any("R_hat^-1" in f for f in fails), fails
