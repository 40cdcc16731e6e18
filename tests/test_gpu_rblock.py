"""GPU parity of R_block built by Algorithm 1 in full (variable block
sizes, tol, maxsize, numproc) on the paper's block-structured R_i,
through the C ABI, against the oracle (dense solves with the oracle's own
Algorithm 1 matrix)."""
import numpy as np
import pytest

from oracle import rhat as RH
from synth import configs as SC
from synth.layout import to_paper_order

from .helpers import OracleCols, rel_err_cols, seeded_vec

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
U = 2.220446049250313e-16
PV = [20, 30, 10, 25, 15]


def problem():
    base = SC.custom_problem(s=200, N=5, q=2, m=3, seed0=4)
    return SC.with_R(base, SC.paper_block_R(PV, seed=7))


@pytest.mark.parametrize("tol,maxsize,numproc", [(np.inf, 0, 0), (0.03, 0, 0), (0.03, 40, 0),
                                                 (0.0, 0, 0), (0.04, 0, 2), (np.inf, 0, 9)])
@pytest.mark.parametrize("shape", ["PD", "PI"])
def test_apply_P_algorithm1_rblock(tol, maxsize, numproc, shape):
    import paper_2105_06975_b200 as W
    prob = problem()
    pc = dict(shape=shape, lhat="LM", k=3, rhat="block", pvec=PV, block_tol=tol,
              maxsize=maxsize, numproc=numproc)
    ctx = W.Context.from_problem(prob, pc)
    ora = OracleCols(prob)
    x = seeded_vec(prob.n, 5)
    y = torch.empty(prob.n, dtype=torch.float64, device="cuda")
    ctx.apply_P(torch.from_numpy(x).cuda(), y)
    torch.cuda.synchronize()
    Rb = RH.r_block(prob.R, PV, tol, maxsize or None, numproc or None)[0]
    kap = max(np.linalg.cond(Rb), np.linalg.cond(prob.B), np.linalg.cond(prob.Q))
    errs = rel_err_cols(y.cpu().numpy(), ora.apply_P(pc, x), prob)
    assert max(errs.values()) <= max(1e-12, 50 * kap * U), errs


def test_solve_with_algorithm1_rblock():
    import paper_2105_06975_b200 as W
    from oracle import krylov as KR
    from .helpers import oracle_precond
    prob = problem()
    pc = dict(shape="PI", lhat="LM", k=3, rhat="block", pvec=PV, block_tol=0.03, numproc=4)
    ctx = W.Context.from_problem(prob, pc)
    b = torch.from_numpy(prob.rhs).cuda()
    x = torch.empty_like(b)
    rep = ctx.solve(b, x, solver="gmres", tol=1e-10, maxit=2000, restart=0)
    ora = OracleCols(prob)
    B = to_paper_order(prob.rhs, prob.s, prob.p, prob.W, prob.m)
    X = to_paper_order(x.cpu().numpy(), prob.s, prob.p, prob.W, prob.m)
    opc = oracle_precond(pc)
    for c in range(prob.m):
        sad = ora.sad[c]
        xo, info = KR.gmres(sad.apply_A, lambda v: sad.apply_Pinv(opc, v), B[c], tol=1e-10,
                            restart=2000, maxit=2000)
        assert rep["converged"][c] and info["converged"]
        assert np.linalg.norm(X[c] - xo) / np.linalg.norm(xo) <= 1e-9
