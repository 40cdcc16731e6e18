"""GPU parity on NEXT-1: the paper's own heat workload -- explicit
Dirichlet forward-Euler M = M_dt^n, 5-point smoothed H as CSR
(P:L561), modified SOAR B/Q, block-structured R_i --
through the C ABI against the oracle."""
import numpy as np
import pytest

from oracle import krylov as KR
from oracle import rhat as RH
from synth import configs as SC
from synth.layout import to_paper_order

from .helpers import OracleCols, oracle_precond, rel_err_cols, seeded_vec

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
U = 2.220446049250313e-16


def WF():
    import paper_2105_06975_b200 as W
    return W


_cache = {}


def get(nsteps, s=200, N=7, m=3):
    key = (nsteps, s, N, m)
    if key not in _cache:
        prob = SC.paper_heat_problem(s=s, N=N, m=m, nsteps=nsteps)
        _cache[key] = (prob, OracleCols(prob))
    return _cache[key]


def cells(prob):
    pv = prob.extra["pvec"]
    return [dict(shape="PD", lhat="LM", k=3, rhat="exact"),
            dict(shape="PD", lhat="LM", k=2, rhat="block", pvec=pv, block_tol=0.05),
            dict(shape="PI", lhat="L", k=1, rhat="me"),
            dict(shape="PI", lhat="LI", k=1, rhat="rr"),
            dict(shape="PD", lhat="L0", k=1, rhat="diag", ridge=0.01)]


def kappa(prob, pc):
    ks = [np.linalg.cond(prob.B + pc.get("ridge", 0.0) * np.eye(prob.s))]
    if pc["rhat"] == "block":
        ks.append(np.linalg.cond(RH.r_block(prob.R, pc["pvec"], pc["block_tol"])[0]))
    elif pc["rhat"] != "diag":
        ks.append(np.linalg.cond(prob.R))
    return max(ks)


@pytest.mark.parametrize("nsteps", [1, 3, 8])
def test_apply_A_and_P(nsteps):
    prob, ora = get(nsteps)
    x = seeded_vec(prob.n, 2)
    for pc in cells(prob):
        ctx = WF().Context.from_problem(prob, pc)
        y = torch.empty(prob.n, dtype=torch.float64, device="cuda")
        ctx.apply_A(torch.from_numpy(x).cuda(), y)
        torch.cuda.synchronize()
        errs = rel_err_cols(y.cpu().numpy(), ora.apply_A(x), prob)
        assert max(errs.values()) <= 1e-12, (pc, errs)
        ctx.apply_P(torch.from_numpy(x).cuda(), y)
        torch.cuda.synchronize()
        errs = rel_err_cols(y.cpu().numpy(), ora.apply_P(pc, x), prob)
        assert max(errs.values()) <= max(1e-12, 50 * kappa(prob, pc) * U), (pc, errs)


@pytest.mark.parametrize("solver,pc", [("minres", dict(shape="PD", lhat="LM", k=3, rhat="exact")),
                                       ("gmres", dict(shape="PI", lhat="LM", k=2, rhat="me"))])
def test_solve(solver, pc):
    prob, ora = get(2, N=5, m=2)
    ctx = WF().Context.from_problem(prob, pc)
    b = torch.from_numpy(prob.rhs).cuda()
    x = torch.empty_like(b)
    rep = ctx.solve(b, x, solver=solver, tol=1e-10, maxit=3000, restart=0)
    B = to_paper_order(prob.rhs, prob.s, prob.p, prob.W, prob.m)
    X = to_paper_order(x.cpu().numpy(), prob.s, prob.p, prob.W, prob.m)
    opc = oracle_precond(pc)
    for c in range(prob.m):
        sad = ora.sad[c]
        if solver == "minres":
            xo, info = KR.minres(sad.apply_A, lambda v: sad.apply_Pinv(opc, v), B[c], tol=1e-10,
                                 maxit=3000)
        else:
            xo, info = KR.gmres(sad.apply_A, lambda v: sad.apply_Pinv(opc, v), B[c], tol=1e-10,
                                restart=3000, maxit=3000)
        assert rep["converged"][c] and info["converged"]
        assert np.linalg.norm(X[c] - xo) / np.linalg.norm(xo) <= 1e-9
        xstar = np.linalg.solve(sad.assemble_A(), B[c])
        assert np.linalg.norm(X[c] - xstar) / np.linalg.norm(xstar) <= 1e-7


def test_sharded_matches_single_rank():
    from .test_gpu_dist import Sharded, apply1, rel
    prob, _ = get(3)
    for pc in cells(prob)[:3]:
        one = WF().Context.from_problem(prob, pc)
        sh = Sharded(prob, pc, 3)
        try:
            x = seeded_vec(prob.n, 9)
            for which in ("apply_A", "apply_P"):
                assert rel(sh.apply(which, x), apply1(one, which, x)) <= 1e-13
        finally:
            sh.close()
            one.close()
