"""Banded covariances (SURVEY 8(f) NEXT-1 follow-up): the compact-support modified
SOAR B, Q (non-zero only for circular lag < maxval) and the
block-structured R_i of the paper's workload, at s large enough that a
64-row tile meets only a band of columns.  The library registers the column ranges
of these matrices and of their Cholesky / IC(0) factors and its DMMA GEMM / TRSM
kernels skip the zero K tiles.  Checked here: (i) applies and solves agree with the
oracle; (ii) the skipped work is really skipped (the library's own flop counters
drop to the band's share); (iii) the result is identical to the dense K loop
(WF4DVAR_BANDED=0) -- the skipped terms are exact zeros and the K tiles that remain
keep their order (at equal TRSM blocking: narrow-band factors otherwise take a single
panel walk, which regroups the same sums)."""
import os
import subprocess
import sys

import numpy as np
import pytest

from synth import configs as SC

from .helpers import OracleCols, rel_err_cols, seeded_vec

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def WF():
    import paper_2105_06975_b200 as W
    return W


_cache = {}


def get():
    if "p" not in _cache:
        prob = SC.paper_heat_problem(s=1024, N=3, m=2, nsteps=2)
        _cache["p"] = (prob, OracleCols(prob))
    return _cache["p"]


def cells(prob):
    pv = prob.extra["pvec"]
    return [dict(shape="PD", lhat="LM", k=2, rhat="exact"),
            dict(shape="PD", lhat="LM", k=2, rhat="block", pvec=pv, block_tol=0.05),
            dict(shape="PD", lhat="LM", k=2, rhat="exact", factor="ichol", ridge=0.01),
            dict(shape="PI", lhat="LM", k=2, rhat="rr")]


def test_band_is_narrow():
    prob, _ = get()
    nz = (prob.B != 0).sum(1)
    assert nz.max() < 0.25 * prob.s   # 199 of 1024 columns per row


@pytest.mark.parametrize("i", range(4))
def test_apply_parity(i):
    prob, ora = get()
    pc = cells(prob)[i]
    x = seeded_vec(prob.n, 11)
    ctx = WF().Context.from_problem(prob, pc)
    y = torch.empty(prob.n, dtype=torch.float64, device="cuda")
    ctx.apply_A(torch.from_numpy(x).cuda(), y)
    torch.cuda.synchronize()
    errs = rel_err_cols(y.cpu().numpy(), ora.apply_A(x), prob)
    assert max(errs.values()) <= 1e-12, errs
    ctx.apply_P(torch.from_numpy(x).cuda(), y)
    torch.cuda.synchronize()
    errs = rel_err_cols(y.cpu().numpy(), ora.apply_P(pc, x), prob)
    assert max(errs.values()) <= 1e-9, (pc, errs)
    ctx.close()


def test_flop_counters_show_the_band():
    prob, _ = get()
    ctx = WF().Context.from_problem(prob, cells(prob)[0])
    x = torch.from_numpy(seeded_vec(prob.n, 3)).cuda()
    y = torch.empty_like(x)
    ctx.profile_enable(True)
    ctx.apply_A(x, y)
    prof = ctx.profile_read()
    ctx.profile_enable(False)
    ncol = prob.W * prob.m
    dense = 2.0 * prob.s * prob.s * ncol + 2.0 * prob.p * prob.p * ncol   # D x1 and R x2
    got = prof["gemm_dmma"]["flops"]
    assert 0 < got < 0.5 * dense, (got, dense)   # B, Q tiles: ~0.3 of dense; R: dense
    ctx.close()


SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_2105_06975_b200 as W
from synth import configs as SC
prob = SC.paper_heat_problem(s=1024, N=3, m=2, nsteps=2)
x = torch.from_numpy(np.random.Generator(np.random.PCG64(5)).standard_normal(prob.n)).cuda()
outs = []
for pc in (dict(shape="PD", lhat="LM", k=2, rhat="exact"),
           dict(shape="PD", lhat="LM", k=2, rhat="exact", factor="ichol", ridge=0.01),
           dict(shape="PI", lhat="LM", k=2, rhat="rr")):
    ctx = W.Context.from_problem(prob, pc)
    y = torch.empty_like(x)
    ctx.apply_A(x, y); outs.append(y.cpu().numpy().copy())
    ctx.apply_P(x, y); outs.append(y.cpu().numpy().copy())
    b = torch.from_numpy(prob.rhs).cuda(); z = torch.empty_like(b)
    ctx.solve(b, z, solver="minres" if pc["shape"] == "PD" else "gmres", tol=1e-10, maxit=40,
              restart=0)
    outs.append(z.cpu().numpy().copy())
    ctx.close()
np.save(sys.argv[2], np.stack(outs))
"""


def test_identical_to_dense_k_loop(tmp_path):
    res = {}
    for flag in ("1", "0"):
        # same super-block size on both sides (a narrow-band factor otherwise takes one
        # panel walk, a different blocking of the same sums)
        # and the same triangular-solve kernel (without registered ranges a factor is
        # dense to the library, which would take the dataflow TRSM)
        env = dict(os.environ, WF4DVAR_BANDED=flag, WF4DVAR_TRSM_BANDED_SB="0",
                   WF4DVAR_TRSM_DF="0")
        out = tmp_path / f"b{flag}.npy"
        r = subprocess.run([sys.executable, "-c", SCRIPT, ROOT, str(out)], env=env,
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        res[flag] = np.load(out)
    assert np.array_equal(res["1"], res["0"])
