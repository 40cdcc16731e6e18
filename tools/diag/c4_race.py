"""configs[4] R_hat = R: is the GPU GMRES(50) history reproducible, and does it match the
oracle recurrence driven by the GPU's own column applies?  Run under different env
settings (WF4DVAR_FORK=0 serialises the operator blocks)."""
import json, os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2105_06975_b200 as W
from oracle import krylov as KR
from synth import configs as SC
from synth.layout import to_paper_order
from tests.helpers import gpu_column_ops
rh = sys.argv[1] if len(sys.argv) > 1 else "exact"
prob = SC.make_problem(4)
pc = dict(shape="PI", lhat="LM", k=4, rhat=rh, block=256)
ctx = W.Context.from_problem(prob, pc)
b = torch.from_numpy(prob.rhs).cuda()
hs = []
for rep in range(2):
    x = torch.empty_like(b)
    r = ctx.solve(b, x, solver="gmres", tol=1e-10, maxit=60, restart=50, history=True)
    hs.append(r["history"][:61, 0].copy())
bp = to_paper_order(prob.rhs, prob.s, prob.p, prob.W, prob.m)[0]
gA, gP = gpu_column_ops(ctx, prob, 0)
_, info = KR.gmres(gA, gP, bp, tol=1e-10, restart=50, maxit=60)
hr = np.array(info["history"])[:61]
print(os.environ.get("TAGENV", ""), rh, "repeat bitwise", np.array_equal(hs[0], hs[1]),
      "max|h0/h1-1| %.2e" % np.max(np.abs(hs[0][1:] / hs[1][1:] - 1)),
      "max|hg/hrec-1| %.2e" % np.max(np.abs(hs[0][1:] / hr[1:] - 1)),
      "it50 gpu %.12f rec %.12f it51 gpu %.12f rec %.12f" % (hs[0][50], hr[50], hs[0][51], hr[51]), flush=True)
