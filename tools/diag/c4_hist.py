"""configs[4] GMRES(50) history: GPU batched vs oracle recurrence with the GPU's column
applies vs the pure oracle (golden), plus per-block apply differences GPU vs oracle."""
import json, os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2105_06975_b200 as W
from oracle import krylov as KR
from oracle.saddle import Precond, Saddle
from synth import configs as SC
from synth.layout import to_paper_order
from tests.helpers import gpu_column_ops
rh = sys.argv[1] if len(sys.argv) > 1 else "me"
gold = json.load(open(os.path.join(ROOT, "tests/golden/c4_gmres_oracle.json")))
rec = [c for c in gold["cells"] if c["cell"]["rhat"] == rh][0]
prob = SC.make_problem(4)
pc = rec["cell"]
ctx = W.Context.from_problem(prob, pc)
b = torch.from_numpy(prob.rhs).cuda(); x = torch.empty_like(b)
r = ctx.solve(b, x, solver="gmres", tol=1e-10, maxit=100, restart=50, history=True)
hg = r["history"][:, 0]
bp = to_paper_order(prob.rhs, prob.s, prob.p, prob.W, prob.m)[0]
gA, gP = gpu_column_ops(ctx, prob, 0)
_, info = KR.gmres(gA, gP, bp, tol=1e-10, restart=50, maxit=100)
hr = np.array(info["history"])
ho = np.array(rec["history"])[:101]
n = min(hr.size, 101)
print("it  gpu            rec(oracle+gpu ops)  oracle")
for i in list(range(0, 12)) + list(range(45, 56)) + list(range(95, n)):
    print(i, "%.12f %.12f %.12f" % (hg[i], hr[i], ho[i]))
print("max |hg/hr-1| %.2e  max |hg/ho-1| %.2e  max |hr/ho-1| %.2e" % (
    np.max(np.abs(hg[1:n] / hr[1:n] - 1)), np.max(np.abs(hg[1:n] / ho[1:n] - 1)), np.max(np.abs(hr[1:n] / ho[1:n] - 1))))
sad = Saddle(prob)
opc = Precond(pc["shape"], pc["lhat"], pc["k"], pc["rhat"], block=pc.get("block", 256))
s_, p_, W_ = prob.s, prob.p, prob.W
for name, v in (("b", bp), ("A P^-1 b", gA(gP(bp)))):
    yo = sad.apply_Pinv(opc, v); yg = gP(v)
    segs = [(0, s_ * W_), (s_ * W_, (s_ + p_) * W_), ((s_ + p_) * W_, (2 * s_ + p_) * W_)]
    print(name, "P^-1 rel diff per block", ["%.2e" % (np.linalg.norm(yg[a:b] - yo[a:b]) / max(np.linalg.norm(yo[a:b]), 1e-300)) for a, b in segs])
    ao = sad.apply_A(v); ag = gA(v)
    print(name, "A rel diff %.2e" % (np.linalg.norm(ag - ao) / np.linalg.norm(ao)))
