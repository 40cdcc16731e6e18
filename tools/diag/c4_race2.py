"""Operator-only reproducibility under the fork/join streams: v <- A P^{-1} v (scaled)
60 times on configs[4] (P_I, L_M(4), R_hat = R); prints a checksum and whether two runs
in the same process agree bitwise."""
import os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2105_06975_b200 as W
from synth import configs as SC
CFG = int(os.environ.get("CFG", "4"))
prob = SC.make_problem(CFG)
cell = dict(shape="PI", lhat="LM", k=4, rhat="exact", block=256) if CFG == 4 else \
    dict(shape="PD", lhat="LM", k=4, rhat="exact")
ctx = W.Context.from_problem(prob, cell)
g = torch.Generator().manual_seed(5)
x0 = torch.randn(prob.n, generator=g, dtype=torch.float64).cuda()
outs = []
NREP = int(os.environ.get('NREP', '2'))
for rep in range(NREP):
    v = x0.clone(); u = torch.empty_like(v); w = torch.empty_like(v)
    for it in range(60):
        mode = os.environ.get("MODE", "PA")
        if mode == "PA":
            ctx.apply_P(v, u); ctx.apply_A(u, w)
        elif mode == "A":
            ctx.apply_A(v, w)
        else:
            ctx.apply_P(v, w)
        v = w / w.norm()
    torch.cuda.synchronize()
    outs.append(v.cpu().numpy())
d = max(np.max(np.abs(outs[0] - o)) for o in outs[1:])
print(os.environ.get("TAGENV", ""), "cfg", CFG, os.environ.get("MODE", "PA"), "repeats bitwise equal:", [bool(np.array_equal(outs[0], o)) for o in outs[1:]], "max diff %.2e" % d,
      "checksum %.17e" % float(np.sum(outs[0] * np.arange(outs[0].size) % 7)), flush=True)
