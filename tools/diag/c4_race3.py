"""Locate the irreproducible elements of one P_I apply on configs[4] with TMA-staged TRSM
coupling GEMMs (WF4DVAR_GEMM_TMA=3): repeat the apply, report which segment / rows /
columns differ from the first result."""
import os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2105_06975_b200 as W
from synth import configs as SC
prob = SC.make_problem(4)
ctx = W.Context.from_problem(prob, dict(shape="PI", lhat="LM", k=4, rhat="exact", block=256))
g = torch.Generator().manual_seed(5)
x = torch.randn(prob.n, generator=g, dtype=torch.float64).cuda()
s, p, Wn, m = prob.s, prob.p, prob.W, prob.m
ld = Wn * m
ref = torch.empty_like(x); ctx.apply_P(x, ref); torch.cuda.synchronize()
R = ref.cpu().numpy()
for rep in range(20):
    y = torch.empty_like(x); ctx.apply_P(x, y); torch.cuda.synchronize()
    Y = y.cpu().numpy()
    d = np.nonzero(Y != R)[0]
    if d.size == 0:
        continue
    seg = np.where(d < s * ld, 1, np.where(d < (s + p) * ld, 2, 3))
    for sg in (1, 2, 3):
        dd = d[seg == sg]
        if dd.size == 0:
            continue
        off = {1: 0, 2: s * ld, 3: (s + p) * ld}[sg]
        rows, cols = (dd - off) // ld, (dd - off) % ld
        rel = np.max(np.abs(Y[dd] - R[dd])) / np.max(np.abs(R[off:off + (p if sg == 2 else s) * ld]))
        print(f"rep {rep}: segment {sg}: {dd.size} elements differ; rows {rows.min()}-{rows.max()} "
              f"(unique row blocks of 64: {sorted(set((rows // 64).tolist()))[:12]}); cols {cols.min()}-{cols.max()} "
              f"(col tiles of 128: {sorted(set((cols // 128).tolist()))[:12]}); max rel {rel:.2e}", flush=True)
print("done", flush=True)
