#!/usr/bin/env python
"""Diagnose the GPU-vs-oracle MINRES iteration count on the smoke cell (BJ.c0, P_D,
L_M(3), R_ME, tol 1e-10): both residual histories side by side, where they first
differ by more than 1e-3 relative, and the oracle run with every apply replaced by
the GPU's own apply output (isolating the Krylov recurrence from the operator
rounding).  Prints JSON."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_2105_06975_b200 as W
    from oracle import krylov as KR
    from oracle.saddle import Precond, Saddle
    from synth import configs as SC
    from synth.layout import from_paper_order, to_paper_order
    prob = SC.make_problem(0)
    s, p, Wn = prob.s, prob.p, prob.W
    cells = [dict(shape="PD", lhat="LM", k=3, rhat="me"), dict(shape="PD", lhat="LM", k=5, rhat="exact"),
             dict(shape="PD", lhat="LM", k=2, rhat="rr")]
    out = []
    for pc in cells:
        ctx = W.Context.from_problem(prob, pc)
        b = torch.from_numpy(prob.rhs).cuda()
        x = torch.empty_like(b)
        rep = ctx.solve(b, x, solver="minres", tol=1e-10, maxit=3000, history=True)
        hg = rep["history"][:, 0]
        hg = hg[~np.isnan(hg)]
        sad = Saddle(prob)
        opc = Precond(pc["shape"], pc["lhat"], pc["k"], pc["rhat"])
        bp = to_paper_order(prob.rhs, s, p, Wn, 1)[0]
        xo, info = KR.minres(sad.apply_A, lambda v: sad.apply_Pinv(opc, v), bp, tol=1e-10,
                             maxit=3000)
        ho = np.array(info["history"])

        # GPU operators inside the oracle's recurrence
        def gA(v):
            vd = torch.from_numpy(from_paper_order(v[None], s, p, Wn)).cuda()
            y = torch.empty_like(vd)
            ctx.apply_A(vd, y)
            return to_paper_order(y.cpu().numpy(), s, p, Wn, 1)[0]

        def gP(v):
            vd = torch.from_numpy(from_paper_order(v[None], s, p, Wn)).cuda()
            y = torch.empty_like(vd)
            ctx.apply_P(vd, y)
            return to_paper_order(y.cpu().numpy(), s, p, Wn, 1)[0]
        _, info_g = KR.minres(gA, gP, bp, tol=1e-10, maxit=3000)
        hog = np.array(info_g["history"])
        # oracle recurrence with the explicit residual every iteration (true residual)
        n = min(len(hg), len(ho))
        rd = np.abs(hg[:n] - ho[:n]) / ho[:n]
        first = int(np.argmax(rd > 1e-3)) if np.any(rd > 1e-3) else None
        rec = dict(cell=pc, it_gpu=int(rep["iters"][0]), it_oracle=info["iters"],
                   it_oracle_with_gpu_ops=info_g["iters"], first_1e3_divergence=first,
                   tail_gpu=[float(v) for v in hg[-12:]], tail_oracle=[float(v) for v in ho[-12:]],
                   tail_oracle_gpu_ops=[float(v) for v in hog[-12:]],
                   reldiff_every10=[float(v) for v in rd[::10]])
        print(json.dumps(rec), flush=True)
        out.append(rec)
        ctx.close()


if __name__ == "__main__":
    main()
