#!/usr/bin/env python
"""configs[0], P_I + full (unrestarted) GMRES: GPU vs oracle residual histories (and the
oracle recurrence with the GPU's applies) side by side, to locate where they part."""
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
    from synth.layout import to_paper_order
    from tests.helpers import gpu_column_ops
    prob = SC.make_problem(0)
    for k, rhat in ((5, "exact"), (3, "me"), (2, "diag")):
        pc = dict(shape="PI", lhat="LM", k=k, rhat=rhat)
        ctx = W.Context.from_problem(prob, pc)
        b = torch.from_numpy(prob.rhs).cuda()
        x = torch.empty_like(b)
        for restart in (0, 50):
            r = ctx.solve(b, x, solver="gmres", tol=1e-10, maxit=3000, restart=restart, history=True)
            hg = r["history"][:, 0]
            hg = hg[~np.isnan(hg)]
            sad = Saddle(prob)
            bp = to_paper_order(prob.rhs, prob.s, prob.p, prob.W, 1)[0]
            opc = Precond("PI", "LM", k, rhat)
            _, io = KR.gmres(sad.apply_A, lambda v: sad.apply_Pinv(opc, v), bp, tol=1e-10,
                             restart=restart, maxit=3000)
            gA, gP = gpu_column_ops(ctx, prob, 0)
            _, ig = KR.gmres(gA, gP, bp, tol=1e-10, restart=restart, maxit=3000)
            ho, hr = np.array(io["history"]), np.array(ig["history"])
            n = min(len(hg), len(ho), len(hr))
            print(json.dumps(dict(k=k, rhat=rhat, restart=restart, it_gpu=int(r["iters"][0]),
                                  it_oracle=io["iters"], it_rec=ig["iters"],
                                  rel_gpu_vs_rec=[float(v) for v in np.abs(hg[1:n] / hr[1:n] - 1)[::5]],
                                  tail_gpu=[float(v) for v in hg[-6:]], tail_oracle=[float(v) for v in ho[-6:]],
                                  tail_rec=[float(v) for v in hr[-6:]])), flush=True)
        ctx.close()


if __name__ == "__main__":
    main()
