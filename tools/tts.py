#!/usr/bin/env python
"""Time-to-solution runs (BASELINE.json metric "time-to-1e-8 residual"): one warm-up
solve, then one solve to --tol with the residual history recorded, for each
--apply-mode given (the default triangular solves vs the opt-in explicit inverses,
DESIGN.md reading A32).  Prints one JSON line per mode."""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--shape", default="PD")
    ap.add_argument("--lhat", default="LM")
    ap.add_argument("--k", type=int, default=4)
    ap.add_argument("--rhat", default="exact")
    ap.add_argument("--block", type=int, default=0)
    ap.add_argument("--solver", default=None)
    ap.add_argument("--restart", type=int, default=50)
    ap.add_argument("--tol", type=float, default=1e-8)
    ap.add_argument("--maxit", type=int, default=5000)
    ap.add_argument("--m", type=int, default=None)
    ap.add_argument("--modes", default="trsm,inverse")
    ap.add_argument("--every", type=int, default=10, help="history subsample stride")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    import torch
    import paper_2105_06975_b200 as W
    from synth import configs as SC
    prob = SC.make_problem(a.config, m=a.m)
    solver = a.solver or ("minres" if a.shape == "PD" else "gmres")
    b = torch.from_numpy(prob.rhs).cuda()
    x = torch.empty_like(b)
    lines = []
    for mode in a.modes.split(","):
        pc = dict(shape=a.shape, lhat=a.lhat, k=a.k, rhat=a.rhat, block=a.block, apply_mode=mode)
        ctx = W.Context.from_problem(prob, pc)
        ctx.solve(b, x, solver=solver, tol=1e-300, maxit=3, restart=a.restart, check_every=10 ** 6)
        torch.cuda.synchronize()
        r = ctx.solve(b, x, solver=solver, tol=a.tol, maxit=a.maxit, restart=a.restart,
                      mark_tol=a.tol, check_every=10, history=True)
        h = r["history"]
        its = np.arange(0, h.shape[0], a.every)
        hmax = np.nanmax(h[its], axis=1)
        hmed = np.nanmedian(h[its], axis=1)
        line = dict(config=a.config, cell=pc, solver=solver, restart=a.restart, tol=a.tol,
                    maxit=a.maxit, m=prob.m, seconds=r["seconds"],
                    seconds_to_tol=r["seconds_to_mark"] if r["seconds_to_mark"] >= 0 else None,
                    iters_to_tol=int(r["iters_to_mark"]),
                    iters=[int(v) for v in r["iters"]], relres=[float(v) for v in r["relres"]],
                    ms_per_iter=r["seconds"] / max(1, int(np.max(r["iters"]))) * 1e3,
                    hist_every=a.every, hist_max=[float(v) for v in hmax],
                    hist_median=[float(v) for v in hmed])
        print(json.dumps({k: v for k, v in line.items() if not k.startswith("hist")}), flush=True)
        lines.append(line)
        ctx.close()
    if a.out:
        json.dump(lines, open(a.out, "w"))


if __name__ == "__main__":
    main()
