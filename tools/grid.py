#!/usr/bin/env python
"""Cell grids of SURVEY 8(d) on one GPU: for every preconditioner cell of a config,
the A+P step rate (K batched Krylov iterations, CUDA events, solver initialisation
taken out) and a real solve to --tol with the residual history (time to 1e-8 =
first iteration at which every RHS is <= 1e-8; BASELINE.json metric).  One JSON line
per cell; --out collects them with the column-0 histories (for comparison with the
oracle's, tools/oracle_hist.py).

Grids (SURVEY 8(d) "Cells to run"):
  c1   GMRES(50) x {P_D, P_I} x {L_0, L_I, L_M(2), L_M(3), L_M(4), L} x
       {R_diag, R_block(50), R_RR, R_ME, R}                      (BJ.c1)
  c3   P_D + MINRES, L_M(k) k in {4, 3, 1, 128 = N+1 (exact L)} x {R, R_diag}
  c2   {P_D + MINRES, P_I + GMRES(50)} x k in {1, 3, 4} x {R_diag, R, R_RR, R_ME}
  c4   P_I + GMRES(50), L_M(4) x {R_diag, R_block(256), R_RR, R_ME, R}
"""
import argparse
import itertools
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

LH = [("L0", 1), ("LI", 1), ("LM", 2), ("LM", 3), ("LM", 4), ("L", 1)]


def grid(name):
    if name == "c1":
        return 1, [dict(shape=s, lhat=l, k=k, rhat=r, block=50, solver="gmres")
                   for s, (l, k), r in itertools.product(("PD", "PI"), LH,
                                                         ("diag", "block", "rr", "me", "exact"))]
    if name == "c3":
        return 3, [dict(shape="PD", lhat="LM", k=k, rhat=r, solver="minres")
                   for r, k in itertools.product(("exact", "diag"), (4, 3, 1, 128))]
    if name == "c2":
        return 2, [dict(shape=s, lhat="LM", k=k, rhat=r, solver=sv)
                   for (s, sv), k, r in itertools.product((("PD", "minres"), ("PI", "gmres")),
                                                         (1, 3, 4), ("diag", "exact", "rr", "me"))]
    if name == "c4":
        return 4, [dict(shape="PI", lhat="LM", k=4, rhat=r, block=256, solver="gmres")
                   for r in ("diag", "block", "rr", "me", "exact")]
    raise SystemExit(f"unknown grid {name}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("grid")
    ap.add_argument("--steps", type=int, default=None, help="timed iterations (default 20; "
                    "GMRES: 50 = one restart cycle)")
    ap.add_argument("--tol", type=float, default=1e-8)
    ap.add_argument("--maxit", type=int, default=2000)
    ap.add_argument("--only", default=None, help="comma list of cell indices")
    ap.add_argument("--apply-mode", default="trsm")
    ap.add_argument("--out", default=None)
    ap.add_argument("--every", type=int, default=1, help="history stride stored in --out")
    a = ap.parse_args()
    import torch
    import paper_2105_06975_b200 as W
    from synth import configs as SC
    cfg, cells = grid(a.grid)
    prob = SC.make_problem(cfg)
    b = torch.from_numpy(prob.rhs).cuda()
    x = torch.empty_like(b)
    res = []
    idx = range(len(cells)) if not a.only else [int(v) for v in a.only.split(",")]
    for i in idx:
        cell = dict(cells[i])
        solver = cell.pop("solver")
        steps = a.steps or (50 if solver == "gmres" else 20)
        t0 = time.time()
        ctx = W.Context.from_problem(prob, dict(cell, apply_mode=a.apply_mode))
        setup_s = time.time() - t0
        kw = dict(solver=solver, restart=50, check_every=10 ** 6)
        ctx.solve(b, x, tol=1e-300, maxit=3, **kw)
        r = ctx.solve(b, x, tol=1e-300, maxit=steps, **kw)
        ms = (r["seconds"] - r["seconds_init"]) / steps * 1e3
        kw["check_every"] = 10
        r = ctx.solve(b, x, tol=a.tol, maxit=a.maxit, mark_tol=1e-8, history=True, **kw)
        h = r["history"]
        its = np.asarray(r["iters"])
        line = dict(grid=a.grid, config=cfg, index=i, cell=cell, solver=solver, restart=50,
                    m=prob.m, setup_s=round(setup_s, 3), ms_per_step=ms,
                    applies_per_s=1e3 / ms, tol=a.tol, maxit=a.maxit,
                    reached_1e8=bool(r["seconds_to_mark"] >= 0),
                    seconds_to_1e8=r["seconds_to_mark"] if r["seconds_to_mark"] >= 0 else None,
                    iters_to_1e8=int(r["iters_to_mark"]),
                    iters_median=float(np.median(its)), iters_max=int(its.max()),
                    relres_max=float(np.max(r["relres"])), solve_seconds=r["seconds"],
                    apply_mode=a.apply_mode)
        print(json.dumps(line), flush=True)
        line["hist_col0"] = [float(v) for v in h[::a.every, 0] if not np.isnan(v)]
        res.append(line)
        ctx.close()
    if a.out:
        json.dump(res, open(a.out, "w"))


if __name__ == "__main__":
    main()
