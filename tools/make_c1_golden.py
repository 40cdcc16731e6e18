#!/usr/bin/env python
"""Writes tests/golden/c1_gmres_oracle.json: the ORACLE's (oracle/ only) right-
preconditioned GMRES(50) (CGS2) on BASELINE.json configs[1], RHS
column 0, for every cell of tools/grid.py's c1 grid: the residual history of the
first --hist iterations, the iteration at which relres <= 1e-8, and -- for the cells
listed in --solve -- the solution to 1e-10 (256 sampled entries at fixed indices and
its 2-norm).  Run on the CPU; the GPU test tests/test_gpu_c1.py compares against it.
usage: python tools/make_c1_golden.py [--part i/n] (parts are merged by --merge)."""
import argparse
import glob
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "tests", "golden", "c1_gmres_oracle.json")   # --config 4: c4_...
SOLVE = {(s, l, k, r) for s in ("PD", "PI") for (l, k, r) in
         (("LM", 4, "exact"), ("L", 1, "exact"), ("L0", 1, "diag"), ("LM", 2, "me"),
          ("LI", 1, "rr"), ("LM", 3, "block"))}
NSAMP = 256


def cells(config=1):
    import itertools
    if config == 4:   # BJ.c4: P_I + GMRES(50), L_M(4), every R_hat
        return [("PI", "LM", 4, r) for r in ("diag", "block", "rr", "me", "exact")]
    LHS = [("L0", 1), ("LI", 1), ("LM", 2), ("LM", 3), ("LM", 4), ("L", 1)]
    return [(s, l, k, r) for s, (l, k), r in itertools.product(
        ("PD", "PI"), LHS, ("diag", "block", "rr", "me", "exact"))]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--part", default="0/1")
    ap.add_argument("--hist", type=int, default=200)
    ap.add_argument("--maxit", type=int, default=3000)
    ap.add_argument("--merge", action="store_true")
    ap.add_argument("--sens", action="store_true",
                    help="rounding sensitivity instead: the oracle's own history under 1e-15 "
                         "relative noise on every P^{-1} output (3 seeds, first --sens-its "
                         "iterations), max over seeds of |h_noisy / h - 1| per iteration")
    ap.add_argument("--sens-its", type=int, default=100)
    ap.add_argument("--noise", default="output", choices=["output", "input"],
                    help="--sens: where the 1e-15 relative noise enters P^{-1}.  'input' is the "
                         "backward-error model of a backward-stable solve, (C + E)^{-1} x = "
                         "C^{-1} (x - E y): its output moves by up to kappa(C) 1e-15 -- the size of "
                         "the differences two correct implementations' triangular solves have "
                         "(reading A34); 'output' (the round-1 model) moves it by 1e-15 only")
    ap.add_argument("--seeds", type=int, default=3)
    ap.add_argument("--config", type=int, default=1, choices=[1, 4])
    a = ap.parse_args()
    global OUT
    if a.config == 4:
        OUT = OUT.replace("c1_gmres", "c4_gmres")
    blk = 50 if a.config == 1 else 256
    if a.merge:
        res = []
        for f in sorted(glob.glob(OUT + ".part*")):
            res += json.load(open(f))
        sens, sens_in = {}, {}
        for f in sorted(glob.glob(OUT + ".sens[0-9]*")):
            sens.update({d["index"]: d["sens"] for d in json.load(open(f))})
        for f in sorted(glob.glob(OUT + ".sensin[0-9]*")):
            sens_in.update({d["index"]: d["sens"] for d in json.load(open(f))})
        for d in res:
            d["sens"] = sens.get(d["index"])
            if d["index"] in sens_in:
                d["sens_in"] = sens_in[d["index"]]
        res.sort(key=lambda d: d["index"])
        json.dump(dict(source="tools/make_c1_golden.py (oracle/ only): oracle.saddle blockwise A, "
                              "P_D / P_I (P:L629-667) and oracle.krylov.gmres (CGS2, restart 50)",
                       config=f"BASELINE.json configs[{a.config}], RHS column 0 (seed 0)",
                       nsamp=NSAMP,
                       cells=res), open(OUT, "w"))
        print(f"{len(res)} cells -> {OUT}")
        return
    from oracle import krylov as KR
    from oracle.saddle import Precond, Saddle
    from synth import configs as SC
    from synth.layout import to_paper_order
    i, n = (int(v) for v in a.part.split("/"))
    prob = SC.make_problem(a.config, m=1)
    bp = to_paper_order(prob.rhs, prob.s, prob.p, prob.W, 1)[0]
    idx = np.sort(np.random.Generator(np.random.PCG64(99)).choice(bp.size, NSAMP, replace=False))
    sad = Saddle(prob)
    res = []
    if a.sens:
        for j, c in enumerate(cells(a.config)):
            if j % n != i:
                continue
            pc = Precond(c[0], c[1], c[2], c[3], block=blk)
            if a.noise == "input":
                run = lambda nz: np.array(KR.gmres(sad.apply_A, lambda v: sad.apply_Pinv(pc, nz(v)),
                                                   bp, tol=1e-10, restart=50,
                                                   maxit=a.sens_its)[1]["history"])
            else:
                run = lambda nz: np.array(KR.gmres(sad.apply_A, lambda v: nz(sad.apply_Pinv(pc, v)),
                                                   bp, tol=1e-10, restart=50,
                                                   maxit=a.sens_its)[1]["history"])
            h0 = run(lambda v: v)
            worst = np.zeros(h0.size)
            for seed in range(1, a.seeds + 1):
                rng = np.random.default_rng(seed)
                h1 = run(lambda v: v * (1 + 1e-15 * rng.standard_normal(v.size)))
                k = min(h1.size, h0.size)
                worst[:k] = np.maximum(worst[:k], np.abs(h1[:k] / h0[:k] - 1))
            res.append(dict(index=j, sens=[float(v) for v in worst]))
            print(j, c, "sens max %.1e" % worst.max(), flush=True)
            json.dump(res, open(OUT + (f".sens{i}" if a.noise == "output" else f".sensin{i}"), "w"))
        return
    for j, c in enumerate(cells(a.config)):
        if j % n != i:
            continue
        t0 = time.time()
        pc = Precond(c[0], c[1], c[2], c[3], block=blk)
        solve = c in SOLVE and a.config == 1
        x, info = KR.gmres(sad.apply_A, lambda v: sad.apply_Pinv(pc, v), bp, tol=1e-10,
                           restart=50, maxit=a.maxit if solve else a.hist)
        h = np.array(info["history"])
        rec = dict(index=j, cell=dict(shape=c[0], lhat=c[1], k=c[2], rhat=c[3], block=blk),
                   history=[float(v) for v in h[:a.hist + 1]],
                   iters=int(info["iters"]), converged=bool(info["converged"]),
                   it_1e8=int(np.argmax(h <= 1e-8)) if np.any(h <= 1e-8) else None,
                   seconds=time.time() - t0)
        if solve and info["converged"]:
            rec.update(x_idx=[int(v) for v in idx], x_samp=[float(v) for v in x[idx]],
                       x_norm=float(np.linalg.norm(x)), true_relres=float(info["relres"]))
        res.append(rec)
        print(json.dumps({k: v for k, v in rec.items() if k not in ("history", "x_idx", "x_samp")}),
              flush=True)
        json.dump(res, open(OUT + f".part{i}", "w"))


if __name__ == "__main__":
    main()
