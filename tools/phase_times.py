"""Per-phase timing of the hot path at a BASELINE config (CUDA events, warm):
apply_A, apply_P, apply_AP and one solver iteration, plus the algorithmic FLOPs,
to locate the gap to the roofline."""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2105_06975_b200 as W  # noqa: E402
from synth import configs as SC  # noqa: E402


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--shape", default="PD")
    ap.add_argument("--k", type=int, default=4)
    ap.add_argument("--rhat", default="exact")
    a = ap.parse_args()
    prob = SC.make_problem(a.config)
    pc = dict(shape=a.shape, lhat="LM", k=a.k, rhat=a.rhat)
    ctx = W.Context.from_problem(prob, pc)
    x = torch.randn(prob.n, dtype=torch.float64, device="cuda")
    t = torch.empty_like(x)
    y = torch.empty_like(x)
    s, p, Wn, m = prob.s, prob.p, prob.W, prob.m
    res = dict(config=a.config, cell=pc)
    res["apply_A_ms"] = timeit(lambda: ctx.apply_A(x, y))
    res["apply_P_ms"] = timeit(lambda: ctx.apply_P(x, y))
    res["apply_AP_ms"] = timeit(lambda: ctx.apply_AP(x, t, y))
    b = torch.from_numpy(prob.rhs).cuda()
    solver = "minres" if a.shape == "PD" else "gmres"
    res["solve10_ms"] = timeit(lambda: ctx.solve(b, y, solver=solver, tol=1e-300, maxit=10,
                                                 check_every=1000), reps=3)
    fA = 2 * Wn * m * (s * s + p * p)
    fP = 2 * Wn * m * ((2 * s * s if a.shape == "PD" else 0) + s * s +
                       (p * p if a.rhat != "diag" else 0))
    res["gflop_A"] = fA / 1e9
    res["gflop_P"] = fP / 1e9
    res["tflops_A"] = fA / res["apply_A_ms"] / 1e9
    res["tflops_P"] = fP / res["apply_P_ms"] / 1e9
    res["tflops_AP"] = (fA + fP) / res["apply_AP_ms"] / 1e9
    ctx.profile_enable(True)
    ctx.apply_A(x, y)
    prA = ctx.profile_read()
    ctx.profile_enable(True)
    ctx.apply_P(x, y)
    prP = ctx.profile_read()
    ctx.profile_enable(False)
    res["A_classes_ms"] = {k: round(v["ms"], 3) for k, v in prA.items() if v["launches"]}
    res["P_classes_ms"] = {k: round(v["ms"], 3) for k, v in prP.items() if v["launches"]}
    res["A_launches"] = {k: v["launches"] for k, v in prA.items() if v["launches"]}
    res["P_launches"] = {k: v["launches"] for k, v in prP.items() if v["launches"]}
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
