"""Experiment: does splitting a GMRES batch over two contexts that run concurrently (two
host threads, own streams) overlap one half's tensor-bound operator applies with the
other half's HBM-bound CGS2?  configs[4] (P_I, L_M(4), R, GMRES(50)), 50 iterations."""
import os, sys, threading, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2105_06975_b200 as W
from synth import configs as SC

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
its = int(sys.argv[2]) if len(sys.argv) > 2 else 50
pc = dict(shape="PI", lhat="LM", k=4, rhat="exact") if cfg == 4 else dict(shape="PD", lhat="LM", k=4, rhat="exact")
solver = "gmres" if cfg == 4 else "minres"
full = SC.make_problem(cfg)
m = full.m
half = SC.make_problem(cfg, m=m // 2)

def mk(prob):
    s = torch.cuda.Stream()
    ctx = W.Context.from_problem(prob, pc, stream=s.cuda_stream)
    b = torch.from_numpy(prob.rhs).cuda()
    x = torch.empty_like(b)
    return ctx, b, x, s

def run(c, n=its):
    ctx, b, x, s = c
    with torch.cuda.stream(s):
        ctx.solve(b, x, solver=solver, tol=1e-300, maxit=n, restart=50, check_every=10)

F = mk(full)
run(F, 3); torch.cuda.synchronize()
t = time.perf_counter(); run(F); torch.cuda.synchronize(); tf = time.perf_counter() - t
print(f"full m={m}: {tf / its * 1e3:.3f} ms/step", flush=True)
del F
torch.cuda.empty_cache()
H = [mk(half), mk(half)]
for h in H:
    run(h, 3)
torch.cuda.synchronize()
t = time.perf_counter(); run(H[0]); run(H[1]); torch.cuda.synchronize(); ts = time.perf_counter() - t
print(f"two halves in sequence: {ts / its * 1e3:.3f} ms per full-batch step", flush=True)
for delay in (0.0, 0.005):
    th = [threading.Thread(target=run, args=(h,)) for h in H]
    torch.cuda.synchronize()
    t = time.perf_counter()
    th[0].start(); time.sleep(delay); th[1].start()
    for x in th: x.join()
    torch.cuda.synchronize(); tc = time.perf_counter() - t
    print(f"two halves concurrently (start offset {delay * 1e3:.0f} ms): {tc / its * 1e3:.3f} ms per full-batch step", flush=True)
