"""Is every apply column-independent?  Column 0 of P^{-1} X and A X must not depend on
the other RHS columns (configs[4] cell P_I, L_M(4), R_ME)."""
import sys, os
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2105_06975_b200 as W
from synth import configs as SC
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
rhat = sys.argv[2] if len(sys.argv) > 2 else "me"
prob = SC.make_problem(cfg)
pc = dict(shape="PI", lhat="LM", k=4, rhat=rhat)
ctx = W.Context.from_problem(prob, pc)
g = torch.Generator().manual_seed(3)
X = torch.randn(prob.n, generator=g, dtype=torch.float64).cuda()
m = prob.m
X0 = X.clone().view(-1, m); X0[:, 1:] = 0; X0 = X0.view(-1)
for name, fn in (("A", ctx.apply_A), ("P", ctx.apply_P)):
    Y = torch.empty_like(X); Y0 = torch.empty_like(X); Y1 = torch.empty_like(X)
    fn(X, Y); fn(X0, Y0); fn(X, Y1)
    torch.cuda.synchronize()
    a = Y.view(-1, m)[:, 0]; b = Y0.view(-1, m)[:, 0]
    d = ((a - b).abs().max() / a.abs().max()).item()
    rep = torch.equal(Y, Y1)
    # per segment
    s, p, Wn = prob.s, prob.p, prob.W
    segs = [(0, s * Wn), (s * Wn, (s + p) * Wn), ((s + p) * Wn, (2 * s + p) * Wn)]
    ds = []
    for lo, hi in segs:
        aa, bb = a[lo:hi], b[lo:hi]
        ds.append(((aa - bb).abs().max() / aa.abs().max().clamp_min(1e-300)).item())
    print(f"cfg {cfg} {rhat} {name}: column 0 with / without the other columns: max rel diff {d:.3e} per segment {['%.2e' % v for v in ds]}; repeat bitwise {rep}", flush=True)
