import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_2105_06975_b200 as W
from paper_2105_06975_b200 import _lib as L
from synth import configs as SC
# small-operator kernels (L96-like sizes), inverse-form TRSM, stream-K tail, banded
g = torch.Generator().manual_seed(1)
for n, nc, blk, up in ((40, 700, 0, False), (200, 130, 7, True), (600, 300, 0, False), (300, 90, 64, True)):
    M = torch.randn(n, n, generator=g, dtype=torch.float64); S = M @ M.T / n + torch.eye(n, dtype=torch.float64)
    if blk:
        mask = torch.zeros(n, n, dtype=torch.bool)
        for a in range(0, n, blk): mask[a:a+blk, a:a+blk] = True
        S = torch.where(mask, S, torch.zeros_like(S))
    F = torch.linalg.cholesky(S); F = (F.T if up else F).contiguous().cuda()
    X = torch.randn(n, nc, generator=g, dtype=torch.float64).cuda(); Y = torch.empty_like(X)
    L.test_trsm(F, X, Y, upper=up, blk=blk)
for (m_, n_, k_) in ((40, 500, 40), (63, 333, 17), (1024, 2432, 256)):
    A = torch.randn(m_, k_, dtype=torch.float64).cuda(); X = torch.randn(k_, n_, dtype=torch.float64).cuda()
    Y = torch.empty(m_, n_, dtype=torch.float64).cuda(); L.test_gemm(A, X, Y)
prob = SC.paper_heat_problem(s=1024, N=2, m=1, nsteps=1)
for pc in (dict(shape="PD", lhat="LM", k=2, rhat="exact"), dict(shape="PD", lhat="LM", k=2, rhat="exact", factor="ichol", ridge=0.01)):
    ctx = W.Context.from_problem(prob, pc)
    x = torch.from_numpy(np.random.default_rng(0).standard_normal(prob.n)).cuda(); y = torch.empty_like(x)
    ctx.apply_A(x, y); ctx.apply_P(x, y)
    yh = np.empty(prob.n); ctx.apply_AP_host(x.cpu().numpy(), yh)
    ctx.close()
prob = SC.make_problem(2)
prob2 = SC.custom_problem(s=40, N=3, q=2, m=64, model="l96", seed0=1) if False else None
torch.cuda.synchronize()
print("ok")
