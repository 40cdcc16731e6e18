"""Two-stream stress test of the library GEMM: the same products launched alone and
concurrently with another stream's GEMM / vector work must agree bitwise."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2105_06975_b200 import _lib as L
g = torch.Generator().manual_seed(1)
shapes = [(2048, 8192, 2048), (2048, 8192, 512), (1024, 8192, 1024), (512, 8192, 512)]
mats = []
for (M, N, K) in shapes:
    A = torch.randn(M, K, generator=g, dtype=torch.float64).cuda()
    X = torch.randn(K, N, generator=g, dtype=torch.float64).cuda()
    mats.append((A, X))
ref = []
for A, X in mats:
    Y = torch.empty(A.shape[0], X.shape[1], dtype=torch.float64, device="cuda")
    L.test_gemm(A, X, Y)
    ref.append(Y)
torch.cuda.synchronize()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
bad = 0
for rep in range(20):
    outs = []
    for i, (A, X) in enumerate(mats):
        s = s1 if i % 2 == 0 else s2
        Y = torch.empty(A.shape[0], X.shape[1], dtype=torch.float64, device="cuda")
        with torch.cuda.stream(s):
            L.test_gemm(A, X, Y, stream=s.cuda_stream)
        outs.append(Y)
    torch.cuda.synchronize()
    for i, Y in enumerate(outs):
        if not torch.equal(Y, ref[i]):
            bad += 1
            print("rep", rep, "shape", shapes[i], "max diff", (Y - ref[i]).abs().max().item(), flush=True)
print(os.environ.get("TAGENV", ""), "concurrent GEMM mismatches:", bad, "of", 20 * len(mats), flush=True)
