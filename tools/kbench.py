"""Micro-benchmark of the DMMA GEMM and TRSM kernels at the configs[3] shapes,
against cuBLAS (torch.matmul / torch.linalg.solve_triangular) on the same box."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2105_06975_b200 import _lib as L  # noqa: E402


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / 1e3)
    return best


def main():
    out = {}
    gemm_shapes = [] if "--trsm-only" in sys.argv else [
        (4096, 8128, 4096), (4096, 8256, 4096), (4096, 8192, 4096), (3072, 8256, 1024),
        (2048, 8256, 1024), (1024, 8192, 1024), (3584, 8192, 512), (1000, 320, 1000)]
    for (M, N, K) in gemm_shapes:
        A = torch.randn(M, K, dtype=torch.float64, device="cuda")
        X = torch.randn(K, N, dtype=torch.float64, device="cuda")
        Y = torch.empty(M, N, dtype=torch.float64, device="cuda")
        t = timeit(lambda: L.test_gemm(A, X, Y))
        tc = timeit(lambda: torch.matmul(A, X, out=Y))
        f = 2.0 * M * N * K
        out[f"gemm_{M}x{N}x{K}"] = dict(ours_tflops=f / t / 1e12, cublas_tflops=f / tc / 1e12,
                                        ours_ms=t * 1e3)
    for (n, ncols) in ([] if "--gemm-only" in sys.argv else [(4096, 8128), (1024, 8192), (1000, 336), (500, 336)]):
        S = torch.randn(n, n, dtype=torch.float64, device="cuda")
        S = S @ S.T / n + torch.eye(n, dtype=torch.float64, device="cuda")
        G = torch.linalg.cholesky(S).contiguous()
        X = torch.randn(n, ncols, dtype=torch.float64, device="cuda")
        Y = torch.empty_like(X)
        t = timeit(lambda: L.test_trsm(G, X, Y, upper=False))
        tc = timeit(lambda: torch.linalg.solve_triangular(G, X, upper=False))
        f = 1.0 * n * n * ncols
        out[f"trsm_{n}x{ncols}"] = dict(ours_tflops=f / t / 1e12, cublas_tflops=f / tc / 1e12,
                                        ours_ms=t * 1e3, cublas_ms=tc * 1e3)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
