"""Kernel-level parity of the FP64 tensor-core building blocks (through the
wf4dvar_testing.h hooks) against plain float64 references: torch matmul and a
triangular solve.  Sizes span several tiles and ragged tails."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def L():
    from paper_2105_06975_b200 import _lib
    return _lib


@pytest.mark.parametrize("M,N,K", [(1, 1, 1), (37, 19, 5), (128, 128, 32), (300, 517, 129),
                                   (1000, 336, 1000), (64, 8128, 512),
                                   # streaming kernel (M, K <= 64)
                                   (40, 5000, 40), (64, 1000, 64), (63, 333, 17)])
@pytest.mark.parametrize("with_z", [False, True])
def test_gemm_vs_float64_reference(M, N, K, with_z):
    g = torch.Generator().manual_seed(M * 7 + N + K)
    A = torch.randn(M, K, generator=g, dtype=torch.float64).cuda()
    X = torch.randn(K, N, generator=g, dtype=torch.float64).cuda()
    Z = torch.randn(M, N, generator=g, dtype=torch.float64).cuda() if with_z else None
    Y = torch.empty(M, N, dtype=torch.float64, device="cuda")
    L().test_gemm(A, X, Y, alpha=-0.5, beta=2.0, Z=Z)
    ref = -0.5 * (A.cpu() @ X.cpu()) + (2.0 * Z.cpu() if with_z else 0.0)
    err = (Y.cpu() - ref).abs().max().item()
    scale = (A.cpu().abs() @ X.cpu().abs()).max().item() + 1.0
    assert err <= 1e-14 * scale * max(1, K) ** 0.5 * 4, err


@pytest.mark.parametrize("M,N,K", [(1024, 2432, 256), (1000, 2500, 200), (3072, 8192, 1024),
                                   (4096, 8192, 128), (4096, 8256, 512)])
def test_gemm_stream_k_tail_vs_float64_reference(M, N, K):
    """Tile counts that leave a nearly empty last wave (304, 320, 4160 tiles of 64x128
    on 296 resident CTAs) take the stream-K hybrid: the data-parallel waves in the
    plain kernel, the last G + r tiles split by k-iterations with parked partials and
    a deterministic fix-up (3072 / 4096 tiles: plain kernel).  Same tolerance as the
    data-parallel kernel, and bitwise-reproducible across launches."""
    g = torch.Generator().manual_seed(M + N + K)
    A = torch.randn(M, K, generator=g, dtype=torch.float64).cuda()
    X = torch.randn(K, N, generator=g, dtype=torch.float64).cuda()
    Z = torch.randn(M, N, generator=g, dtype=torch.float64).cuda()
    Y = torch.empty(M, N, dtype=torch.float64, device="cuda")
    L().test_gemm(A, X, Y, alpha=1.5, beta=-1.0, Z=Z)
    ref = 1.5 * (A @ X) - Z     # cuBLAS DGEMM as the float64 reference at this size
    scale = (A.abs() @ X.abs()).max().item() + 1.0
    assert (Y - ref).abs().max().item() <= 1e-14 * scale * K ** 0.5 * 4
    Y2 = torch.empty_like(Y)
    L().test_gemm(A, X, Y2, alpha=1.5, beta=-1.0, Z=Z)
    assert torch.equal(Y, Y2)


def test_gemm_strided_views_and_odd_ld():
    # odd leading dimensions force the 8-byte cp.async path
    A = torch.randn(51, 77, dtype=torch.float64, device="cuda")[:, :33]
    X = torch.randn(33, 45, dtype=torch.float64, device="cuda")[:, 1:44]
    Y = torch.zeros(51, 43, dtype=torch.float64, device="cuda")
    L().test_gemm(A, X, Y)
    torch.testing.assert_close(Y, A @ X, rtol=1e-13, atol=1e-13)


def test_gemm_pair_store_alignment_paths():
    """The epilogues write each accumulator pair as one 16-byte store (and read the beta term
    as one 16-byte load) only when base and leading dimension allow it: even ld with an
    8-byte-offset base, and an odd last column, must take the 8-byte path."""
    g = torch.Generator().manual_seed(11)
    A = torch.randn(130, 96, generator=g, dtype=torch.float64).cuda()
    X = torch.randn(96, 300, generator=g, dtype=torch.float64).cuda()
    Zb = torch.randn(130, 302, generator=g, dtype=torch.float64).cuda()
    Yb = torch.full((130, 302), 7.0, dtype=torch.float64, device="cuda")
    ref = 2.0 * (A @ X)
    for yo, zo, ncol in ((1, 1, 300), (0, 1, 300), (1, 0, 300), (0, 0, 299), (0, 0, 300)):
        Yb.fill_(7.0)
        Y, Z = Yb[:, yo:yo + ncol], Zb[:, zo:zo + ncol]
        L().test_gemm(A, X[:, :ncol], Y, alpha=2.0, beta=-1.0, Z=Z)
        torch.testing.assert_close(Y, ref[:, :ncol] - Z, rtol=1e-13, atol=1e-12)
        # nothing written outside the view
        assert (Yb[:, :yo] == 7.0).all() and (Yb[:, yo + ncol:] == 7.0).all()


@pytest.mark.parametrize("upper", [False, True])
def test_trsm_pair_store_misaligned_base(upper):
    """Contiguous operands whose storage starts 8 bytes off a 16-byte boundary (even ld):
    the panel / dataflow kernels must fall back to 8-byte stores."""
    n, ncols = 600, 40
    g = torch.Generator().manual_seed(3)
    M = torch.randn(n, n, generator=g, dtype=torch.float64)
    Gl = torch.linalg.cholesky(M @ M.T / n + torch.eye(n, dtype=torch.float64))
    F = (Gl.T if upper else Gl).contiguous()
    X = torch.randn(n, ncols, generator=g, dtype=torch.float64)
    ref = torch.linalg.solve_triangular(F, X, upper=upper)
    buf = torch.zeros(n * ncols + 2, dtype=torch.float64, device="cuda")
    for off in (0, 1):
        Y = buf[off:off + n * ncols].view(n, ncols)
        assert Y.is_contiguous() and (Y.data_ptr() % 16 == 8 * off)
        buf.zero_()
        L().test_trsm(F.cuda(), X.cuda(), Y, upper=upper)
        torch.cuda.synchronize()
        assert ((Y.cpu() - ref).norm() / ref.norm()).item() <= 1e-12
        assert buf[off + n * ncols:].abs().max().item() == 0.0 and buf[:off].abs().sum().item() == 0.0


@pytest.mark.parametrize("n,ncols,blk", [(5, 3, 0), (64, 64, 0), (130, 17, 0), (600, 40, 0),
                                         (1000, 336, 0), (2048, 96, 0), (500, 21, 50),
                                         (256, 64, 64),
                                         # thread-per-column kernel (segments <= 64 rows)
                                         (40, 5000, 0), (50, 333, 0), (200, 700, 7),
                                         (17, 129, 0), (300, 260, 64)])
@pytest.mark.parametrize("upper", [False, True])
def test_trsm_vs_float64_reference(n, ncols, blk, upper):
    g = torch.Generator().manual_seed(n + ncols + blk)
    M = torch.randn(n, n, generator=g, dtype=torch.float64)
    S = M @ M.T / n + torch.eye(n, dtype=torch.float64)
    if blk:
        mask = torch.zeros(n, n, dtype=torch.bool)
        for a in range(0, n, blk):
            mask[a:a + blk, a:a + blk] = True
        S = torch.where(mask, S, torch.zeros_like(S))
    Gl = torch.linalg.cholesky(S)
    F = (Gl.T if upper else Gl).contiguous()
    X = torch.randn(n, ncols, generator=g, dtype=torch.float64)
    Y = torch.empty(n, ncols, dtype=torch.float64, device="cuda")
    Fd, Xd = F.cuda(), X.cuda()
    L().test_trsm(Fd, Xd, Y, upper=upper, blk=blk)
    torch.cuda.synchronize()
    Yc = Y.cpu()
    ref = torch.linalg.solve_triangular(F, X, upper=upper)
    # backward error of the triangular solve (implementation independent)
    bwd = ((F @ Yc - X).norm() / (F.norm() * Yc.norm())).item()
    assert bwd <= 1e-15 * 4, bwd
    fwd = ((Yc - ref).norm() / ref.norm()).item()
    assert fwd <= 1e-12, fwd


@pytest.mark.parametrize("upper", [False, True])
def test_trsm_dataflow_bitwise_reproducible(upper):
    """n = 1000, 336 columns takes the dataflow TRSM (k_trsm_df): its CTAs consume their
    dependency tiles as they are published, so arrival order varies run to run; the
    summation order must not (lower: increasing-k sweeps; upper: one tile per sweep)."""
    n, ncols = 1000, 336
    g = torch.Generator().manual_seed(11)
    M = torch.randn(n, n, generator=g, dtype=torch.float64)
    S = M @ M.T / n + torch.eye(n, dtype=torch.float64)
    F = torch.linalg.cholesky(S)
    F = (F.T if upper else F).contiguous().cuda()
    X = torch.randn(n, ncols, generator=g, dtype=torch.float64).cuda()
    outs = []
    for _ in range(6):
        Y = torch.empty(n, ncols, dtype=torch.float64, device="cuda")
        L().test_trsm(F, X, Y, upper=upper)
        outs.append(Y)
    torch.cuda.synchronize()
    for Y in outs[1:]:
        assert torch.equal(Y, outs[0])


def test_trsm_in_place():
    n, ncols = 700, 50
    S = torch.randn(n, n, dtype=torch.float64)
    S = S @ S.T / n + torch.eye(n, dtype=torch.float64)
    G = torch.linalg.cholesky(S).contiguous()   # LAPACK returns Fortran strides
    X = torch.randn(n, ncols, dtype=torch.float64)
    Yd = X.clone().cuda()
    Gd = G.cuda()
    L().test_trsm(Gd, Yd, Yd, upper=False)
    torch.cuda.synchronize()
    torch.testing.assert_close(Yd.cpu(), torch.linalg.solve_triangular(G, X, upper=False),
                               rtol=1e-12, atol=1e-12)


SUBST = r"""
import sys, torch
sys.path.insert(0, sys.argv[1])
from paper_2105_06975_b200 import _lib
g = torch.Generator().manual_seed(4)
for n, ncols, upper in ((600, 40, False), (600, 40, True), (130, 17, False)):
    M = torch.randn(n, n, generator=g, dtype=torch.float64)
    S = M @ M.T / n + torch.eye(n, dtype=torch.float64)
    F = torch.linalg.cholesky(S)
    F = (F.T if upper else F).contiguous()
    X = torch.randn(n, ncols, generator=g, dtype=torch.float64)
    Y = torch.empty(n, ncols, dtype=torch.float64, device="cuda")
    _lib.test_trsm(F.cuda(), X.cuda(), Y, upper=upper)
    torch.cuda.synchronize()
    Yc = Y.cpu()
    bwd = ((F @ Yc - X).norm() / (F.norm() * Yc.norm())).item()
    assert bwd <= 4e-15, (n, upper, bwd)
print("ok")
"""


def test_trsm_substitution_form():
    """The diagonal tiles' substitution form (WF4DVAR_TRSM_INV=0, the pre-A31 path)
    stays available and backward stable."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", SUBST, root], capture_output=True, text=True,
                       env=dict(os.environ, WF4DVAR_TRSM_INV="0"), timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


def test_gemm_stream_k_concurrent_streams_and_repeats():
    """Stream-K GEMMs on two streams at once (as the fork/join blocks of A and P run
    them) keep separate parked partials and flags, and the consumer-reset flags make
    back-to-back launches (and graph replays) on one stream safe."""
    M, N, K = 1024, 2432, 256          # 304 tiles: the stream-K tail path
    g = torch.Generator().manual_seed(21)
    mats = []
    for _ in range(2):
        A = torch.randn(M, K, generator=g, dtype=torch.float64).cuda()
        X = torch.randn(K, N, generator=g, dtype=torch.float64).cuda()
        mats.append((A, X, A @ X))
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    for rep in range(6):
        outs = []
        for (A, X, _), s in zip(mats, (s1, s2)):
            Y = torch.empty(M, N, dtype=torch.float64, device="cuda")
            with torch.cuda.stream(s):
                L().test_gemm(A, X, Y, stream=s.cuda_stream)
                L().test_gemm(A, X, Y, stream=s.cuda_stream)   # same stream, back to back
            outs.append(Y)
        torch.cuda.synchronize()
        for (A, X, ref), Y in zip(mats, outs):
            scale = (A.abs() @ X.abs()).max().item()
            assert (Y - ref).abs().max().item() <= 1e-14 * scale * K ** 0.5 * 4, rep


GRAPH_SK = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_2105_06975_b200 as W
from synth import configs as SC
prob = SC.custom_problem(s=4096, N=8, q=4, m=64, seed0=5)
ctx = W.Context.from_problem(prob, dict(shape="PD", lhat="LM", k=2, rhat="exact"))
b = torch.from_numpy(prob.rhs).cuda()
outs = []
for _ in range(2):
    x = torch.empty_like(b)
    ctx.solve(b, x, solver="minres", tol=1e-300, maxit=40)
    outs.append(x.cpu().numpy())
np.save(sys.argv[2], np.stack(outs))
"""


def test_stream_k_inside_captured_graphs(tmp_path):
    """s = 4096, 576 columns: the D product (320 tiles of 64x128) takes the stream-K
    tail and the problem (n = 5.3M) runs MINRES as replayed CUDA graphs.  Replays of
    the captured stream-K launches must give exactly the eager result (the flags are
    re-armed by their consumer, not tied to a captured epoch)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for graphs in ("1", "0"):
        out = tmp_path / f"g{graphs}.npy"
        r = subprocess.run([sys.executable, "-c", GRAPH_SK, root, str(out)], capture_output=True,
                           text=True, env=dict(os.environ, WF4DVAR_GRAPHS=graphs), timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        res[graphs] = np.load(out)
    assert np.array_equal(res["1"][0], res["1"][1])   # replays are deterministic
    assert np.array_equal(res["1"][0], res["0"][0])   # and equal to eager launches


@pytest.mark.parametrize("M,N,K", [(1000, 336, 1000), (500, 336, 500), (64, 8128, 512)])
def test_gemm_split_k_concurrent_streams(M, N, K):
    """Too few 64x128 tiles to fill the GPU (48, 24, 64): the tile-config fallback by
    default, split-K (per-stream partial workspaces, fixed-order reduction) with
    WF4DVAR_GEMM_SPLITK=1 -- same tolerance, bitwise reproducible, and independent
    launches on two streams at once (the split-K path: test_gemm_split_k_opt_in)."""
    g = torch.Generator().manual_seed(M + N + K)
    mats = []
    for _ in range(2):
        A = torch.randn(M, K, generator=g, dtype=torch.float64).cuda()
        X = torch.randn(K, N, generator=g, dtype=torch.float64).cuda()
        Z = torch.randn(M, N, generator=g, dtype=torch.float64).cuda()
        mats.append((A, X, Z, 0.75 * (A @ X) - 2.0 * Z))
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    first = None
    for rep in range(4):
        outs = []
        for (A, X, Z, _), s in zip(mats, (s1, s2)):
            Y = torch.empty(M, N, dtype=torch.float64, device="cuda")
            with torch.cuda.stream(s):
                L().test_gemm(A, X, Y, alpha=0.75, beta=-2.0, Z=Z, stream=s.cuda_stream)
            outs.append(Y)
        torch.cuda.synchronize()
        for (A, X, Z, ref), Y in zip(mats, outs):
            scale = (A.abs() @ X.abs()).max().item() + 1.0
            assert (Y - ref).abs().max().item() <= 1e-14 * scale * K ** 0.5 * 4, rep
        if first is None:
            first = [o.clone() for o in outs]
        else:
            assert all(torch.equal(a, b) for a, b in zip(first, outs))


SPLITK = r"""
import sys, torch
sys.path.insert(0, sys.argv[1])
from paper_2105_06975_b200 import _lib
g = torch.Generator().manual_seed(9)
for (M, N, K) in ((1000, 336, 1000), (500, 336, 500), (64, 8128, 512), (300, 517, 700)):
    A = torch.randn(M, K, generator=g, dtype=torch.float64).cuda()
    X = torch.randn(K, N, generator=g, dtype=torch.float64).cuda()
    Z = torch.randn(M, N, generator=g, dtype=torch.float64).cuda()
    Y = torch.empty(M, N, dtype=torch.float64, device="cuda")
    _lib.test_gemm(A, X, Y, alpha=0.5, beta=1.5, Z=Z)
    Y2 = torch.empty_like(Y)
    _lib.test_gemm(A, X, Y2, alpha=0.5, beta=1.5, Z=Z)
    ref = 0.5 * (A @ X) + 1.5 * Z
    scale = (A.abs() @ X.abs()).max().item() + 1.0
    assert (Y - ref).abs().max().item() <= 1e-14 * scale * K ** 0.5 * 4, (M, N, K)
    assert torch.equal(Y, Y2)
print("ok")
"""


def test_gemm_split_k_opt_in():
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", SPLITK, root], capture_output=True, text=True,
                       env=dict(os.environ, WF4DVAR_GEMM_SPLITK="1"), timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]
