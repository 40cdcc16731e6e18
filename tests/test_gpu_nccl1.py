"""GPU: the NCCL transport on one device (a 1-rank communicator).

Every gpurun box has a single B200 and NCCL refuses two ranks on one GPU, so the
multi-GPU NCCL exchange cannot run here; this checks the rest of the NCCL path --
dlopen of libnccl.so.2, ncclGetUniqueId / ncclCommInitRank through the C ABI, and
the collectives the solver issues (allreduce of the Krylov inner products,
allgather of the L_I window sums) -- against the transport-free context."""
import numpy as np
import pytest

from synth import configs as SC

from .helpers import seeded_vec

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("pc,solver", [(dict(shape="PD", lhat="LI", k=1, rhat="exact"), "minres"),
                                       (dict(shape="PI", lhat="LM", k=3, rhat="rr"), "gmres")])
def test_nccl_one_rank_matches_plain(pc, solver):
    import paper_2105_06975_b200 as W
    prob = SC.custom_problem(s=200, N=7, q=2, m=3, seed0=2)
    plain = W.Context.from_problem(prob, pc)
    nc = W.Context.from_problem(prob, pc, rank=0, world=1, nccl_id=W.nccl_unique_id())
    x = torch.from_numpy(seeded_vec(prob.n, 4)).cuda()
    for which in ("apply_A", "apply_P"):
        y1, y2 = torch.empty_like(x), torch.empty_like(x)
        getattr(plain, which)(x, y1)
        getattr(nc, which)(x, y2)
        torch.cuda.synchronize()
        assert torch.equal(y1, y2), which
    b = torch.from_numpy(prob.rhs).cuda()
    x1, x2 = torch.empty_like(b), torch.empty_like(b)
    r1 = plain.solve(b, x1, solver=solver, tol=1e-10, maxit=2000, restart=0)
    r2 = nc.solve(b, x2, solver=solver, tol=1e-10, maxit=2000, restart=0)
    assert np.array_equal(r1["iters"], r2["iters"])
    assert torch.equal(x1, x2)
