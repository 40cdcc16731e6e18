"""Algorithm 1 host logic on the CPU: the block structure the
library computes for R_block (wf4dvar_rblock_plan, the setup step of create)
against the oracle's Algorithm 1 (oracle/rhat.py r_block), and the paper's
block-structured synthetic R_i recipe (synth.paper_block_R)."""
import numpy as np
import pytest

from oracle import rhat as RH
from synth import configs as SC

PVECS = [[20, 30, 10, 25, 15], [8] * 12 + [4], [50, 50], [7, 1, 9, 3, 12, 5, 13]]


def _Rs():
    out = []
    for i, pv in enumerate(PVECS):
        out.append((pv, SC.paper_block_R(pv, seed=i)))
        rng = np.random.default_rng(i)
        A = rng.standard_normal((sum(pv), sum(pv)))
        out.append((pv, A @ A.T / sum(pv) + 0.1 * np.eye(sum(pv))))
    return out


@pytest.mark.parametrize("maxsize", [0, 10, 40])
@pytest.mark.parametrize("numproc", [0, 2, 4, 20])
def test_library_blocks_match_oracle_algorithm1(maxsize, numproc):
    import paper_2105_06975_b200 as W
    for pv, R in _Rs():
        _, _, normvec = RH.r_block(R, pv)
        for tol in [0.0, float(np.min(normvec)) * 0.999, float(np.median(normvec)),
                    float(np.max(normvec)) * 1.001, np.inf]:
            got = W.rblock_plan(R, pv, tol, maxsize, numproc)
            ref = RH.r_block(R, pv, tol, maxsize or None, numproc or None)[1]
            assert got == [(int(a), int(b)) for a, b in ref], (pv, tol, maxsize, numproc)


def test_tol_limits():
    import paper_2105_06975_b200 as W
    pv, R = _Rs()[0]
    assert W.rblock_plan(R, pv, 0.0) == [(0, sum(pv))]                  # no cut
    st = np.concatenate([[0], np.cumsum(pv)])
    assert W.rblock_plan(R, pv, np.inf) == list(zip(st[:-1], st[1:]))    # every cut


def test_rblock_plan_rejects_bad_pvec():
    import paper_2105_06975_b200 as W
    R = np.eye(10)
    with pytest.raises(W.WF4DVarError):
        W.rblock_plan(R, [3, 3, 3])        # sum(pvec) != p


def test_paper_block_R_recipe():
    pv = [20, 30, 10, 25, 15]
    R = SC.paper_block_R(pv, seed=3)
    assert np.allclose(R, R.T)
    lam = np.linalg.eigvalsh(R)
    assert lam[0] > 0
    # "if the minimum eigenvalue of R_i is less than 1 it is increased to ... 0.41"
    assert lam[0] >= 0.41 - 1e-12
    # pcorr_k = 0: the corresponding off-diagonal block is uncorrelated
    nb = len(pv)
    R0 = SC.paper_block_R(pv, pcorr=np.zeros(nb * (nb - 1) // 2), seed=3)
    st = np.concatenate([[0], np.cumsum(pv)])
    for k in range(nb):
        for l in range(k + 1, nb):
            assert not R0[st[k]:st[k + 1], st[l]:st[l + 1]].any()
    # then Algorithm 1 with any finite tol > 0 recovers exactly the pvec blocks
    import paper_2105_06975_b200 as W
    assert W.rblock_plan(R0, pv, 1e-12) == list(zip(st[:-1], st[1:]))
