"""Multi-rank (time-window-sharded) host logic on the CPU: world_size 2-4 gloo
process groups.

What is checked: the library's own partition (wf4dvar_partition) and L_hat
chain schedule (wf4dvar_chain_plan) -- the host logic that decides which windows
each rank updates at each chain step and when a running chain state crosses a
rank boundary -- executed rank by rank with the oracle's model matrices and real
point-to-point messages (torch.distributed gloo send/recv), must reproduce the
oracle's global L_hat^{-1} / L_hat^{-T} (Lemma 4.2) exactly.  The halo
pattern the ABI documents for L / L^T and the allgather pattern of
the L_I scan are exercised the same way.  The CUDA kernels that
consume these schedules are covered on the GPU (test_gpu_dist.py).
"""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import lhat as LH

CASES = [(5, 2), (5, 3), (10, 4), (10, 1), (10, 10), (16, 4), (16, 3), (7, 7), (9, 2)]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _Ms(N, s, seed=0):
    rng = np.random.default_rng(seed)
    return [rng.standard_normal((s, s)) / math.sqrt(s) for _ in range(N)]


def _send(t, peer):
    dist.send(torch.from_numpy(np.ascontiguousarray(t)), peer)


def _recv(shape, peer):
    buf = torch.empty(shape, dtype=torch.float64)
    dist.recv(buf, peer)
    return buf.numpy()


def _chain_solve_sharded(W_, k, Ms, r, rank, world, transpose):
    """Run the library's chain plan on this rank's windows (emulating the kernel
    z_w = r_w + M_w z_{w-1} / z_w = r_w + M_{w+1}^T z_{w+1} and the hand-offs)."""
    import paper_2105_06975_b200 as WF
    w0, w1 = WF.partition(W_, world, rank)
    z = [r[w].copy() for w in range(w0, w1)]
    s = r[0].shape[0]
    halo = None
    if k <= 1:
        return z
    for st in WF.chain_plan(W_, k, w0, w1, transpose):
        # ordered so that gloo's blocking send/recv cannot deadlock: sends first
        # travel away from the receiving direction
        if st["send"]:
            _send(z[-1] if not transpose else z[0], rank + 1 if not transpose else rank - 1)
        if st["recv"]:
            halo = _recv((s,), rank - 1 if not transpose else rank + 1)
        for first, stride, count in st["launches"]:
            for t in range(count):
                wl = first + t * stride
                wg = w0 + wl
                if not transpose:
                    src = z[wl - 1] if wl >= 1 else halo
                    z[wl] = z[wl] + Ms[wg - 1] @ src
                else:
                    src = z[wl + 1] if wl + 1 < len(z) else halo
                    z[wl] = z[wl] + Ms[wg].T @ src
    return z


def _worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2105_06975_b200 as WF
        fails = []
        s = 3
        for W_, k in CASES:
            if world > W_:
                continue
            N = W_ - 1
            Ms = _Ms(N, s, seed=W_ * 100 + k)
            rng = np.random.default_rng(7)
            r = [rng.standard_normal(s) for _ in range(W_)]
            w0, w1 = WF.partition(W_, world, rank)
            for transpose in (False, True):
                kind = "L" if k == W_ else "LM"
                z = _chain_solve_sharded(W_, k, Ms, r, rank, world, transpose)
                allz = [None] * world
                dist.all_gather_object(allz, (w0, z))
                if rank == 0:
                    zg = [v for _, zz in sorted(allz, key=lambda t: t[0]) for v in zz]
                    ref = (LH.solve_T if transpose else LH.solve)(kind, Ms, r, None if kind == "L" else k)
                    err = max(np.abs(a - b).max() for a, b in zip(zg, ref))
                    if err > 1e-12:
                        fails.append((W_, k, transpose, err))
            # L x and L^T x with the ABI's halo pattern: x3 of the last window goes to
            # rank+1 (for L), x1 of the first window to rank-1 (for L^T)
            x = [rng.standard_normal(s) for _ in range(W_)]
            xl = [x[w].copy() for w in range(w0, w1)]
            lo = hi = None
            if rank + 1 < world:
                _send(xl[-1], rank + 1)
            if rank > 0:
                lo = _recv((s,), rank - 1)
                _send(xl[0], rank - 1)
            if rank + 1 < world:
                hi = _recv((s,), rank + 1)
            Lx = [xl[i] - Ms[w0 + i - 1] @ (xl[i - 1] if i else lo) if w0 + i >= 1 else xl[i].copy()
                  for i in range(len(xl))]
            LTx = [xl[i] - Ms[w0 + i].T @ (xl[i + 1] if i + 1 < len(xl) else hi)
                   if w0 + i + 1 < W_ else xl[i].copy() for i in range(len(xl))]
            # L_I scan: local inclusive scan + allgather of per-rank totals (rank order)
            sc = list(np.cumsum(np.array(xl), axis=0))
            tots = [None] * world
            dist.all_gather_object(tots, sc[-1])
            pre = sum((tots[q] for q in range(rank)), np.zeros(s))
            LIinv = [v + pre for v in sc]
            allv = [None] * world
            dist.all_gather_object(allv, (w0, Lx, LTx, LIinv))
            if rank == 0:
                parts = sorted(allv, key=lambda t: t[0])
                g = lambda i: [v for p in parts for v in p[i]]
                for name, got, ref in (("L", g(1), LH.apply("L", Ms, x)),
                                       ("LT", g(2), LH.apply_T("L", Ms, x)),
                                       ("LI^-1", g(3), LH.solve("LI", Ms, x))):
                    err = max(np.abs(a - b).max() for a, b in zip(got, ref))
                    if err > 1e-12:
                        fails.append((W_, name, err))
        if rank == 0:
            out_q.put(fails)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3, 4])
def test_sharded_chain_schedule_matches_oracle(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    fails = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert fails == []


def test_partition_is_contiguous_and_balanced():
    import paper_2105_06975_b200 as WF
    for W_ in (1, 5, 21, 32, 128):
        for world in range(1, min(W_, 9) + 1):
            b = [WF.partition(W_, world, r) for r in range(world)]
            assert b[0][0] == 0 and b[-1][1] == W_
            assert all(b[i][1] == b[i + 1][0] for i in range(world - 1))
            sizes = [e - s for s, e in b]
            assert max(sizes) - min(sizes) <= 1 and min(sizes) >= 1
    assert WF.partition(128, 8, 3) == (48, 64)


def test_chain_plan_single_rank_reproduces_lemma42_launches():
    """world = 1: forward step j updates windows j, j+k, ... (w mod k == j); backward
    step j the windows j before their chain end; no messages."""
    import paper_2105_06975_b200 as WF
    for W_, k in ((128, 4), (21, 4), (5, 3), (7, 7)):
        f = WF.chain_plan(W_, k, 0, W_, 0)
        assert [st["j"] for st in f] == list(range(1, min(k, W_)))
        for st in f:
            assert not st["recv"] and not st["send"]
            first, stride, count = st["launches"][0]
            assert first == st["j"] and stride == k and count == (W_ - 1 - st["j"]) // k + 1
        b = WF.chain_plan(W_, k, 0, W_, 1)
        for st in b:
            covered = sorted(f0 + t * sd for f0, sd, c in st["launches"] for t in range(c))
            ends = [min((w // k + 1) * k, W_) - 1 for w in covered]
            assert all(e - w == st["j"] for w, e in zip(covered, ends))


def test_aligned_chains_need_no_messages():
    """k divides every rank's first window (c3: 128 windows, k = 4, 1-8 ranks):
    the parallel-in-time preconditioner needs no communication."""
    import paper_2105_06975_b200 as WF
    for world in (1, 2, 4, 8):
        for r in range(world):
            b, e = WF.partition(128, world, r)
            for tr in (0, 1):
                assert all(not st["recv"] and not st["send"]
                           for st in WF.chain_plan(128, 4, b, e, tr))


def test_local_global_windows_roundtrip():
    import paper_2105_06975_b200 as WF
    s, p, W_, m = 4, 2, 7, 3
    v = np.arange((2 * s + p) * W_ * m, dtype=np.float64)
    for world in (1, 2, 3):
        bounds = [WF.partition(W_, world, r) for r in range(world)]
        parts = [WF.local_windows(v, s, p, W_, m, b, e) for b, e in bounds]
        assert sum(x.size for x in parts) == v.size
        np.testing.assert_array_equal(WF.global_windows(parts, s, p, m, bounds), v)
