"""Host-side logic of the subtree-sharded path on CPU.

* ShardPlan invariants for many tree shapes and rank counts.
* The real TorchComm point-to-point exchange over gloo (world_size 2 and 4,
  127.0.0.1 rendezvous): every rank fills the update / solve-block slots of
  the fronts it owns, runs the same transfer methods ShardedFactorization
  uses, and checks it received exactly the slots its parents need.
"""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2306_08994_b200 import _lib
from paper_2306_08994_b200.distributed import ShardPlan, ShardedFactorization, TorchComm


def level_sizes(n_leaves):
    s = [n_leaves]
    while s[-1] > 1:
        s.append((s[-1] + 1) // 2)
    return s


@pytest.mark.parametrize("n_leaves", [1, 2, 5, 7, 8, 13, 64, 100, 1000, 4096])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_shard_plan_invariants(n_leaves, world):
    sizes = level_sizes(n_leaves)
    sp = ShardPlan(sizes, world)
    for L, ls in enumerate(sp.levels):
        # every front owned by exactly one rank; owned ranges contiguous and disjoint
        cover = np.zeros(sizes[L], dtype=int)
        for r, (f0, f1) in enumerate(ls.ranges):
            cover[f0:f1] += 1
            assert np.all(ls.owner[f0:f1] == r)
        assert np.all(cover == 1)
        if L > 0:
            # a subtree below the split never changes owner
            for c in range(sizes[L - 1]):
                if L <= sp.split:
                    assert ls.owner[c >> 1] == sp.levels[L - 1].owner[c]
            # every remote child of an owned parent is transferred into a held slot
            for c, q, p in sp.upward(L):
                lo, hi = sp.levels[L - 1].slots[p]
                assert lo <= c < hi and q != p
    if n_leaves >= world:
        assert all(f1 > f0 for f0, f1 in sp.levels[sp.split].ranges)


class _FakeLevel:
    def __init__(self, n, upd, max_m):
        self.n_fronts, self.upd_stride, self.fac_stride, self.aux_stride = n, upd, 4, 0
        self.max_m = max_m
        v = _lib.LevelView()
        v.n_fronts, v.max_m, v.max_k = n, max_m, 1
        self.view = v


class _FakeDP:
    """Just the attributes ShardedFactorization's buffer logic reads."""

    def __init__(self, sizes):
        self.device = torch.device("cpu")
        self.levels = [_FakeLevel(n, 3 + L, 2 + L) for L, n in enumerate(sizes)]
        self.lib = _lib.load()
        self.n_pivots = 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, sizes, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dp = _FakeDP(sizes)
        sh = ShardedFactorization(dp, world, TorchComm(), ranks=[rank])
        st = sh.state[rank]
        errors = []
        # factor-direction transfers of update slots, level by level
        for L in range(1, len(sizes)):
            f0, f1 = sh.shard.levels[L - 1].ranges[rank]
            for c in range(f0, f1):
                st.upd_slot(L - 1, c).fill_(1000.0 * L + c)
            sh._transfer_upward(L)
            p0, p1 = sh.shard.levels[L].ranges[rank]
            for p in range(p0, p1):
                for c in (2 * p, 2 * p + 1):
                    if c < sizes[L - 1]:
                        got = st.upd_slot(L - 1, c)
                        if not torch.all(got == 1000.0 * L + c):
                            errors.append(("up", L, c))
        # solve-block transfers (forward up, backward down)
        sh._prepare_solve(2)
        for L in range(len(sizes) - 2, -1, -1):
            p0, p1 = sh.shard.levels[L + 1].ranges[rank]
            for p in range(p0, p1):
                sh._blk_slot(rank, L + 1, p, 2).fill_(-7.0 * (L + 1) - p)
            sh._move(sh.shard.downward(L), L + 1, 2)
            c0, c1 = sh.shard.levels[L].ranges[rank]
            for c in range(c0, c1):
                got = sh._blk_slot(rank, L + 1, c >> 1, 2)
                if not torch.all(got == -7.0 * (L + 1) - (c >> 1)):
                    errors.append(("down", L, c))
        q.put((rank, errors))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n_leaves", [(2, 13), (2, 64), (4, 37), (4, 256)])
def test_gloo_exchanges(world, n_leaves):
    sizes = level_sizes(n_leaves)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, sizes, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=60) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs)
    for r in range(world):
        assert results[r] == [], results[r]
