"""Multi-process (gloo, world_size 2 and 3, CPU) test of the robot-sharded
admission protocol `rounds.sharded_topk`: local top-k' candidates, one
all-gather, identical merge on every rank, local application of the global
k-th key.  The device primitives are replaced by a numpy twin (same contract
as rounds.CudaShardOps), so this exercises the host protocol without a GPU."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

SENTINEL = np.array([np.iinfo(np.uint64).max] * 2, np.uint64)


def _sorted_idx(k):
    return np.lexsort((k[:, 1], k[:, 0]))


class NumpyShardOps:
    def __init__(self):
        self.admitted = None

    def local_candidates(self, keys, kl, kg):
        out = np.tile(SENTINEL, (kg, 1))
        out[:kl] = keys[_sorted_idx(keys)[:kl]]
        return out

    def all_gather(self, cand):
        t = torch.from_numpy(cand.view(np.int64).copy())
        outs = [torch.empty_like(t) for _ in range(dist.get_world_size())]
        dist.all_gather(outs, t)
        return torch.cat(outs).numpy().view(np.uint64)

    def merge(self, runs, W, kg, want_kth):
        s = runs[_sorted_idx(runs)]
        return s[:kg], (s[kg - 1] if want_kth else None)

    def apply(self, keys, k, kth):
        if k == 0:
            self.admitted = np.zeros(len(keys), bool)
        elif kth is None:
            self.admitted = np.ones(len(keys), bool)
        else:
            self.admitted = (keys[:, 0] < kth[0]) | ((keys[:, 0] == kth[0]) & (keys[:, 1] <= kth[1]))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, sizes, k, seed, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2605_11381_b200.rounds import sharded_topk
        rng = np.random.default_rng(seed)
        total = sum(sizes)
        allkeys = np.stack([rng.integers(0, 50, total, dtype=np.uint64) << np.uint64(50),
                            (rng.integers(0, 1000, total, dtype=np.uint64) << np.uint64(24))
                            | np.arange(total, dtype=np.uint64)], 1)
        lo = sum(sizes[:rank])
        mine = allkeys[lo:lo + sizes[rank]]
        ops = NumpyShardOps()
        kg, edge = sharded_topk(mine, len(mine), k, sizes, ops)
        q.put((rank, kg, None if edge is None else edge.copy(), ops.admitted, lo))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("sizes,k", [([100, 100], 10), ([5, 300], 40), ([0, 50], 7),
                                     ([30, 20], 80), ([1000, 1, 999], 500), ([3, 3, 3], 9)])
def test_sharded_topk_equals_global(sizes, k):
    world = len(sizes)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, sizes, k, 17, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(17)
    total = sum(sizes)
    allkeys = np.stack([rng.integers(0, 50, total, dtype=np.uint64) << np.uint64(50),
                        (rng.integers(0, 1000, total, dtype=np.uint64) << np.uint64(24))
                        | np.arange(total, dtype=np.uint64)], 1)
    order = _sorted_idx(allkeys)
    kg = min(k, total)
    want = np.zeros(total, bool)
    want[order[:kg]] = True
    got = np.zeros(total, bool)
    for rank, kgr, edge, adm, lo in res:
        assert kgr == kg
        got[lo:lo + len(adm)] = adm
        if kg:
            assert np.array_equal(edge, allkeys[order[:kg]])   # identical ordered S_e everywhere
    assert np.array_equal(got, want)
