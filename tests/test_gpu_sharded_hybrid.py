"""The robot-sharded round with a cloud tier (rounds.ShardedHybridRound): 2
ranks sharing cuda:0 over gloo.  Edge and cloud placements, every rank's
masks, skip counters and refetch flags must equal the single-GPU
HybridDecisionRound over the whole fleet (itself pinned to the reference's
hybrid plan())."""

from __future__ import annotations

import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from test_gpu_sharded import _port

pytestmark = pytest.mark.gpu

K, CAP = 3000, 1500


def _engines():
    from paper_2605_11381_b200 import engines as eng
    edge = eng.EngineProfile(tier="edge", capacity=K, max_batch=256,
                             points=((1, 150_000), (256, 400_000)))
    cloud = eng.EngineProfile(tier="cloud", capacity=CAP, max_batch=512,
                              points=((1, 80_000), (512, 250_000)))
    net = eng.NetworkModel(base_latency_us=20_000, uplink_bps=int(4e7), downlink_bps=int(1e9))
    return edge, cloud, net


def _payload(n):
    return np.random.default_rng(5).choice(np.array([100_000, 300_000, 2_000_000], np.int64), n)


def _worker(rank, world, port, sizes, window, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2605_11381_b200 import engines as eng, fleet as fl, rounds, synthetic
        lo = sum(sizes[:rank])
        soa = synthetic.fleet_soa(sum(sizes), seed=21)
        mine = {k2: (v[lo:lo + sizes[rank]] if isinstance(v, np.ndarray) and k2 != "slots" else v)
                for k2, v in soa.items()}
        off = soa["hist_off"][lo:lo + sizes[rank]]
        nsl = np.maximum(soa["n_exec"], soa["n_gen"])[lo:lo + sizes[rank]]
        rows = np.concatenate([np.arange(o, o + n) for o, n in zip(off, nsl)])
        mine["slots"] = soa["slots"][rows]
        mine["hist_off"] = np.concatenate([[0], np.cumsum(nsl)[:-1]]).astype(np.int64)
        mine["n"] = sizes[rank]
        sched = fl.sched_struct("kairos", 10, 5, 150_000, 166_667, synthetic.NOW, 30,
                                int(soa["issued_at"].min()))
        fleet = fl.DeviceFleet.from_host(mine)
        edge, cloud, net = _engines()
        rnd = rounds.ShardedHybridRound(sizes[rank], K, sched, CAP, window=window)
        up = eng.transfer_time_batch(net, torch.from_numpy(_payload(sum(sizes))[lo:lo + sizes[rank]]).cuda(),
                                     eng.UP)
        rnd.set_cloud(up, eng.cloud_thresholds(edge, cloud, net, 0, 0, rnd.k_global, rnd.cap))
        rnd.urgency(fleet)
        rnd.admit(fleet)
        torch.cuda.synchronize()
        q.put((rank, rnd.admitted.cpu().numpy(), fleet.t["skipped"].cpu().numpy(),
               rnd.refetch.cpu().numpy(), rnd.global_edge[: rnd.k_global].cpu().numpy(),
               rnd.cloud().cpu().numpy(), rnd.widened))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("sizes,window", [([30000, 20000], None), ([30000, 20000], 100),
                                          ([700, 9000], None)])
def test_sharded_hybrid_matches_single_gpu(sizes, window):
    from paper_2605_11381_b200 import engines as eng, fleet as fl, rounds, synthetic
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, len(sizes), port, sizes, window, q))
             for r in range(len(sizes))]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in sizes], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    n = sum(sizes)
    soa = synthetic.fleet_soa(n, seed=21)
    sched = fl.sched_struct("kairos", 10, 5, 150_000, 166_667, synthetic.NOW, 30,
                            int(soa["issued_at"].min()))
    fleet = fl.DeviceFleet.from_host(soa)
    edge, cloud, net = _engines()
    ref = rounds.HybridDecisionRound(n, K, sched, CAP)
    ref.set_cloud(eng.transfer_time_batch(net, torch.from_numpy(_payload(n)).cuda(), eng.UP),
                  eng.cloud_thresholds(edge, cloud, net, 0, 0, ref.k, ref.cap))
    ref.urgency(fleet)
    ref.admit(fleet)
    torch.cuda.synchronize()
    assert np.array_equal(np.concatenate([r[1] for r in res]), ref.admitted.cpu().numpy())
    assert np.array_equal(np.concatenate([r[2] for r in res]), fleet.t["skipped"].cpu().numpy())
    assert np.array_equal(np.concatenate([r[3] for r in res]), ref.refetch.cpu().numpy())
    ref_cloud_keys = ref.keys[ref.cloud().long()].cpu().numpy()
    assert len(ref_cloud_keys) > 0
    ref_edge = ref.outputs().edge_keys.cpu().numpy()
    for r in res:  # identical ordered global S_e and offload order on every rank
        assert np.array_equal(r[4], ref_edge)
        assert np.array_equal(r[5], ref_cloud_keys)
    if window == 100:
        assert res[0][6] > 0  # the narrow window had to widen
