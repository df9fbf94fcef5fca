"""The robot-sharded decision round (rounds.ShardedDecisionRound) with its CUDA
primitives: 2 ranks sharing cuda:0 over gloo (one B200 in this environment; on
a multi-GPU box the same code runs one rank per GPU over NCCL).  Global
admission, the ordered global S_e and every rank's masks / skip counters must
equal a single-GPU DecisionRound over the whole fleet."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as orc

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, sizes, k, q, overlap=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2605_11381_b200 import fleet as fl, rounds, synthetic
        lo = sum(sizes[:rank])
        soa = synthetic.fleet_soa(sum(sizes), seed=21)
        mine = {k2: (v[lo:lo + sizes[rank]] if isinstance(v, np.ndarray) and k2 != "slots" else v)
                for k2, v in soa.items()}
        # re-base this shard's CSR history
        off = soa["hist_off"][lo:lo + sizes[rank]]
        nsl = np.maximum(soa["n_exec"], soa["n_gen"])[lo:lo + sizes[rank]]
        rows = np.concatenate([np.arange(o, o + n) for o, n in zip(off, nsl)]) if len(off) else []
        mine["slots"] = soa["slots"][np.asarray(rows, np.int64)] if len(rows) else np.zeros((1, 4), np.int64)
        mine["hist_off"] = np.concatenate([[0], np.cumsum(nsl)[:-1]]).astype(np.int64)
        mine["n"] = sizes[rank]
        base = int(soa["issued_at"].min())
        sched = fl.sched_struct("kairos", 10, 5, 150_000, 166_667, synthetic.NOW, 30, base)
        fleet = fl.DeviceFleet.from_host(mine)
        rnd = rounds.ShardedDecisionRound(sizes[rank], k, sched)
        H = None
        if overlap:  # the bench's N > 1 path: horizons || (urgency + sharded admission)
            prev, cand, off = synthetic.chunks(sum(sizes), seed=22)
            sl = slice(lo, lo + sizes[rank])
            inputs = rounds.DivergenceInputs(prev[sl].contiguous(), cand[sl].contiguous(), 0.9,
                                             offset=off[sl].contiguous())
            rnd.run_overlapped(fleet, inputs, reserve_sms=24)
            H = rnd.H.cpu().numpy()
        else:
            rnd.urgency(fleet)
            rnd.admit(fleet)
        torch.cuda.synchronize()
        q.put((rank, rnd.admitted.cpu().numpy(), fleet.t["skipped"].cpu().numpy(),
               rnd.global_edge[: rnd.k_global].cpu().numpy(), H))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("sizes,k,overlap", [([30000, 20000], 4096, False),
                                             ([100, 5000], 300, False),
                                             ([2000, 2000], 3990, False),
                                             ([30000, 20000], 4096, True)])
def test_sharded_round_matches_single_gpu(sizes, k, overlap):
    from paper_2605_11381_b200 import fleet as fl, rounds, synthetic
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, len(sizes), port, sizes, k, q, overlap))
             for r in range(len(sizes))]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in sizes], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    soa = synthetic.fleet_soa(sum(sizes), seed=21)
    sched = fl.sched_struct("kairos", 10, 5, 150_000, 166_667, synthetic.NOW, 30,
                            int(soa["issued_at"].min()))
    fleet = fl.DeviceFleet.from_host(soa)
    ref = rounds.DecisionRound(sum(sizes), k, sched)
    if overlap:
        prev, cand, off = synthetic.chunks(sum(sizes), seed=22)
        ref.run(fleet, rounds.DivergenceInputs(prev, cand, 0.9, offset=off))
    else:
        ref.urgency(fleet)
        ref.admit(fleet)
    torch.cuda.synchronize()
    if overlap:
        assert np.array_equal(np.concatenate([r[4] for r in res]), ref.H.cpu().numpy())
        assert np.array_equal(np.concatenate([r[4] for r in res]), orc.divergence_batch(
            prev.cpu().numpy(), cand.cpu().numpy(), 0.9, off.cpu().numpy()))
    adm = np.concatenate([r[1] for r in res])
    skp = np.concatenate([r[2] for r in res])
    assert np.array_equal(adm, ref.admitted.cpu().numpy())
    assert np.array_equal(skp, fleet.t["skipped"].cpu().numpy())
    for r in res:  # identical ordered global S_e on every rank == single-GPU S_e keys
        assert np.array_equal(r[3], ref.edge_keys[:k].cpu().numpy())
    # and == the oracle's plan() (not only the single-GPU round): membership,
    # skip counters, and the global S_e order (the key's low 24 bits carry
    # the robot's global lexrank == its index here)
    orc_res = orc.plan_soa(soa, "kairos", 10, 5, 150_000, 166_667, synthetic.NOW, 30, k)
    assert np.array_equal(adm, orc_res["admitted"])
    assert np.array_equal(skp, orc_res["skipped_out"])
    kk = min(k, sum(sizes))
    for r in res:
        assert np.array_equal(r[3][:, 1] & 0xFFFFFF, orc_res["order"][:kk])


def _dup_worker(rank, world, port, q):
    """Both ranks hold the same robots with shard-local ranks: every key occurs
    on both shards, which the merge must report instead of over-admitting."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2605_11381_b200 import fleet as fl, rounds, synthetic
        soa = synthetic.fleet_soa(3000, seed=23)
        sched = fl.sched_struct("kairos", 10, 5, 150_000, 166_667, synthetic.NOW, 30,
                                int(soa["issued_at"].min()))
        rnd = rounds.ShardedDecisionRound(3000, 500, sched)
        fleet = fl.DeviceFleet.from_host(soa)
        rnd.urgency(fleet)
        rnd.admit(fleet)
        try:
            rnd.check()
            q.put((rank, "no error"))
        except ValueError as e:
            q.put((rank, str(e)))
        # mismatched round scalars are rejected up front
        other = fl.sched_struct("kairos", 10, 5, 150_000, 166_667, synthetic.NOW, 30,
                                int(soa["issued_at"].min()) - rank)
        try:
            rounds.ShardedDecisionRound(3000, 500, other)
            q.put((rank, "no error"))
        except ValueError as e:
            q.put((rank, str(e)))
    finally:
        dist.destroy_process_group()


def test_sharded_duplicate_keys_flagged():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_dup_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    msgs = [q.get(timeout=300) for _ in range(4)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert sum("same priority key" in m for _, m in msgs) == 2
    assert sum("same kr_sched" in m for _, m in msgs) == 2


def _nccl_capture_worker(port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        from paper_2605_11381_b200 import fleet as fl, rounds, synthetic
        R, k = 50_000, 4096
        soa = synthetic.fleet_soa(R, seed=31)
        fleet = fl.DeviceFleet.from_host(soa)
        sched = fl.sched_struct("kairos", 10, 5, 150_000, 166_667, synthetic.NOW, 30,
                                int(soa["issued_at"].min()))
        prev, cand, off = synthetic.chunks(R, seed=32)
        inputs = rounds.DivergenceInputs(prev, cand, 0.9, offset=off)
        rnd = rounds.ShardedDecisionRound(R, k, sched)
        skipped0 = fleet.t["skipped"].clone()
        rnd.capture(fleet, inputs, reserve_sms=10, layout="split")
        outs = []
        for _ in range(3):  # capture() ran one (warm-up) round; replay three more
            rnd.replay()
            torch.cuda.synchronize()
            outs.append((rnd.admitted.cpu().numpy(), fleet.t["skipped"].cpu().numpy().copy(),
                         rnd.global_edge[: rnd.k_global].cpu().numpy(), rnd.H.cpu().numpy()))
        rnd.check()
        q.put((skipped0.cpu().numpy(), outs, None))
    except Exception as e:  # noqa: BLE001
        q.put((None, None, repr(e)))
    finally:
        dist.destroy_process_group()


def test_sharded_round_captured_over_nccl():
    """The sharded round captured in CUDA graphs with the NCCL all-gather
    inside (one rank): every replayed round == the oracle's plan on the evolving
    skip counters, horizons == the oracle's."""
    from paper_2605_11381_b200 import synthetic
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_capture_worker, args=(_port(), q))
    p.start()
    skipped0, outs, err = q.get(timeout=600)
    p.join(timeout=60)
    assert err is None, err
    R, k = 50_000, 4096
    soa = synthetic.fleet_soa(R, seed=31)
    prev, cand, off = synthetic.chunks(R, seed=32)
    H = orc.divergence_batch(prev.cpu().numpy(), cand.cpu().numpy(), 0.9, off.cpu().numpy())
    # capture() runs one eager warm-up round (recording executes nothing);
    # replay i sees the skip counters after 1 + i rounds
    cur = dict(soa)
    cur["skipped"] = skipped0.copy()
    for _ in range(1):
        res = orc.plan_soa(cur, "kairos", 10, 5, 150_000, 166_667, synthetic.NOW, 30, k)
        cur["skipped"] = res["skipped_out"]
    for adm, sk, edge, h in outs:
        res = orc.plan_soa(cur, "kairos", 10, 5, 150_000, 166_667, synthetic.NOW, 30, k)
        assert np.array_equal(adm, res["admitted"])
        assert np.array_equal(sk, res["skipped_out"])
        assert np.array_equal(h, H)
        cur["skipped"] = res["skipped_out"]
        del edge
