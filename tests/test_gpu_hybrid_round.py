"""Fleet-scale hybrid round (rounds.HybridDecisionRound: full order, edge
admission, phase-3 cloud offload scan) against the reference's own hybrid
plan() decisions (tests/golden/plan_cloud.json: 80 instances, 381 cloud
placements), and against the object-level plan() on a synthetic fleet."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import golden_io

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def kb():
    import paper_2605_11381_b200 as kb
    return kb


def _hybrid(kb, pending, states, edge, cloud, net, now, cfg, edge_in_flight, cloud_in_flight,
            window=None):
    from paper_2605_11381_b200 import engines as eng, fleet as fl, rounds, scheduler as sch
    from paper_2605_11381_b200 import device as dev
    reqs = list(pending)
    n = len(reqs)
    rank = sch._ranks([r.task_id for r in reqs])
    issued = np.array([r.issued_at for r in reqs], np.int64)
    sched = fl.sched_struct(cfg.policy, cfg.buckets, cfg.aging_interval, cfg.stale_threshold,
                            cfg.default_exec_estimate, int(now), 1, sch._issued_base(issued))
    fleet = fl.DeviceFleet.from_host(fl.host_soa(reqs, states, rank))
    k = min(max(0, edge.capacity - edge_in_flight) if edge is not None else 0, n)
    cloud_avail = max(0, cloud.capacity - cloud_in_flight) if cloud is not None else 0
    cap = min(cloud_avail, n - k) if (cloud is not None and net is not None) else 0
    rnd = rounds.HybridDecisionRound(n, k, sched, cap, window=window)
    if rnd.cap:
        payload = dev.tensor(np.array([r.payload_bytes for r in reqs], np.int64), torch.int64)
        rnd.set_cloud(eng.transfer_time_batch(net, payload, eng.UP),
                      eng.cloud_thresholds(edge, cloud, net, edge_in_flight, cloud_in_flight, k,
                                           rnd.cap))
    rnd.urgency(fleet)
    rnd.admit(fleet)
    out = rnd.outputs()
    order = rnd.full_order().cpu().numpy()
    cloud_ix = [int(i) for i in rnd.cloud().cpu().numpy()]
    skipped = fleet.t["skipped"].cpu().numpy()
    edge_ids = [reqs[i].task_id for i in out.edge_idx.cpu().numpy()]
    in_cloud = set(cloud_ix)
    deferred = [[reqs[i].task_id, int(skipped[i])] for i in order[k:] if int(i) not in in_cloud]
    refetch = sorted(reqs[i].task_id for i in np.nonzero(out.refetch.cpu().numpy())[0])
    return edge_ids, [reqs[i].task_id for i in cloud_ix], deferred, refetch, {
        reqs[i].task_id: int(skipped[i]) for i in range(n)}


@pytest.mark.parametrize("window", [None, 1, 3])
def test_hybrid_round_matches_reference_plans(kb, window):
    """Every reference hybrid plan; windows of 1 and 3 ranks force the
    full-order fallback whenever the scan needs more."""
    bad = []
    for ii, inst in enumerate(golden_io.plan_cloud_instances()):
        states, pending = golden_io.build_objects(inst, kb)
        if not pending:
            continue
        mk = lambda d: None if d is None else kb.EngineProfile(
            tier=d["tier"], capacity=d["capacity"], max_batch=d["max_batch"],
            points=tuple(tuple(p) for p in d["points"]))
        cfg = kb.SchedulerConfig(policy=inst["policy"], buckets=inst["buckets"],
                                 aging_interval=inst["aging_interval"],
                                 stale_threshold=inst["stale_threshold"],
                                 default_exec_estimate=inst["default_exec_estimate"])
        edge, cloud, deferred, refetch, skipped = _hybrid(
            kb, pending, states, mk(inst["edge"]), mk(inst["cloud"]), kb.NetworkModel(**inst["net"]),
            inst["now"], cfg, inst["edge_in_flight"], inst["cloud_in_flight"], window)
        exp = inst["expected"]
        exp_skipped = {r["task_id"]: exp["skipped_after"][r["task_id"]] for r in inst["pending"]}
        if (edge, cloud, deferred, refetch, skipped) != (exp["edge"], exp["cloud"],
                                                          exp["deferred"], exp["refetch"],
                                                          exp_skipped):
            bad.append(ii)
    assert not bad, bad[:5]


@pytest.mark.parametrize("window", [None, 64])
def test_hybrid_round_matches_plan_at_scale(kb, window):
    """A 20k-request synthetic planning round: the fleet-scale hybrid round
    and the object-level plan() (itself pinned to the reference) agree."""
    rng = np.random.default_rng(3)
    n, now = 20_000, 50_000_000
    states, pending = {}, []
    for i in range(n):
        tid = f"t{i:05d}"
        st = kb.TaskState(task_id=tid, t_start=int(rng.integers(0, 10_000_000)),
                          skipped=int(rng.integers(0, 4)))
        t = st.t_start
        es = t
        rounds_ = int(rng.integers(1, 4))
        for j in range(rounds_):
            gs = t + int(rng.integers(0, 200_000))
            ge = gs + int(rng.integers(100_000, 400_000))
            st.begin_generation(j, gs)
            st.finish_generation(j, ge)
            es = ge + int(rng.integers(0, 50_000))
            ee = es + int(rng.integers(300_000, 1_600_000))
            st.record_execution(j, es, ee, 50)
            t = ee - int(rng.integers(0, 300_000))
        states[tid] = st
        issued = min(now - 1, t + int(rng.integers(0, 100_000)))
        pending.append(kb.PendingRequest(
            task_id=tid, round_id=rounds_, issued_at=issued,
            obs_captured_at=issued - int(rng.integers(0, 400_000)),
            last_exec_info=kb.LastExecInfo(es, int(rng.integers(0, 50))),
            payload_bytes=int(rng.choice([100_000, 300_000, 2_000_000])), skipped=0))
    edge = kb.EngineProfile(tier="edge", capacity=2048, max_batch=64,
                            points=((1, 150_000), (64, 400_000)))
    cloud = kb.EngineProfile(tier="cloud", capacity=512, max_batch=128,
                             points=((1, 80_000), (128, 200_000)))
    net = kb.NetworkModel(base_latency_us=20_000, uplink_bps=200_000_000,
                          downlink_bps=1_000_000_000)
    cfg = kb.SchedulerConfig()
    import copy
    states2 = copy.deepcopy(states)
    p = kb.plan(pending, states, edge, cloud, net, now, cfg)
    edge_ids, cloud_ids, deferred, refetch, skipped = _hybrid(
        kb, pending, states2, edge, cloud, net, now, cfg, 0, 0, window)
    assert edge_ids == [r.task_id for r in p.edge]
    assert cloud_ids == [r.task_id for r in p.cloud] and len(cloud_ids) > 0
    assert deferred == [[r.task_id, r.skipped] for r in p.deferred]
    assert refetch == sorted(p.refetch_task_ids)
    assert skipped == {t: s.skipped for t, s in states.items()}


@pytest.mark.parametrize("layout,reserve", [("urgency_first", 10), ("split", 10), ("split", -1)])
def test_hybrid_round_overlapped_equals_sequential(kb, layout, reserve):
    """The bench's overlapped hybrid round (horizons on the main stream, the
    urgency / admission / offload scan with its one 4-byte read on a side
    stream) decides exactly what the sequential round decides, over several
    evolving rounds of a 2^17-robot fleet."""
    from paper_2605_11381_b200 import engines as eng, fleet as fl, rounds, synthetic
    R, k = 1 << 17, 4096
    soa = synthetic.fleet_soa(R, seed=30)
    prev, cand, off = synthetic.chunks(R, seed=31)
    edge = kb.EngineProfile(tier="edge", capacity=k, max_batch=256, points=((1, 150_000), (256, 400_000)))
    cloud = kb.EngineProfile(tier="cloud", capacity=1024, max_batch=512, points=((1, 80_000), (512, 250_000)))
    net = kb.NetworkModel(base_latency_us=20_000, uplink_bps=400_000_000, downlink_bps=1_000_000_000)
    sched = fl.sched_struct("kairos", 10, 5, 150_000, 166_667, synthetic.NOW, 30,
                            int(soa["issued_at"].min()))
    payload = torch.from_numpy(np.random.default_rng(32).choice(
        np.array([100_000, 300_000, 2_000_000], np.int64), R)).cuda()
    inp = rounds.DivergenceInputs(prev, cand, 0.9, offset=off)
    outs = []
    for overlapped in (False, True):
        fleet = fl.DeviceFleet.from_host(soa)
        rnd = rounds.HybridDecisionRound(R, k, sched, cloud.capacity)
        rnd.set_cloud(eng.transfer_time_batch(net, payload, eng.UP),
                      eng.cloud_thresholds(edge, cloud, net, 0, 0, k, rnd.cap))
        seq = []
        for _ in range(3):  # skip counters evolve between rounds
            o = (rnd.run_overlapped(fleet, inp, reserve_sms=reserve, layout=layout) if overlapped
                 else rnd.run(fleet, inp))
            torch.cuda.synchronize()
            seq.append([t.cpu().clone() for t in (o.horizon, o.admitted, o.refetch, o.edge_idx,
                                                 rnd.cloud(), fleet.t["skipped"])])
        outs.append(seq)
    for a, b in zip(*outs):
        for x, y in zip(a, b):
            assert torch.equal(x, y)
    assert outs[0][0][4].numel() > 0  # the cloud tier placed requests
