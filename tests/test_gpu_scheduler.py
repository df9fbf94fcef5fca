"""Steps 2-3 on the GPU vs the reference's golden plans, intermediates and the
SPEC / reference-test goldens: bit-exact orders, memberships, waits, ratios."""

from __future__ import annotations

import numpy as np
import pytest
import torch

import golden_io
from oracle import oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def kb():
    import paper_2605_11381_b200 as kb
    return kb


def test_time_golden(kb):
    rows = golden_io.time_rows()
    for row in rows[::5]:
        assert kb.us_from_actions(row["count"], row["hz"]) == row["us"], row
    # batched path, all rows grouped by hz
    by_hz = {}
    for row in rows:
        by_hz.setdefault(row["hz"], []).append(row)
    for hz, rs in by_hz.items():
        c = torch.tensor([r["count"] for r in rs], dtype=torch.int64, device="cuda")
        out = kb.us_from_actions_batch(c, hz).cpu().tolist()
        assert out == [r["us"] for r in rs], hz


@pytest.mark.parametrize("small", [True, False])
def test_plan_golden(kb, small, monkeypatch):
    """Every golden plan through the one-launch small path (kr_plan_small,
    zero-copy staging) and through the general multi-kernel path."""
    from paper_2605_11381_b200 import scheduler
    if not small:
        monkeypatch.setattr(scheduler, "SMALL_PLAN_MAX", 0)
    for ii, inst in enumerate(golden_io.plan_instances()):
        states, pending = golden_io.build_objects(inst, kb)
        edge = kb.EngineProfile(tier="edge", capacity=inst["capacity"], max_batch=1,
                                points=((1, 1000),))
        cfg = kb.SchedulerConfig(policy=inst["policy"], buckets=inst["buckets"],
                                 aging_interval=inst["aging_interval"],
                                 stale_threshold=inst["stale_threshold"],
                                 default_exec_estimate=inst["default_exec_estimate"])
        p = kb.plan(pending, states, edge, None, None, inst["now"], cfg,
                    edge_in_flight=inst["edge_in_flight"])
        exp = inst["expected"]
        assert [r.task_id for r in p.edge] == exp["edge"], ii
        assert [[r.task_id, r.skipped] for r in p.deferred] == exp["deferred"], ii
        assert sorted(p.refetch_task_ids) == exp["refetch"], ii
        assert {t: s.skipped for t, s in states.items()} == exp["skipped_after"], ii
        assert p.cloud == ()


def test_urgency_intermediates_golden(kb):
    from paper_2605_11381_b200 import fleet as fl
    for inst in golden_io.plan_instances()[::3]:
        states, pending = golden_io.build_objects(inst, kb)
        f = fl.DeviceFleet.from_objects(pending, states)
        base = min(r.issued_at for r in pending)
        sched = fl.sched_struct(inst["policy"], inst["buckets"], inst["aging_interval"],
                                inst["stale_threshold"], inst["default_exec_estimate"],
                                inst["now"], inst["control_hz"], base)
        u = fl.urgency(f, sched, intermediates=True)
        for i, r in enumerate(pending):
            it = inst["intermediates"][r.task_id]
            assert int(u.total_wait[i]) == it["total_wait"]
            assert float(u.wr[i]) == it["wr"]
            assert int(u.bucket[i]) == it["bucket"]
            assert int(u.est[i]) == it["est"]
            assert int(u.need_time[i]) == it["need_time"]


def test_waiting_reference_goldens(kb):
    from test_oracle_golden import WAITS
    I = kb.Interval
    for g1, e1, g2, e2, w in WAITS:
        assert kb.round_wait(I(*g1), I(*e1), I(*g2), I(*e2)) == w
    L = kb.WaitLedger.from_waits
    assert kb.wait_ratio(L([200_000, 300_000]), 0, 2_000_000) == 0.25
    assert kb.wait_ratio(L([3_000_000]), 0, 2_500_000) == 1.0
    with pytest.raises(ValueError):
        kb.wait_ratio(L([]), 5, 5)
    st = kb.TaskState(task_id="t", t_start=0)
    for j, (gs, ge, es, ee) in enumerate([(0, 400_000, 400_000, 500_000),
                                          (900_000, 1_300_000, 1_300_000, 1_400_000)]):
        st.begin_generation(j, gs)
        st.finish_generation(j, ge)
        st.record_execution(j, es, ee, 1)
    assert kb.ledger_from_history(st) == kb.WaitLedger((500_000,), 500_000)
    assert kb.current_wait_ratio(st, 2_000_000) == 0.25
    st2 = kb.TaskState(task_id="t", t_start=0)
    st2.begin_generation(0, 0); st2.finish_generation(0, 400_000)
    st2.record_execution(0, 400_000, 500_000, 1)
    st2.begin_generation(1, 650_000)
    assert kb.ledger_from_history(st2).total_wait == 250_000
    assert kb.current_wait_ratio(kb.TaskState(task_id="x", t_start=100), 100) == 0.0


def test_bucket_and_order_spec_goldens(kb):
    cfg = kb.SchedulerConfig()
    assert kb.assign_bucket(0.37, 0, cfg) == 3
    assert kb.assign_bucket(1.0, 0, cfg) == 9
    assert kb.assign_bucket(0.0, 12, cfg) == 2
    with pytest.raises(ValueError):
        kb.assign_bucket(1.5, 0, cfg)
    mk = lambda t, s=0, at=0: kb.PendingRequest(t, 1, at, at, kb.LastExecInfo(0, 0), 0, s)
    assert [r.task_id for r in kb.order_within_bucket([mk("r2"), mk("r1")],
                                                      {"r1": 900_000, "r2": 300_000}, cfg)] == ["r1", "r2"]
    assert [r.task_id for r in kb.order_within_bucket([mk("r2", 0), mk("r1", 2)],
                                                      {"r1": 300_000, "r2": 300_000}, cfg)] == ["r1", "r2"]
    st = kb.TaskState(task_id="t", t_start=0)
    assert kb.estimate_exec_latency(st, 123) == 123
    st.begin_generation(0, 0); st.finish_generation(0, 1); st.record_execution(0, 5, 900_005, 27)
    assert kb.estimate_exec_latency(st, 123) == 900_000


def test_plan_rejects_unknown_and_duplicates(kb):
    cfg = kb.SchedulerConfig()
    mk = lambda t: kb.PendingRequest(t, 0, 0, 0, kb.LastExecInfo(0, 0), 0)
    with pytest.raises(ValueError, match="unknown task"):
        kb.plan([mk("a")], {}, None, None, None, 10, cfg)
    st = {"a": kb.TaskState("a", 0)}
    with pytest.raises(ValueError):
        kb.plan([mk("a"), mk("a")], st, None, None, None, 10, cfg)
    assert kb.plan([], st, None, None, None, 10, cfg).edge == ()


def test_fig4_scenario(kb):
    """pkg/scratch_fig4.py's kairos policy loop (kairos_choose_factory) with the
    drop-in `plan`: identical service orders to the reference's run."""
    g = golden_io.fig4()
    MS = 1000
    for c in g["candidates"]:
        durs = [[d * MS for d in task] for task in c["durs"]]
        gen = c["gen"] * MS
        n = len(durs)
        states = {str(i): kb.TaskState(task_id=str(i), t_start=0) for i in range(n)}
        profile = kb.EngineProfile(tier="edge", capacity=1, max_batch=1, points=((1, gen),))
        cfg = kb.SchedulerConfig(policy="kairos", buckets=10, aging_interval=5,
                                 stale_threshold=10**12, default_exec_estimate=gen)
        rounds_done, ready_at, order, t = [0] * n, [0] * n, [], 0
        total = sum(len(d) for d in durs)
        while len(order) < total:
            ready = [i for i in range(n) if rounds_done[i] < len(durs[i]) and ready_at[i] <= t]
            if not ready:
                t = min(ready_at[i] for i in range(n) if rounds_done[i] < len(durs[i]))
                continue
            pending = [kb.PendingRequest(task_id=str(i), round_id=rounds_done[i],
                                         issued_at=ready_at[i], obs_captured_at=ready_at[i],
                                         last_exec_info=kb.LastExecInfo(0, 0), payload_bytes=0,
                                         skipped=states[str(i)].skipped) for i in ready]
            now = max(t, max(ready_at[i] for i in ready) + 1)
            pick = int(kb.plan(pending, states, profile, None, None, now, cfg).edge[0].task_id)
            j = rounds_done[pick]
            sid = str(pick)
            states[sid].begin_generation(j, t)
            states[sid].finish_generation(j, t + gen)
            states[sid].record_execution(j, t + gen, t + gen + durs[pick][j], 1)
            states[sid].accumulated_generation += gen
            order.append(pick)
            ready_at[pick] = t + gen + durs[pick][j]
            rounds_done[pick] += 1
            t = t + gen
        assert order == c["kairos"], c["durs"]


def test_plan_cloud_golden(kb):
    """Phase 3: plan() with a cloud tier and network model vs the reference."""
    for ii, inst in enumerate(golden_io.plan_cloud_instances()):
        states, pending = golden_io.build_objects(inst, kb)
        mk = lambda d: None if d is None else kb.EngineProfile(
            tier=d["tier"], capacity=d["capacity"], max_batch=d["max_batch"],
            points=tuple(tuple(p) for p in d["points"]))
        net = kb.NetworkModel(**inst["net"])
        cfg = kb.SchedulerConfig(policy=inst["policy"], buckets=inst["buckets"],
                                 aging_interval=inst["aging_interval"],
                                 stale_threshold=inst["stale_threshold"],
                                 default_exec_estimate=inst["default_exec_estimate"])
        p = kb.plan(pending, states, mk(inst["edge"]), mk(inst["cloud"]), net, inst["now"], cfg,
                    edge_in_flight=inst["edge_in_flight"], cloud_in_flight=inst["cloud_in_flight"])
        exp = inst["expected"]
        assert [r.task_id for r in p.edge] == exp["edge"], ii
        assert [r.task_id for r in p.cloud] == exp["cloud"], ii
        assert [[r.task_id, r.skipped] for r in p.deferred] == exp["deferred"], ii
        assert sorted(p.refetch_task_ids) == exp["refetch"], ii
        assert {t: s.skipped for t, s in states.items()} == exp["skipped_after"], ii


def test_engine_reference_goldens(kb):
    prof = kb.EngineProfile(tier="edge", capacity=4, max_batch=4, points=((1, 150_000), (4, 200_000)))
    assert kb.batch_latency(prof, 2) == 166_667
    wan = kb.NetworkModel(base_latency_us=100_000, uplink_bps=10**9, downlink_bps=10**9)
    assert kb.transfer_time(wan, 1_250_000, "up") == 110_000
    assert kb.cloud_round_trip(wan, 300_000, 0, 150_000) == 352_400
    with pytest.raises(kb.ProfileError):
        kb.EngineProfile(tier="edge", capacity=1, max_batch=2, points=((1, 10), (2, 100)))


@pytest.mark.parametrize("n,k,policy", [(1, 1, "kairos"), (7, 3, "kairos"), (33, 0, "fifo"),
                                        (200, 64, "las"), (1000, 64, "kairos"),
                                        (4096, 1024, "kairos"), (2500, 2500, "kairos")])
def test_plan_small_vs_oracle(kb, n, k, policy):
    """kr_plan_small on synthetic fleets vs the oracle's plan (order, refetch,
    skip counters), through the C ABI with the columns in mapped pinned host
    memory: P = next power of two of n (bitonic padding), k = 0 and k = n."""
    import ctypes
    from paper_2605_11381_b200 import _lib, fleet as fl, synthetic
    soa = synthetic.fleet_soa(n, seed=n + k)
    soa["lexrank"] = np.random.default_rng(n).permutation(n).astype(np.int32)
    base = int(soa["issued_at"].min())
    sched = fl.sched_struct(policy, 10, 5, 150_000, 166_667, synthetic.NOW, 30, base)
    pinned = {key: torch.from_numpy(np.ascontiguousarray(v)).pin_memory()
              for key, v in soa.items() if key != "n"}
    fs = fl.DeviceFleet.from_tensors(pinned).c_struct()
    out = torch.empty(3 * n + 1, dtype=torch.int32).pin_memory()
    _lib.check(_lib.load().kr_plan_small(ctypes.byref(fs), ctypes.byref(sched), k,
                                         out.data_ptr(), None), "kr_plan_small")
    torch.cuda.synchronize()
    res = orc.plan_soa(soa, policy, 10, 5, 150_000, 166_667, synthetic.NOW, 30, k)
    o = out.numpy()
    assert np.array_equal(o[:n], res["order"])
    assert np.array_equal(o[n:2 * n], res["refetch"])
    assert np.array_equal(o[2 * n:3 * n], res["skipped_out"])
    assert o[3 * n] == 0
