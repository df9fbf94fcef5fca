"""§8(f) row 2: the simulator's planning loop against the device-resident
incremental ledger.  The reference simulator's own run (five scenarios,
recorded in tests/golden/sim_replay.json by make_golden.py) is replayed:
every TaskState mutation goes through `LedgerStates`, every plan() call must
reproduce the reference decision (edge / cloud / deferred with skip counters /
refetch), and the ledger's running wait totals must equal the oracle's
full-history ledger at every planning instant."""

from __future__ import annotations

import numpy as np
import pytest

import golden_io
from oracle import oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def kb():
    import paper_2605_11381_b200 as kb
    return kb


def _profile(kb, d):
    return None if d is None else kb.EngineProfile(tier=d["tier"], capacity=d["capacity"],
                                                   max_batch=d["max_batch"],
                                                   points=tuple(tuple(p) for p in d["points"]))


def _replay(kb, sc, states, check_waits=False):
    cfg = kb.SchedulerConfig(policy=sc["policy"], buckets=sc["buckets"],
                             aging_interval=sc["aging_interval"],
                             stale_threshold=sc["stale_threshold"],
                             default_exec_estimate=sc["default_exec_estimate"])
    edge, cloud = _profile(kb, sc["edge"]), _profile(kb, sc["cloud"])
    net = None if sc["net"] is None else kb.NetworkModel(**sc["net"])
    shadow = golden_io.replay_log(sc)  # host mirror for the oracle wait totals
    plans = 0
    for e in sc["log"]:
        _, _, host = next(shadow)
        k = e["k"]
        if k == "new":
            states[e["t"]] = kb.TaskState(task_id=e["t"], t_start=e["a"])
        elif k == "bg":
            states[e["t"]].begin_generation(e["j"], e["a"])
        elif k == "fg":
            states[e["t"]].finish_generation(e["j"], e["a"])
            states[e["t"]].accumulated_generation += e["c"]
        elif k == "rx":
            states[e["t"]].record_execution(e["j"], e["a"], e["b"], e.get("h", 1))
        else:
            pending = [kb.PendingRequest(task_id=r["task_id"], round_id=r["round_id"],
                                         issued_at=r["issued_at"],
                                         obs_captured_at=r["obs_captured_at"],
                                         last_exec_info=kb.LastExecInfo(*r["last_exec_info"]),
                                         payload_bytes=r["payload_bytes"], skipped=r["skipped"])
                       for r in e["pending"]]
            d = kb.plan(pending, states, edge, cloud, net, e["now"], cfg,
                        edge_in_flight=e["eif"], cloud_in_flight=e["cif"])
            exp = e["exp"]
            where = (sc["name"], plans)
            assert [r.task_id for r in d.edge] == exp["edge"], where
            assert [r.task_id for r in d.cloud] == exp["cloud"], where
            assert [[r.task_id, r.skipped] for r in d.deferred] == exp["deferred"], where
            assert sorted(d.refetch_task_ids) == exp["refetch"], where
            if check_waits:
                for tid, st in host.items():
                    fleet = orc.fleet_from_objects(
                        [type("R", (), {"task_id": tid, "issued_at": 0, "obs_captured_at": 0,
                                        "skipped": 0, "last_exec_info": type("L", (), {
                                            "remaining_actions": 0})()})()], host)
                    w = orc.total_wait(fleet["slots"], int(fleet["n_exec"][0]),
                                       int(fleet["n_gen"][0]))
                    assert states.ledger.total_wait(tid) == w, (where, tid)
            plans += 1
    return plans


def test_sim_replay_on_device_ledger(kb):
    total = 0
    for sc in golden_io.sim_scenarios():
        total += _replay(kb, sc, kb.LedgerStates())
    assert total > 700


def test_sim_replay_plain_states_matches(kb):
    """The same loop through the object-packing plan() path (plain dict)."""
    sc = golden_io.sim_scenarios()[1]
    assert _replay(kb, sc, {}) > 100


def test_ledger_growth_and_running_waits(kb):
    """Tiny initial capacity (2 tasks x 1 round) forces task and history growth
    mid-run; running totals equal the oracle's full-history ledger at every
    planning instant."""
    for sc in golden_io.sim_scenarios()[:2]:
        _replay(kb, sc, kb.LedgerStates(tasks=2, rounds=1), check_waits=True)


def test_ledger_rejects_out_of_order(kb):
    L = kb.DeviceLedger(tasks=4, rounds=4)
    L.add_task("a", 0)
    L.begin_generation("a", 0, 10)
    L.flush()
    L.record_execution("a", 1, 20, 30)  # round 0 not recorded yet
    with pytest.raises(ValueError, match="out of order"):
        L.flush()
