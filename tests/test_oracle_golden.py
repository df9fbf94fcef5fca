"""Pin the CPU oracle (oracle/) to the reference: every golden vector produced by
running /root/reference itself (tests/golden/make_golden.py) plus the hand-written
goldens of the reference test suite (pkg/tests/*.py) and SPEC.md examples."""

from __future__ import annotations

import math

import numpy as np
import pytest

import golden_io
from oracle import oracle as orc


def test_confidence_golden():
    bad = []
    for i, (u, t, hmin, exp) in enumerate(golden_io.confidence_cases()):
        if orc.decide_horizon_conf(u, t, hmin) != exp:
            bad.append(i)
    assert not bad, f"{len(bad)} confidence mismatches, first {bad[:5]}"


def test_confidence_batch_matches_scalar():
    rng = np.random.default_rng(5)
    U = (rng.uniform(0, 1, (257, 6, 50)) * rng.uniform(0.5, 2, (257, 1, 50))).astype(np.float32)
    U[:, -1, 30:] *= 1.8
    H = orc.horizon_conf_batch(U, 0.4, 5, nthreads=2)
    for r in range(0, 257, 17):
        assert H[r] == orc.decide_horizon_conf(U[r].astype(np.float64), 0.4, 5)


def test_sweep_golden():
    """Reference sweep_thresholds means == the oracle's per-shape sums / len(seq)."""
    for rounds, cfgs, exp in golden_io.sweep_cases():
        totals = np.zeros(len(cfgs), np.int64)
        groups = {}
        for u in rounds:
            groups.setdefault(u.shape, []).append(u)
        for g in groups.values():
            totals += orc.sweep_sums(np.stack(g), cfgs)
        assert [int(t) / len(rounds) for t in totals] == exp


def test_divergence_golden_horizon_and_cosine():
    bad_h, bad_c = [], []
    for i, (ref, cand, thr, exp, cos) in enumerate(golden_io.divergence_cases()):
        if orc.round_optimal_horizon(ref, cand, thr) != exp:
            bad_h.append(i)
        mine = [orc.cosine(cand[j], ref[j]) for j in range(len(cos))]
        if not np.array_equal(np.array(mine, dtype=np.float64), cos):  # bit-exact
            bad_c.append(i)
    assert not bad_h and not bad_c, (bad_h[:5], bad_c[:5])


def test_divergence_golden_haswell_order():
    """The reference's cosines under numpy's OpenBLAS Haswell core (Zen hosts
    run the same kernel): the oracle's Haswell ddot order reproduces every one
    bit-for-bit, and the SkylakeX order does not (the fixture has teeth)."""
    cases = golden_io.divergence_cases("divergence_haswell.npz")
    prev = orc.set_dot_order("haswell")
    try:
        bad_h, bad_c = [], []
        for i, (ref, cand, thr, exp, cos) in enumerate(cases):
            if orc.round_optimal_horizon(ref, cand, thr) != exp:
                bad_h.append(i)
            mine = np.array([orc.cosine(cand[j], ref[j]) for j in range(len(cos))])
            if not np.array_equal(mine, cos):
                bad_c.append(i)
        assert not bad_h and not bad_c, (bad_h[:5], bad_c[:5])
        orc.set_dot_order("skylakex")
        differ = sum(not np.array_equal(
            np.array([orc.cosine(cand[j], ref[j]) for j in range(len(cos))]), cos)
            for ref, cand, thr, exp, cos in cases)
        assert differ > 100
    finally:
        orc.set_dot_order(prev)


def test_divergence_batch_ragged_matches_scalar():
    rng = np.random.default_rng(6)
    R, S, Lp, Lc, D = 40, 3, 20, 16, 7
    prev = rng.normal(size=(R, Lp, D)).astype(np.float32)
    cand = np.repeat(prev[:, None, 2:18], S, axis=1) + rng.normal(0, 0.2, (R, S, Lc, D)).astype(np.float32)
    off = rng.integers(0, 6, R).astype(np.int32)
    lp = rng.integers(5, Lp + 1, R).astype(np.int32)
    lc = rng.integers(0, Lc + 1, R).astype(np.int32)
    H, cos = orc.divergence_batch(prev, cand, 0.9, off, lp, lc, want_cos=True)
    for r in range(R):
        ref = prev[r, off[r]:lp[r]].astype(np.float64)
        hs = [orc.round_optimal_horizon(ref, cand[r, s, :lc[r]].astype(np.float64), 0.9)
              for s in range(S)]
        assert H[r] == min(hs)


def test_time_golden():
    for row in golden_io.time_rows():
        assert orc.us_from_actions(row["count"], row["hz"]) == row["us"], row


# reference tests/test_core.py:31-67 and SPEC.md:69-80
@pytest.mark.parametrize("count,hz,us", [(10, 30, 333_333), (50, 30, 1_666_667), (0, 30, 0),
                                         (0, 7.5, 0), (1, 2, 500_000), (1, 3, 333_333),
                                         (2, 3, 666_667), (30, 30, 1_000_000)])
def test_time_reference_goldens(count, hz, us):
    assert orc.us_from_actions(count, hz) == us


# reference tests/test_waiting.py:20-73 fixtures, as 2-round histories
WAITS = [
    ((1_600_000, 2_000_000), (2_000_000, 2_300_000), (2_500_000, 2_900_000), (2_900_000, 3_200_000), 500_000),
    ((0, 300_000), (300_000, 500_000), (310_000, 610_000), (700_000, 900_000), 10_000),
    ((0, 300_000), (300_000, 600_000), (450_000, 750_000), (750_000, 1_050_000), 150_000),
    ((0, 200_000), (200_000, 400_000), (200_000, 400_000), (999_000, 1_199_000), 0),
    ((0, 200_000), (200_000, 1_100_000), (1_100_000, 1_300_000), (1_300_000, 2_200_000), 200_000),
    ((0, 300_000), (300_000, 1_000_000), (600_000, 900_000), (1_033_333, 1_733_333), 33_333),
    ((0, 100_000), (100_000, 700_000), (200_000, 300_000), (650_000, 1_250_000), 0),
    ((0, 1), (1, 4), (2, 3), (9, 12), 5),
]


@pytest.mark.parametrize("g1,e1,g2,e2,w", WAITS)
def test_round_wait_reference_goldens(g1, e1, g2, e2, w):
    slots = np.array([[*g1, *e1], [*g2, *e2]], np.int64)
    assert orc.total_wait(slots, 2, 2) == w


def test_ledger_in_flight_reference_goldens():
    # tests/test_waiting.py:176-189
    assert orc.total_wait(np.array([[0, 400_000, 400_000, 500_000], [650_000, 0, 0, 0]]), 1, 2) == 250_000
    assert orc.total_wait(np.array([[0, 100_000, 100_000, 900_000], [200_000, 300_000, 0, 0]]), 1, 2) == 0


def test_wait_ratio_and_bucket_reference_goldens():
    assert orc.current_wait_ratio(500_000, 0, 2_000_000) == 0.25       # test_waiting.py:105
    assert orc.current_wait_ratio(3_000_000, 0, 2_500_000) == 1.0      # :109
    assert orc.current_wait_ratio(0, 100, 100) == 0.0                  # :191
    assert orc.assign_bucket(0.37, 0, 10, 5) == 3
    assert orc.assign_bucket(1.0, 0, 10, 5) == 9
    assert orc.assign_bucket(0.0, 12, 10, 5) == 2


def test_plan_golden():
    for ii, inst in enumerate(golden_io.plan_instances()):
        states, pending = golden_io.ns_objects(inst)
        fleet = orc.fleet_from_objects(pending, states)
        avail = max(0, inst["capacity"] - inst["edge_in_flight"])
        res = orc.plan_soa(fleet, inst["policy"], inst["buckets"], inst["aging_interval"],
                           inst["stale_threshold"], inst["default_exec_estimate"], inst["now"],
                           inst["control_hz"], avail)
        ids = [r.task_id for r in pending]
        order = [ids[i] for i in res["order"]]
        exp = inst["expected"]
        n_edge = res["n_edge"]
        assert order[:n_edge] == exp["edge"], ii
        assert [[ids[i], int(res["skipped_out"][i])] for i in res["order"][n_edge:]] == exp["deferred"], ii
        assert sorted(ids[i] for i in np.nonzero(res["refetch"])[0]) == exp["refetch"], ii
        for i, t in enumerate(ids):
            assert res["skipped_out"][i] == exp["skipped_after"][t]
            it = inst["intermediates"][t]
            assert res["total_wait"][i] == it["total_wait"]
            assert res["wr"][i] == it["wr"]          # bit-exact fp64
            assert res["bucket"][i] == it["bucket"]
            assert res["est"][i] == it["est"]
            assert res["need_time"][i] == it["need_time"]


def test_plan_cloud_golden():
    """Phase 3 (hybrid edge / cloud placement) restatement vs the reference."""
    for ii, inst in enumerate(golden_io.plan_cloud_instances()):
        states, pending = golden_io.ns_objects(inst)
        fleet = orc.fleet_from_objects(pending, states)
        payload = [r["payload_bytes"] for r in inst["pending"]]
        res = orc.plan_tiers(fleet, payload, inst["policy"], inst["buckets"], inst["aging_interval"],
                             inst["stale_threshold"], inst["default_exec_estimate"], inst["now"],
                             inst["edge"], inst["cloud"], inst["net"], inst["edge_in_flight"],
                             inst["cloud_in_flight"])
        ids = [r.task_id for r in pending]
        exp = inst["expected"]
        order = [ids[i] for i in res["order"]]
        assert order[:res["n_edge"]] == exp["edge"], ii
        assert [ids[i] for i in res["cloud_order"]] == exp["cloud"], ii
        deferred = [[ids[i], int(res["skipped_out"][i])] for i in res["order"] if res["tier"][i] == 0]
        assert deferred == exp["deferred"], ii
        assert sorted(ids[i] for i in np.nonzero(res["refetch"])[0]) == exp["refetch"], ii
        assert {t: int(res["skipped_out"][i]) for i, t in enumerate(ids)} == exp["skipped_after"], ii


def test_sim_replay_golden():
    """Every plan() decision of five reference simulator runs (edge-only and
    hybrid, kairos / fifo / las, event-driven and fixed-interval planning),
    re-derived by the oracle from the recorded TaskState history."""
    n = 0
    for sc in golden_io.sim_scenarios():
        for kind, e, states in golden_io.replay_log(sc):
            if kind != "plan":
                continue
            pending = golden_io.pending_objects(e)
            fleet = orc.fleet_from_objects(pending, states)
            res = orc.plan_tiers(fleet, [r.payload_bytes for r in pending], sc["policy"],
                                 sc["buckets"], sc["aging_interval"], sc["stale_threshold"],
                                 sc["default_exec_estimate"], e["now"], sc["edge"], sc["cloud"],
                                 sc["net"], e["eif"], e["cif"])
            ids = [r.task_id for r in pending]
            order = [ids[i] for i in res["order"]]
            exp = e["exp"]
            assert order[:res["n_edge"]] == exp["edge"], (sc["name"], n)
            assert [ids[i] for i in res["cloud_order"]] == exp["cloud"], (sc["name"], n)
            deferred = [[ids[i], int(res["skipped_out"][i])] for i in res["order"][res["n_edge"]:]
                        if res["tier"][i] == 0]
            assert deferred == exp["deferred"], (sc["name"], n)
            assert sorted(ids[i] for i in np.nonzero(res["refetch"])[0]) == exp["refetch"]
            n += 1
    assert n > 700


def test_engine_model_goldens():
    # reference tests/test_engines.py: interpolation 166,667; transfer 110,000; round trip 352,400
    prof = {"capacity": 4, "max_batch": 4, "points": [[1, 150_000], [4, 200_000]]}
    assert orc.batch_latency(prof, 2) == 166_667          # test_engines.py:37-39
    assert orc.batch_latency(prof, 4) == 200_000          # test_engines.py:34
    wan = {"base_latency_us": 100_000, "uplink_bps": 10**9, "downlink_bps": 10**9}
    assert orc.transfer_time(wan, 1_250_000, True) == 110_000   # test_engines.py:93
    # cloud_round_trip(WAN, 300_000, 0, 150_000) == 352_400 (test_engines.py:120)
    assert orc.transfer_time(wan, 300_000, True) + 150_000 + orc.transfer_time(wan, 0, False) == 352_400
