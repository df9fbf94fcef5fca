"""The full decision round (rounds.DecisionRound: divergence horizon + urgency +
top-k admission) on a synthetic fleet vs the CPU oracle, bit-exact."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import oracle as orc

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("R,k,S,D", [(1 << 15, 1024, 1, 7), (5000, 64, 8, 7), (3000, 300, 1, 32),
                                     (777, 777, 1, 7), (1000, 0, 1, 7), (1024, 64, 1, 7),
                                     (4096, 4000, 1, 7)])
def test_decision_round_vs_oracle(R, k, S, D):
    from paper_2605_11381_b200 import fleet as fl, rounds, synthetic
    soa = synthetic.fleet_soa(R, seed=R + k)
    prev, cand, off = synthetic.chunks(R, seed=R, S=S, D=D, Lp=50 if D == 7 else 64,
                                       Lc=50 if D == 7 else 64)
    fleet = fl.DeviceFleet.from_host(soa)
    base = int(soa["issued_at"].min())
    sched = fl.sched_struct("kairos", 10, 5, 150_000, 166_667, synthetic.NOW, 30, base)
    rnd = rounds.DecisionRound(R, k, sched)
    out = rnd.run(fleet, rounds.DivergenceInputs(prev, cand, 0.9, offset=off))
    torch.cuda.synchronize()
    # step 1
    H = orc.divergence_batch(prev.cpu().numpy(), cand.cpu().numpy(), 0.9, off.cpu().numpy())
    assert np.array_equal(out.horizon.cpu().numpy(), H)
    # steps 2-3
    res = orc.plan_soa(soa, "kairos", 10, 5, 150_000, 166_667, synthetic.NOW, 30, k)
    assert np.array_equal(out.need_time.cpu().numpy(), res["need_time"])
    assert np.array_equal(out.admitted.cpu().numpy(), res["admitted"])
    assert np.array_equal(out.refetch.cpu().numpy(), res["refetch"])
    assert np.array_equal(fleet.t["skipped"].cpu().numpy(), res["skipped_out"])
    if k:
        assert np.array_equal(out.edge_idx.cpu().numpy(), res["order"][:k])


@pytest.mark.parametrize("policy", ["fifo", "las"])
def test_round_baseline_policies(policy):
    from paper_2605_11381_b200 import fleet as fl, rounds, synthetic
    R, k = 4000, 333
    soa = synthetic.fleet_soa(R, seed=9)
    fleet = fl.DeviceFleet.from_host(soa)
    sched = fl.sched_struct(policy, 10, 5, 150_000, 166_667, synthetic.NOW, 30,
                            int(soa["issued_at"].min()))
    rnd = rounds.DecisionRound(R, k, sched)
    rnd.urgency(fleet)
    rnd.admit(fleet)
    res = orc.plan_soa(soa, policy, 10, 5, 150_000, 166_667, synthetic.NOW, 30, k)
    assert np.array_equal(rnd.edge_idx.cpu().numpy(), res["order"][:k])
    assert np.array_equal(rnd.admitted.cpu().numpy(), res["admitted"])


def test_graph_replay_matches_eager():
    from paper_2605_11381_b200 import fleet as fl, rounds, synthetic
    R, k = 20000, 512
    soa = synthetic.fleet_soa(R, seed=4)
    prev, cand, off = synthetic.chunks(R, seed=5)
    sched = fl.sched_struct("kairos", 10, 5, 150_000, 166_667, synthetic.NOW, 30,
                            int(soa["issued_at"].min()))
    f1 = fl.DeviceFleet.from_host(soa)
    r1 = rounds.DecisionRound(R, k, sched)
    o1 = r1.run(f1, rounds.DivergenceInputs(prev, cand, 0.9, offset=off))
    eager = [t.clone() for t in (o1.horizon, o1.need_time, o1.admitted, o1.refetch, o1.edge_idx)]
    skip_after_one = f1.t["skipped"].clone()
    f2 = fl.DeviceFleet.from_host(soa)
    r2 = rounds.DecisionRound(R, k, sched)
    r2.capture(f2, rounds.DivergenceInputs(prev, cand, 0.9, offset=off))  # runs one round
    f2.t["skipped"].copy_(torch.from_numpy(soa["skipped"]).cuda())
    o2 = r2.replay()
    torch.cuda.synchronize()
    for a, b in zip(eager, (o2.horizon, o2.need_time, o2.admitted, o2.refetch, o2.edge_idx)):
        assert torch.equal(a, b)
    assert torch.equal(skip_after_one, f2.t["skipped"])


@pytest.mark.parametrize("R,k,rounds_", [(1 << 16, 8192, 60), (1 << 14, 5000, 30)])
def test_multi_round_replay_vs_oracle(R, k, rounds_):
    """Successive decision rounds on one fleet: skip counters evolve (aging
    drives most robots into the top bucket with tied aged estimates, so the
    admitted set concentrates in few large bins).  Every round must match the
    oracle's plan() on the same evolving state."""
    from paper_2605_11381_b200 import fleet as fl, rounds, synthetic
    soa = synthetic.fleet_soa(R, seed=77)
    fleet = fl.DeviceFleet.from_host(soa)
    sched = fl.sched_struct("kairos", 10, 5, 150_000, 166_667, synthetic.NOW, 30,
                            int(soa["issued_at"].min()))
    rnd = rounds.DecisionRound(R, k, sched)
    for r in range(rounds_):
        rnd.urgency(fleet)
        rnd.admit(fleet)
        res = orc.plan_soa(soa, "kairos", 10, 5, 150_000, 166_667, synthetic.NOW, 30, k)
        torch.cuda.synchronize()
        assert np.array_equal(rnd.edge_idx.cpu().numpy(), res["order"][:k]), r
        assert np.array_equal(rnd.admitted.cpu().numpy(), res["admitted"]), r
        assert np.array_equal(fleet.t["skipped"].cpu().numpy(), res["skipped_out"]), r
        soa["skipped"] = res["skipped_out"]


@pytest.mark.parametrize("layout,reserve", [("split", 16), ("urgency_first", 12)])
def test_concurrent_replay_matches_eager(layout, reserve):
    """Urgency + admission (or admission after a whole-GPU urgency pass) on a
    side stream over reserved SMs, concurrent with the horizon kernel:
    identical outputs to the sequential eager round."""
    from paper_2605_11381_b200 import fleet as fl, rounds, synthetic
    R, k = 1 << 17, 2048
    soa = synthetic.fleet_soa(R, seed=8)
    prev, cand, off = synthetic.chunks(R, seed=9)
    sched = fl.sched_struct("kairos", 10, 5, 150_000, 166_667, synthetic.NOW, 30,
                            int(soa["issued_at"].min()))
    f1 = fl.DeviceFleet.from_host(soa)
    r1 = rounds.DecisionRound(R, k, sched)
    o1 = r1.run(f1, rounds.DivergenceInputs(prev, cand, 0.9, offset=off))
    eager = [t.clone() for t in (o1.horizon, o1.need_time, o1.admitted, o1.refetch, o1.edge_idx)]
    f2 = fl.DeviceFleet.from_host(soa)
    r2 = rounds.DecisionRound(R, k, sched)
    r2.capture(f2, rounds.DivergenceInputs(prev, cand, 0.9, offset=off), reserve_sms=reserve,
               layout=layout)
    f2.t["skipped"].copy_(torch.from_numpy(soa["skipped"]).cuda())
    o2 = r2.replay()
    torch.cuda.synchronize()
    for a, b in zip(eager, (o2.horizon, o2.need_time, o2.admitted, o2.refetch, o2.edge_idx)):
        assert torch.equal(a, b)


@pytest.mark.parametrize("storage", [torch.float32, torch.float64])
def test_confidence_round_vs_oracle(storage):
    """A decision round with the confidence-threshold policy (update
    magnitudes) instead of the divergence horizon, eager and as the captured
    urgency-first concurrent graphs."""
    from paper_2605_11381_b200 import HorizonPolicyConfig, fleet as fl, rounds, synthetic
    R, k = 1 << 16, 1024
    soa = synthetic.fleet_soa(R, seed=31)
    U = synthetic.magnitudes(R, seed=32, dtype=storage)
    cfg = HorizonPolicyConfig.confidence(0.4, 5)
    sched = fl.sched_struct("kairos", 10, 5, 150_000, 166_667, synthetic.NOW, 30,
                            int(soa["issued_at"].min()))
    H = orc.horizon_conf_batch(U.cpu().numpy(), 0.4, 5)
    res = orc.plan_soa(soa, "kairos", 10, 5, 150_000, 166_667, synthetic.NOW, 30, k)
    for graph in (False, True):
        fleet = fl.DeviceFleet.from_host(soa)
        rnd = rounds.DecisionRound(R, k, sched)
        inp = rounds.ConfidenceInputs(U, cfg)
        if graph:
            rnd.capture(fleet, inp, reserve_sms=12, layout="urgency_first")
            fleet.t["skipped"].copy_(torch.from_numpy(soa["skipped"]).cuda())
            out = rnd.replay()
        else:
            out = rnd.run(fleet, inp)
        torch.cuda.synchronize()
        assert np.array_equal(out.horizon.cpu().numpy(), H)
        assert np.array_equal(out.edge_idx.cpu().numpy(), res["order"][:k])
        assert np.array_equal(fleet.t["skipped"].cpu().numpy(), res["skipped_out"])


def test_mixed_fleet_round_vs_oracle():
    """configs[2]-style heterogeneous fleet: arms (64x7 divergence), humanoids
    (64x32 divergence) and a confidence-policy group in one round, the groups'
    horizon kernels on forked streams; eager and captured."""
    from paper_2605_11381_b200 import HorizonPolicyConfig, fleet as fl, rounds, synthetic
    na, nh, nc, k = 3000, 2000, 1500, 700
    R = na + nh + nc
    soa = synthetic.fleet_soa(R, seed=41)
    pa, ca, oa = synthetic.chunks(na, seed=42, Lp=64, Lc=64, D=7)
    ph, chh, oh = synthetic.chunks(nh, seed=43, Lp=64, Lc=64, D=32)
    U = synthetic.magnitudes(nc, seed=44)
    inp = rounds.MixedInputs([(0, rounds.DivergenceInputs(pa, ca, 0.9, offset=oa)),
                              (na, rounds.DivergenceInputs(ph, chh, 0.9, offset=oh)),
                              (na + nh, rounds.ConfidenceInputs(U, HorizonPolicyConfig.confidence(0.4, 5)))])
    H = np.concatenate([
        orc.divergence_batch(pa.cpu().numpy(), ca.cpu().numpy(), 0.9, oa.cpu().numpy()),
        orc.divergence_batch(ph.cpu().numpy(), chh.cpu().numpy(), 0.9, oh.cpu().numpy()),
        orc.horizon_conf_batch(U.cpu().numpy(), 0.4, 5)])
    sched = fl.sched_struct("kairos", 10, 5, 150_000, 166_667, synthetic.NOW, 30,
                            int(soa["issued_at"].min()))
    res = orc.plan_soa(soa, "kairos", 10, 5, 150_000, 166_667, synthetic.NOW, 30, k)
    for graph in (False, True):
        fleet = fl.DeviceFleet.from_host(soa)
        rnd = rounds.DecisionRound(R, k, sched)
        if graph:
            rnd.capture(fleet, inp, reserve_sms=12, layout="urgency_first")
            fleet.t["skipped"].copy_(torch.from_numpy(soa["skipped"]).cuda())
            out = rnd.replay()
        else:
            out = rnd.run(fleet, inp)
        torch.cuda.synchronize()
        assert np.array_equal(out.horizon.cpu().numpy(), H)
        assert np.array_equal(out.edge_idx.cpu().numpy(), res["order"][:k])


def test_round_flags_raise_out_of_range_keys():
    """A fleet round keeps the urgency pass's validation word: a request whose
    issue time lies >= 2^40 µs after the packed key's base cannot be keyed
    exactly (plan() raises there), so check() raises the same ValueError;
    an in-range round leaves the word clear.  Also: a hybrid round's kth
    output is the k-th key of its ordered candidates."""
    from paper_2605_11381_b200 import fleet as fl, rounds, synthetic
    R, k = 5000, 100
    soa = synthetic.fleet_soa(R, seed=61)
    good = fl.sched_struct("kairos", 10, 5, 150_000, 166_667, synthetic.NOW, 30,
                           int(soa["issued_at"].min()))
    rnd = rounds.DecisionRound(R, k, good)
    out = rnd.run(rounds_fleet := fl.DeviceFleet.from_host(soa),
                  rounds.DivergenceInputs(*synthetic.chunks(R, seed=62)[:2], 0.9))
    rnd.check()
    assert int(out.flags.item()) == 0
    bad = fl.sched_struct("kairos", 10, 5, 150_000, 166_667, synthetic.NOW, 30,
                          int(soa["issued_at"].min()) - (1 << 41))
    rnd2 = rounds.DecisionRound(R, k, bad)
    rnd2.urgency(rounds_fleet)
    rnd2.admit(rounds_fleet)
    with pytest.raises(ValueError, match="packed sort-key range"):
        rnd2.check()
    rnd2.check()  # reset after raising
    hyb = rounds.HybridDecisionRound(R, k, good, cloud_cap=0)
    hyb.urgency(rounds_fleet)
    hyb.admit(rounds_fleet)
    o = hyb.outputs()
    assert torch.equal(o.kth[0], o.edge_keys[k - 1])


@pytest.mark.parametrize("policy", ["kairos", "fifo", "las"])
def test_prepared_select_equals_separate_reset(policy):
    """kr_urgency_prep + kr_select_admit_prepared (the urgency pass's last CTA
    prepares the select state and restores the statistics) decide exactly what
    kr_urgency + kr_select_admit decide, over evolving rounds, eager and
    graph-captured, and match the oracle."""
    from paper_2605_11381_b200 import fleet as fl, rounds, synthetic
    R, k = 1 << 17, 3000
    soa = synthetic.fleet_soa(R, seed=41)
    prev, cand, off = synthetic.chunks(R, seed=42)
    sched = fl.sched_struct(policy, 10, 5, 150_000, 166_667, synthetic.NOW, 30,
                            int(soa["issued_at"].min()))
    inp = rounds.DivergenceInputs(prev, cand, 0.9, offset=off)
    runs = []
    for prepared, graph in ((False, False), (True, False), (True, True)):
        fleet = fl.DeviceFleet.from_host(soa)
        rnd = rounds.DecisionRound(R, k, sched)
        assert rnd.prepared
        rnd.prepared = prepared
        if graph:
            rnd.capture(fleet, inp, reserve_sms=8)  # runs one round
            fleet.t["skipped"].copy_(torch.from_numpy(soa["skipped"]).cuda())
        seq = []
        for _ in range(3):
            o = rnd.replay() if graph else rnd.run(fleet, inp)
            torch.cuda.synchronize()
            seq.append([t.cpu().clone() for t in (o.keys, o.admitted, o.refetch, o.edge_idx,
                                                 o.edge_keys, o.kth, fleet.t["skipped"])])
        rnd.check()
        runs.append(seq)
    for other in runs[1:]:
        for a, b in zip(runs[0], other):
            for x, y in zip(a, b):
                assert torch.equal(x, y)
    res = orc.plan_soa(soa, policy, 10, 5, 150_000, 166_667, synthetic.NOW, 30, k)
    assert np.array_equal(runs[1][0][3].numpy(), res["order"][:k])
    assert np.array_equal(runs[1][0][1].numpy(), res["admitted"])
