"""Synthetic traces on the device (synth.py / kr_synth.cu vs workload.py:296-456).

RNG bit parity with numpy's Generator is not a goal; parity
is (1) the construction, checked exactly on every generated round: horizons
== the oracle's decide_horizon of the round's magnitudes, trigger placement,
the action budget, the uncertain tail rule u[-1, tail] == bump * mean, and
(2) the distributions, against statistics of 3000-task families the reference
itself generated (tests/golden/synth_stats.json)."""
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


def _setting(kb, s):
    spec = kb.SyntheticSpec(**s["spec"])
    kind, pol_kw = s["policy"]
    pol = (kb.HorizonPolicyConfig.confidence(**pol_kw) if kind == "confidence"
           else kb.HorizonPolicyConfig.static(**pol_kw))
    return spec, pol, s["gen_latency"]


@pytest.mark.parametrize("i", [0, 1, 2])
def test_distribution_matches_reference(kb, i):
    s = golden_io.synth()["settings"][i]
    spec, pol, lat = _setting(kb, s)
    fam = kb.synthesize_family(spec, pol, lat, 3000, seed=5)
    got, ref = golden_io.synth_stats(fam, s["spec"]), s["stats"]
    rel = lambda k: abs(got[k] - ref[k]) / max(abs(ref[k]), 1e-9)
    assert got["tasks"] == ref["tasks"]
    assert rel("rounds_per_task") < 0.03
    assert rel("horizon_mean") < 0.02
    assert abs(got["horizon_std"] - ref["horizon_std"]) < 0.08 * ref["horizon_std"] + 1e-9
    tv = 0.5 * np.abs(np.array(got["horizon_hist"]) - np.array(ref["horizon_hist"])).sum()
    assert tv < 0.04, tv
    assert rel("trigger_mean") < 0.03
    assert rel("tail_mean") < 0.05
    assert rel("u0_mean") < 0.01
    assert abs(got["success_mean"] - ref["success_mean"]) < 0.03


@pytest.mark.parametrize("i", [0, 1, 2])
def test_construction_exact(kb, i):
    s = golden_io.synth()["settings"][i]
    spec, pol, lat = _setting(kb, s)
    fam = kb.synthesize_family(spec, pol, lat, 150, seed=11, with_trajectories=True,
                               trajectory_dim=4)
    slack = kb.generation_slack_actions(lat, spec.control_hz)
    steps = []
    for t in fam:
        assert t.control_hz == spec.control_hz and len(t.rounds) >= 1
        hs = [r.horizon for r in t.rounds]
        assert sum(hs) >= spec.action_budget > sum(hs[:-1])  # workload.py:404, 433
        prev = None
        for j, r in enumerate(t.rounds):
            u = np.asarray(r.update_magnitudes.u)
            assert u.shape == (spec.diffusion_steps, spec.chunk_size)
            assert r.round_id == j and r.chunk_size == spec.chunk_size
            exp_h = (min(pol.static_h, spec.chunk_size) if pol.kind == "static"
                     else orc.decide_horizon_conf(u, pol.threshold, pol.min_horizon))
            assert r.horizon == exp_h
            exp_t = 0 if prev is None else min(max(0, prev - slack), prev - 1)
            assert r.trigger_action_index == exp_t
            prev = r.horizon
            # the uncertain tail is a suffix of columns with u[-1] == bump * mean
            tail = u[-1] == spec.bump_factor * u[:-1].mean(axis=0)
            n = int(tail.sum())
            assert tail[spec.chunk_size - n:].all()
            assert n <= round(min(1.0, 2 * spec.uncertain_fraction) * spec.chunk_size) + 1
            assert np.isfinite(u).all() and (u >= 0).all()
            tr = np.asarray(r.action_trajectory)
            assert tr.shape == (r.horizon, 4)
            steps.append(np.diff(np.vstack([np.zeros((1, 4)), tr]), axis=0))
    st = np.vstack(steps)
    assert abs(st.mean()) < 0.003 and abs(st.std() - 0.05) < 0.003  # normal(0, 0.05) steps


def test_deterministic_and_launch_independent(kb):
    spec, pol = kb.SyntheticSpec(), kb.HorizonPolicyConfig.confidence()
    a = kb.synthesize_family_columns(spec, pol, 100_000, 64, seed=3, rounds_per_launch=8)
    b = kb.synthesize_family_columns(spec, pol, 100_000, 64, seed=3, rounds_per_launch=3)
    c = kb.synthesize_family_columns(spec, pol, 100_000, 64, seed=4)
    for name in ("round_off", "round_id", "trigger_action_index", "horizon", "U", "success"):
        assert torch.equal(getattr(a, name), getattr(b, name)), name
    assert not torch.equal(a.U[:10], c.U[:10])
    one = kb.synthesize_trace(spec, pol, 100_000, seed=3, task_id="solo")
    first = a.to_traces()[0]
    assert one.task_id == "solo" and first.task_id == "task-0000"
    assert [r.horizon for r in one.rounds] == [r.horizon for r in first.rounds]
    assert all(np.array_equal(x.update_magnitudes.u, y.update_magnitudes.u)
               for x, y in zip(one.rounds, first.rounds))


def test_too_slow_generation_raises_reference_message(kb):
    with pytest.raises(ValueError) as e:
        kb.synthesize_trace(kb.SyntheticSpec(), kb.HorizonPolicyConfig.static(2), 100_000, 0)
    assert str(e.value) == golden_io.synth()["too_slow_error"]


def test_traces_round_trip_through_ingest(kb, tmp_path):
    """Device-synthesised traces written with store_traces and read back by the
    native reader are the same traces."""
    fam = kb.synthesize_family(kb.SyntheticSpec(), kb.HorizonPolicyConfig.confidence(), 100_000,
                               20, seed=9, with_trajectories=True)
    p = tmp_path / "synth.jsonl"
    kb.store_traces(fam, p)
    back = kb.load_traces(p)
    assert [kb.trace_to_dict(t) for t in back] == [kb.trace_to_dict(t) for t in fam]


def test_cmd_gen_traces_then_pareto(kb, tmp_path, capsys):
    """gen-traces (cli.py:32-53) on the device, then the pareto sweep over it."""
    import json
    from paper_2605_11381_b200.synth import cmd_gen_traces
    spec = tmp_path / "spec.json"
    spec.write_text(json.dumps({"count": 12, "seed": 4, "gen_latency_us": 100_000,
                                "action_budget": 90}))
    assert cmd_gen_traces(spec, tmp_path / "out", h_min=5) == 0
    assert "wrote 12 traces to" in capsys.readouterr().out
    fam = kb.load_traces(tmp_path / "out" / "traces.jsonl")
    assert len(fam) == 12 and all(sum(r.horizon for r in t.rounds) >= 90 for t in fam)
    with pytest.raises(ValueError, match="--static-h is required"):
        cmd_gen_traces(spec, tmp_path / "o2", policy="static")
    assert kb.traces.cmd_pareto(tmp_path / "out" / "traces.jsonl", tmp_path / "p.csv") == 0
