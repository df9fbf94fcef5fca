"""Loaders for the reference-generated fixtures in tests/golden/ (see make_golden.py)."""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


def confidence_cases():
    z = np.load(GOLDEN / "horizon_confidence.npz")
    out = []
    for i, (k, n) in enumerate(z["shapes"]):
        u = z["u"][z["offsets"][i]:z["offsets"][i + 1]].reshape(k, n)
        out.append((u, float(z["threshold"][i]), int(z["min_horizon"][i]), int(z["expected"][i])))
    return out


def sweep_cases():
    """[(rounds: list of [K,N] arrays, configs: list of (kind, static_h, threshold,
    min_horizon), expected means)] -- kind 1 = confidence, 0 = static."""
    z = np.load(GOLDEN / "sweep.npz")
    out = []
    for i in range(len(z["seq_off"]) - 1):
        rounds = []
        for j in range(z["seq_off"][i], z["seq_off"][i + 1]):
            k, n = z["shapes"][j]
            rounds.append(z["u"][z["offsets"][j]:z["offsets"][j + 1]].reshape(k, n))
        lo, hi = z["cfg_off"][i], z["cfg_off"][i + 1]
        cfgs = [(int(z["kind"][c]), int(z["static_h"][c]), float(z["threshold"][c]),
                 int(z["min_horizon"][c])) for c in range(lo, hi)]
        out.append((rounds, cfgs, [float(x) for x in z["expected"][lo:hi]]))
    return out


def divergence_cases(name: str = "divergence.npz"):
    """divergence.npz: cosines from numpy's OpenBLAS SkylakeX core (this host);
    divergence_haswell.npz: the same reference run under its Haswell core."""
    z = np.load(GOLDEN / name)
    out = []
    for i in range(len(z["thr"])):
        ref = z["ref"][z["ref_off"][i]:z["ref_off"][i + 1]].reshape(z["ref_shapes"][i])
        cand = z["cand"][z["cand_off"][i]:z["cand_off"][i + 1]].reshape(z["cand_shapes"][i])
        cos = z["cos"][z["cos_off"][i]:z["cos_off"][i + 1]]
        out.append((ref, cand, float(z["thr"][i]), int(z["expected"][i]), cos))
    return out


def time_rows():
    return json.loads((GOLDEN / "time.json").read_text())


def plan_instances():
    return json.loads((GOLDEN / "plan.json").read_text())


def fig4():
    return json.loads((GOLDEN / "fig4.json").read_text())


def build_objects(inst, mod):
    """Rebuild TaskState / PendingRequest objects of module `mod` (any package
    exposing the reference's core types) from a plan fixture."""
    states = {}
    for s in inst["states"]:
        st = mod.TaskState(task_id=s["task_id"], t_start=s["t_start"], skipped=s["skipped"],
                           accumulated_generation=s["accumulated_generation"])
        for j, gs in enumerate(s["gen_starts"]):
            st.begin_generation(j, gs)
            if s["gen_ends"][j] is not None:
                st.finish_generation(j, s["gen_ends"][j])
        for j, (es, ee) in enumerate(s["exec_intervals"]):
            st.record_execution(j, es, ee, s["horizons"][j])
        states[st.task_id] = st
    pending = [mod.PendingRequest(task_id=r["task_id"], round_id=r["round_id"],
                                  issued_at=r["issued_at"], obs_captured_at=r["obs_captured_at"],
                                  last_exec_info=mod.LastExecInfo(*r["last_exec_info"]),
                                  payload_bytes=r["payload_bytes"], skipped=r["skipped"])
               for r in inst["pending"]]
    return states, pending


def ns_objects(inst):
    """Duck-typed stand-ins (SimpleNamespace) for the fixture's states / requests."""
    from types import SimpleNamespace as NS
    states = {}
    for s in inst["states"]:
        states[s["task_id"]] = NS(
            task_id=s["task_id"], t_start=s["t_start"], skipped=s["skipped"],
            accumulated_generation=s["accumulated_generation"],
            gen_starts=list(s["gen_starts"]), gen_ends=list(s["gen_ends"]),
            exec_intervals=[NS(start=a, end=b) for a, b in s["exec_intervals"]])
    pending = [NS(task_id=r["task_id"], issued_at=r["issued_at"],
                  obs_captured_at=r["obs_captured_at"], skipped=r["skipped"],
                  last_exec_info=NS(exec_start=r["last_exec_info"][0],
                                    remaining_actions=r["last_exec_info"][1]))
               for r in inst["pending"]]
    return states, pending


def plan_cloud_instances():
    return json.loads((GOLDEN / "plan_cloud.json").read_text())


def sim_scenarios():
    return json.loads((GOLDEN / "sim_replay.json").read_text())


def replay_log(scenario):
    """Walk a recorded simulator log: yields ("event", entry) for every
    TaskState mutation and ("plan", entry, states) at each plan() call, with
    `states` the duck-typed task states (SimpleNamespace) as of that call."""
    from types import SimpleNamespace as NS
    states = {}
    for e in scenario["log"]:
        k = e["k"]
        if k == "plan":
            yield "plan", e, states
            continue
        if k == "new":
            states[e["t"]] = NS(task_id=e["t"], t_start=e["a"], skipped=0,
                                accumulated_generation=0, gen_starts=[], gen_ends=[],
                                exec_intervals=[])
        else:
            st = states[e["t"]]
            if k == "bg":
                st.gen_starts.append(e["a"])
                st.gen_ends.append(None)
            elif k == "fg":
                st.gen_ends[e["j"]] = e["a"]
                st.accumulated_generation += e["c"]
            elif k == "rx":
                st.exec_intervals.append(NS(start=e["a"], end=e["b"]))
        yield "event", e, states


def pending_objects(entry):
    from types import SimpleNamespace as NS
    return [NS(task_id=r["task_id"], round_id=r["round_id"], issued_at=r["issued_at"],
               obs_captured_at=r["obs_captured_at"], payload_bytes=r["payload_bytes"],
               skipped=r["skipped"],
               last_exec_info=NS(exec_start=r["last_exec_info"][0],
                                 remaining_actions=r["last_exec_info"][1]))
            for r in entry["pending"]]


TRACES_DIR = GOLDEN / "traces"


def traces_expected():
    return json.loads((GOLDEN / "traces_expected.json").read_text())


def synth():
    return json.loads((GOLDEN / "synth_stats.json").read_text())


def synth_stats(traces, spec_kw) -> dict:
    """Distribution summary of a trace family (computed the same way for the
    reference in make_golden.py and for the device synthesis in
    tests/test_gpu_synth.py)."""
    N = spec_kw.get("chunk_size", 50)
    bump = spec_kw.get("bump_factor", 1.8)
    hs, trig, nunc, u0, rpt = [], [], [], [], []
    for t in traces:
        rpt.append(len(t.rounds))
        for r in t.rounds:
            hs.append(r.horizon)
            trig.append(r.trigger_action_index)
            u = np.asarray(r.update_magnitudes.u)
            nunc.append(int((u[-1] == bump * u[:-1].mean(axis=0)).sum()))
            u0.append(float(u[0].mean()))
    hist = np.bincount(np.array(hs), minlength=N + 1)
    return {"tasks": len(traces), "rounds": len(hs), "rounds_per_task": float(np.mean(rpt)),
            "horizon_mean": float(np.mean(hs)), "horizon_std": float(np.std(hs)),
            "horizon_hist": (hist / hist.sum()).tolist(), "trigger_mean": float(np.mean(trig)),
            "tail_mean": float(np.mean(nunc)), "u0_mean": float(np.mean(u0)),
            "success_mean": float(np.mean([t.success for t in traces]))}
