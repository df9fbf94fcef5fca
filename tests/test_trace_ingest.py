"""§8(f) row 4 host side: the native JSONL trace reader (kr_trace_parse) vs
trace files written by the reference's store_traces and the reference
load_traces' TraceFormatError fields on malformed variants (CPU only: the
reader is host code; the Pareto sweep over its columns is in
test_gpu_traces.py)."""

from __future__ import annotations

import json

import numpy as np
import pytest

import golden_io
from paper_2605_11381_b200 import traces as tr


def _ref_dicts(path):
    return [json.loads(line) for line in path.read_text().splitlines() if line.strip()]


@pytest.mark.parametrize("name", ["a_arms.jsonl", "b_humanoid.jsonl", "c_mixed.jsonl"])
def test_load_matches_reference_files(name):
    path = golden_io.TRACES_DIR / name
    loaded = tr.load_traces(path)
    assert [tr.trace_to_dict(t) for t in loaded] == _ref_dicts(path)


def test_trace_dir_columns():
    cols = tr.load_trace_columns(golden_io.TRACES_DIR)
    ref = [d for f in sorted(golden_io.TRACES_DIR.glob("*.jsonl")) for d in _ref_dicts(f)]
    assert cols.task_ids == [d["task_id"] for d in ref]
    rounds = [r for d in ref for r in d["rounds"]]
    assert cols.n_rounds == len(rounds)
    assert cols.horizon.tolist() == [r["horizon"] for r in rounds]
    assert cols.trigger_action_index.tolist() == [r["trigger_action_index"] for r in rounds]
    groups = cols.magnitude_groups()
    assert sum(len(idx) for idx, _ in groups.values()) == len(rounds)
    for (K, N), (idx, U) in groups.items():
        for j, r in zip(idx, U):
            assert np.array_equal(r, np.asarray(rounds[j]["update_magnitudes"]))
    # trajectories (ragged-capable rows) survive exactly
    for r_i, r in enumerate(rounds):
        if r["action_trajectory"] is None:
            assert cols.traj_rows[r_i] == -1
        else:
            rows = [cols.traj[cols.traj_off[k]:cols.traj_off[k + 1]].tolist()
                    for k in range(cols.traj_row0[r_i], cols.traj_row0[r_i] + cols.traj_rows[r_i])]
            assert rows == r["action_trajectory"]


@pytest.mark.parametrize("case", golden_io.traces_expected()["cases"], ids=lambda c: c["name"])
def test_validation_matches_reference(case):
    if "ok" in case:
        assert [tr.trace_to_dict(t) for t in tr._objects(tr.parse_jsonl(case["text"]))] == case["ok"]
        return
    with pytest.raises(tr.TraceFormatError) as info:
        tr.parse_jsonl(case["text"])
    e = info.value
    assert str(e) == case["error"]
    assert (e.line, e.task_id, e.round_id, e.raw_message) == (
        case["line"], case["task_id"], case["round_id"], case["raw"])


def test_reference_suite_validation_cases():
    """reference tests/test_workload.py:72-123 against trace_from_dict."""
    base = tr.trace_to_dict(tr.load_traces(golden_io.TRACES_DIR / "a_arms.jsonl")[0])
    d = json.loads(json.dumps(base))
    d["rounds"][1]["trigger_action_index"] = d["rounds"][0]["horizon"]
    with pytest.raises(tr.TraceFormatError, match="round 1") as info:
        tr.trace_from_dict(d, line=7)
    assert (info.value.round_id, info.value.task_id, info.value.line) == (1, base["task_id"], 7)
    d = json.loads(json.dumps(base))
    del d["control_hz"]
    with pytest.raises(tr.TraceFormatError, match="control_hz"):
        tr.trace_from_dict(d)


def test_empty_and_roundtrip(tmp_path):
    p = tmp_path / "empty.jsonl"
    p.write_text("")
    assert tr.load_traces(p) == []
    traces = tr.load_traces(golden_io.TRACES_DIR / "c_mixed.jsonl")
    q = tmp_path / "rt.jsonl"
    tr.store_traces(traces, q)
    assert q.read_text() == (golden_io.TRACES_DIR / "c_mixed.jsonl").read_text()


def test_multithreaded_parse_order_and_first_error():
    """A multi-MB buffer is split across host threads: traces come back in file
    order, line numbers count across the cuts, and the earliest bad line wins."""
    lines = [l for f in sorted(golden_io.TRACES_DIR.glob("*.jsonl"))
             for l in f.read_text().splitlines() if l.strip()]
    body = []
    for i in range(400):
        d = json.loads(lines[i % len(lines)])
        d["task_id"] = f"task-{i:05d}"
        body.append(json.dumps(d, separators=(",", ":")))
        if i % 7 == 0:
            body.append("   ")  # blank lines still count
    text = "\n".join(body) + "\n"
    assert len(text) > 4 << 20
    cols = tr.parse_jsonl(text)
    assert cols.task_ids == [f"task-{i:05d}" for i in range(400)]
    assert [tr.trace_to_dict(t) for t in tr._objects(cols)] == \
        [json.loads(b) for b in body if b.strip()]
    # two bad lines in different thirds of the file: the first one is reported
    bad = list(body)
    i1, i2 = len(bad) // 3 + 5, 2 * len(bad) // 3
    bad[i2] = "{broken"
    bad[i1] = bad[i1].replace('"horizon":', '"horizon":0,"x":', 1)
    d1 = json.loads(bad[i1])
    with pytest.raises(tr.TraceFormatError) as info:
        tr.parse_jsonl("\n".join(bad) + "\n")
    assert info.value.line == i1 + 1
    assert info.value.task_id == d1["task_id"]
