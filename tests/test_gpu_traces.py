"""§8(f) rows 3 + 4 end to end: reference trace files -> native columns ->
device magnitudes -> one kr_horizon_sweep pass per shape -> the exact CSV the
reference's `roboserve pareto` wrote over the same directory."""

from __future__ import annotations

import pytest

import golden_io

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("key", ["default", "custom"])
def test_pareto_matches_reference_cli(key, tmp_path):
    from paper_2605_11381_b200 import traces as tr
    exp = golden_io.traces_expected()["pareto"][key]
    a = exp["args"]
    kw = {}
    for flag, name, cast in (("--static-grid", "static_grid", str),
                             ("--threshold-grid", "threshold_grid", str), ("--h-min", "h_min", int)):
        if flag in a:
            kw[name] = cast(a[a.index(flag) + 1])
    out = tmp_path / "p.csv"
    assert tr.cmd_pareto(golden_io.TRACES_DIR, out, **kw) == 0
    assert out.read_text() == exp["csv"]


def test_pareto_requires_magnitudes(tmp_path):
    from paper_2605_11381_b200 import traces as tr
    traces = tr.load_traces(golden_io.TRACES_DIR / "c_mixed.jsonl")
    r = traces[1].rounds[2]
    stripped = tr.RoundRecord(r.round_id, r.trigger_action_index, r.horizon, r.chunk_size)
    traces[1] = tr.TaskTrace(traces[1].task_id, traces[1].control_hz, traces[1].obs_payload_bytes,
                             traces[1].action_payload_bytes, traces[1].success,
                             traces[1].rounds[:2] + (stripped,) + traces[1].rounds[3:])
    tr.store_traces(traces, tmp_path / "x.jsonl")
    with pytest.raises(ValueError, match=f"trace '{traces[1].task_id}' round 2 has no update"):
        tr.pareto_rows(tmp_path)
