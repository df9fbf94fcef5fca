"""The native object packer (_kr_pack, csrc/kr_pack.c) vs a plain-Python
restatement of the fleet layout (host logic, CPU): every column and the CSR
history of reference-shaped TaskState / PendingRequest objects, including
in-flight generations (gen_end None), generation / execution padding, empty
histories, numpy integer fields, and the error behaviour."""

from __future__ import annotations

import numpy as np
import pytest

import paper_2605_11381_b200 as kb
from paper_2605_11381_b200 import fleet as fl


def python_soa(pending, states, rank_of):
    n = len(pending)
    cols = {k: [] for k in fl.INT_FIELDS64 + fl.INT_FIELDS32}
    rows = []
    for req in pending:
        st = states[req.task_id]
        ne, ng = len(st.exec_intervals), len(st.gen_starts)
        for k, v in (("t_start", st.t_start), ("issued_at", req.issued_at),
                     ("obs_captured_at", req.obs_captured_at),
                     ("accum_gen", st.accumulated_generation), ("hist_off", len(rows)),
                     ("remaining", req.last_exec_info.remaining_actions),
                     ("lexrank", rank_of[req.task_id]), ("skipped", req.skipped),
                     ("n_exec", ne), ("n_gen", ng)):
            cols[k].append(v)
        for j in range(max(ne, ng)):
            gs = st.gen_starts[j] if j < ng else 0
            ge = st.gen_ends[j] if j < ng and st.gen_ends[j] is not None else 0
            es, ee = (st.exec_intervals[j].start, st.exec_intervals[j].end) if j < ne else (0, 0)
            rows.append((gs, ge, es, ee))
    out = {k: np.asarray(v, np.int64 if k in fl.INT_FIELDS64 else np.int32)
           for k, v in cols.items()}
    out["slots"] = np.asarray(rows or [(0, 0, 0, 0)], np.int64).reshape(-1, 4)
    out["n"] = n
    return out


def fleet_objects(n, seed):
    rng = np.random.default_rng(seed)
    states, pending = {}, []
    for i in range(n):
        tid = f"task-{i}"
        st = kb.TaskState(task_id=tid, t_start=int(rng.integers(0, 10**7)))
        t = st.t_start
        for j in range(int(rng.integers(0, 5))):
            st.begin_generation(j, t)
            if rng.random() < 0.9 or j < 1:
                st.finish_generation(j, t + int(rng.integers(1, 10**5)))
                st.record_execution(j, t + 10**5, t + 10**5 + int(rng.integers(1, 10**6)), 5)
                t += 2 * 10**6
            else:
                break  # in flight: generation started, not finished, not executed
        if rng.random() < 0.3:
            st.begin_generation(len(st.gen_starts), t + 7)  # in-flight successor
        st.accumulated_generation = int(rng.integers(0, 10**6))
        states[tid] = st
        pending.append(kb.PendingRequest(tid, len(st.exec_intervals), t + 3, t - 5,
                                         kb.LastExecInfo(t, int(rng.integers(0, 50))), 10,
                                         skipped=int(rng.integers(0, 9))))
    return states, pending


@pytest.mark.parametrize("n", [0, 1, 7, 300, 5000])
def test_native_pack_matches_python(n):
    states, pending = fleet_objects(n, seed=n)
    rank = {t: i for i, t in enumerate(sorted(r.task_id for r in pending))}
    got = fl.host_soa(pending, states, rank)
    exp = python_soa(pending, states, rank)
    for k in fl.INT_FIELDS64 + fl.INT_FIELDS32 + ("slots",):
        assert np.array_equal(got[k], exp[k]), k
    assert got["n"] == n


def test_native_pack_numpy_ints_and_errors():
    states, pending = fleet_objects(5, seed=3)
    rank = {t: np.int64(i) for i, t in enumerate(sorted(states))}
    st0 = states[pending[0].task_id]
    st0.t_start = np.int64(st0.t_start)
    exp = python_soa(pending, states, rank)
    got = fl.host_soa(pending, states, rank)
    assert np.array_equal(got["lexrank"], exp["lexrank"])
    assert got["t_start"][0] == int(st0.t_start)
    with pytest.raises(KeyError):
        fl.host_soa(pending, {}, rank)
    with pytest.raises(KeyError):
        fl.host_soa(pending, states, {})
    st0.t_start = "late"
    with pytest.raises(TypeError):
        fl.host_soa(pending, states, rank)
    st0.t_start = 0
    big = {t: 1 << 40 for t in rank}
    with pytest.raises(OverflowError):
        fl.host_soa(pending, states, big)


@pytest.mark.parametrize("n,k,with_cloud", [(1, 1, False), (7, 3, False), (300, 0, False),
                                            (300, 120, True), (2000, 2000, False)])
def test_native_finish_matches_python(n, k, with_cloud):
    """_kr_pack.finish (the plan's result objects from the device read-back)
    equals the plain-Python construction of scheduler.py:223-241: edge prefix,
    deferred bumped copies (offloaded requests excluded), refetch ids, and every
    TaskState.skipped updated."""
    import copy
    from paper_2605_11381_b200 import _kr_pack, scheduler as sch
    states, pending = fleet_objects(n, seed=n + k)
    rng = np.random.default_rng(n)
    order = rng.permutation(n).astype(np.int32)
    refetch = (rng.random(n) < 0.3).astype(np.int32)
    skipped = rng.integers(0, 20, n).astype(np.int32)
    cloud = np.zeros(n, np.int32)
    if with_cloud:
        cloud[order[k:][rng.random(n - k) < 0.2]] = 1
    buf = np.concatenate([order, refetch, skipped])
    a = buf.ctypes.data
    states_py = copy.deepcopy(states)
    before = [r.skipped for r in pending]
    edge, deferred, ref = _kr_pack.finish(pending, states, a, a + 4 * n, a + 8 * n, n, k,
                                          cloud.ctypes.data if with_cloud else 0, sch._bumped)
    exp_edge = tuple(pending[i] for i in order[:k])
    exp_def = tuple(sch._bumped(pending[i], int(skipped[i])) for i in order[k:] if not cloud[i])
    exp_ref = frozenset(pending[i].task_id for i in np.nonzero(refetch)[0])
    for i in order:
        states_py[pending[i].task_id].skipped = int(skipped[i])
    assert edge == exp_edge and all(a_ is b_ for a_, b_ in zip(edge, exp_edge))
    assert deferred == exp_def
    assert all(type(d) is type(e) for d, e in zip(deferred, exp_def))
    assert ref == exp_ref and isinstance(ref, frozenset)
    assert {t: s.skipped for t, s in states.items()} == {t: s.skipped for t, s in states_py.items()}
    # the originals are untouched (bumped copies, not mutation)
    assert [r.skipped for r in pending] == before


def test_native_finish_errors():
    from paper_2605_11381_b200 import _kr_pack, scheduler as sch
    states, pending = fleet_objects(3, seed=1)
    buf = np.array([0, 1, 5, 0, 0, 0, 1, 1, 1], np.int32)  # index 5 out of range
    a = buf.ctypes.data
    with pytest.raises(ValueError):
        _kr_pack.finish(pending, states, a, a + 12, a + 24, 3, 1, 0, sch._bumped)
    del states[pending[0].task_id]
    buf = np.array([0, 1, 2, 0, 0, 0, 1, 1, 1], np.int32)
    a = buf.ctypes.data
    with pytest.raises(KeyError):
        _kr_pack.finish(pending, states, a, a + 12, a + 24, 3, 1, 0, sch._bumped)
