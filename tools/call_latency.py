"""Per-call latency of the scalar / object-level drop-in API against the
reference on the SAME host: the reference is the unmodified
roboserve vendored under baseline/_ref (tools/vendor_reference.sh), timed in
the same process on one core; ours is this package on the B200.

    python tools/call_latency.py > profiles/r2_call_latency.jsonl

Calls (reference file:line): plan at 4 / 16 / 128 / 1,024 / 8,192 pending
(scheduler.py:254-276, the simulator's call pattern), decide_horizon
(horizon.py:108), round_optimal_horizon (workload.py:471), us_from_actions
(core.py:31), exec_end_from_piggyback (core.py:157), current_wait_ratio
(waiting.py:96).  Median of repeated calls after warm-up."""
import json
import os
import statistics
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "baseline" / "_ref"))
import numpy as np  # noqa: E402

import paper_2605_11381_b200 as ours  # noqa: E402
import roboserve as ref  # noqa: E402

assert Path(ref.__file__).resolve().is_relative_to(ROOT / "baseline" / "_ref")


def instance(kb, n, seed=0):
    rng = np.random.default_rng(seed)
    now = 50_000_000
    states, pending = {}, []
    for i in range(n):
        tid = f"t{i:05d}"
        st = kb.TaskState(task_id=tid, t_start=int(rng.integers(0, 10_000_000)))
        t = es = st.t_start
        for j in range(int(rng.integers(1, 4))):
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
        pending.append(kb.PendingRequest(task_id=tid, round_id=len(st.exec_intervals),
                                         issued_at=issued,
                                         obs_captured_at=issued - int(rng.integers(0, 400_000)),
                                         last_exec_info=kb.LastExecInfo(es, int(rng.integers(0, 50))),
                                         payload_bytes=300_000, skipped=0))
    return states, pending, now


def timed(fn, reps):
    for _ in range(max(3, reps // 10)):
        fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts)


def emit(call, size, t_ref, t_ours):
    print(json.dumps({"call": call, "size": size, "reference_us": round(1e6 * t_ref, 2),
                      "b200_us": round(1e6 * t_ours, 2), "speedup": round(t_ref / t_ours, 2)}),
          flush=True)


def main():
    import torch
    torch.cuda.init()
    print(json.dumps({"host": os.uname().nodename, "cpu_threads": os.cpu_count(),
                      "gpu": torch.cuda.get_device_name(0),
                      "reference": "roboserve (baseline/_ref), one core, same process"}))
    for n in (4, 16, 128, 1024, 8192):
        res = []
        for kb in (ref, ours):
            states, pending, now = instance(kb, n)
            edge = kb.EngineProfile(tier="edge", capacity=64, max_batch=64,
                                    points=((1, 150_000), (64, 400_000)))
            cfg = kb.SchedulerConfig()
            reps = 200 if n <= 128 else (30 if n <= 1024 else 7)
            res.append(timed(lambda: kb.plan(pending, states, edge, None, None, now, cfg), reps))
        emit("plan", n, *res)
    rng = np.random.default_rng(1)
    u = rng.uniform(0.1, 2.0, (6, 50))
    res = []
    for kb in (ref, ours):
        mags = kb.UpdateMagnitudes(u)
        cfg = kb.HorizonPolicyConfig.confidence(0.4, 5)
        res.append(timed(lambda: kb.decide_horizon(cfg, mags), 500))
    emit("decide_horizon", "6x50", *res)
    a = rng.standard_normal((50, 7))
    b = a + 0.2 * rng.standard_normal((50, 7))
    res = [timed(lambda: ref.workload.round_optimal_horizon(a, b, 0.9), 300),
           timed(lambda: ours.round_optimal_horizon(a, b, 0.9), 300)]
    emit("round_optimal_horizon", "50x7", *res)
    res = [timed(lambda: kb.us_from_actions(37, 30), 1000) for kb in (ref, ours)]
    emit("us_from_actions", 1, *res)
    res = []
    for kb in (ref, ours):
        states, pending, now = instance(kb, 1)
        res.append(timed(lambda: kb.exec_end_from_piggyback(pending[0], 30), 1000))
    emit("exec_end_from_piggyback", 1, *res)
    res = []
    for kb in (ref, ours):
        states, pending, now = instance(kb, 1)
        st = states[pending[0].task_id]
        res.append(timed(lambda: kb.current_wait_ratio(st, now), 1000))
    emit("current_wait_ratio", 1, *res)


if __name__ == "__main__":
    main()
