"""Per-call latency of the object-level plan() (the simulator's call pattern):
    python tools/plan_latency.py            # this package (B200)
    python tools/plan_latency.py --reference  # the reference package (CPU, build container)"""
import json
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

if "--reference" in sys.argv:
    sys.path.insert(0, "/root/reference/pkg/src")
    import roboserve as kb  # noqa: E402
else:
    import paper_2605_11381_b200 as kb  # noqa: E402


def instance(n, seed=0):
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
        pending.append(kb.PendingRequest(task_id=tid, round_id=len(st.exec_intervals), issued_at=issued,
                                         obs_captured_at=issued - int(rng.integers(0, 400_000)),
                                         last_exec_info=kb.LastExecInfo(es, int(rng.integers(0, 50))),
                                         payload_bytes=300_000, skipped=0))
    return states, pending, now


edge = kb.EngineProfile(tier="edge", capacity=64, max_batch=64, points=((1, 150_000), (64, 400_000)))
cfg = kb.SchedulerConfig()
for n in (16, 128, 1024, 8192):
    states, pending, now = instance(n)
    ts = []
    for _ in range(15):
        t0 = time.perf_counter()
        kb.plan(pending, states, edge, None, None, now, cfg)
        ts.append(time.perf_counter() - t0)
    print(json.dumps({"impl": "reference" if "--reference" in sys.argv else "b200", "pending": n,
                      "ms_median": round(1e3 * statistics.median(ts[3:]), 3)}))
