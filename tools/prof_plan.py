"""Where the time of one small plan() call goes (the simulator's call sizes):
    python tools/prof_plan.py [n ...]
Times each host step of scheduler.plan's one-launch path separately (median
of 300 calls) and the whole call."""
import ctypes
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import call_latency as cl  # noqa: E402
from paper_2605_11381_b200 import _lib, fleet as fl, scheduler as sc  # noqa: E402

kb = cl.ours


def med(fn, reps=300):
    for _ in range(20):
        fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return 1e6 * statistics.median(ts)


for n in [int(a) for a in sys.argv[1:]] or [4, 16, 128]:
    states, pending, now = cl.instance(kb, n)
    edge = kb.EngineProfile(tier="edge", capacity=64, max_batch=64, points=((1, 150_000), (64, 400_000)))
    cfg = kb.SchedulerConfig()
    reqs = sc._checked_pending(pending, states)
    rank = sc._ranks([r.task_id for r in reqs])
    sched = _lib.KrSched(0, 10, 5, 0, 150_000, 166_667, now, 1, 1,
                         int(min(r.issued_at for r in reqs)))
    lib = _lib.load()
    fs, out, d = fl.pack_mapped(reqs, states, rank, 4 * (3 * n + 1))
    st = torch.cuda.current_stream()

    def launch_sync():
        lib.kr_plan_small(ctypes.byref(fs), ctypes.byref(sched), min(64, n), d, st.cuda_stream)
        st.synchronize()

    parts = {
        "whole plan()": lambda: kb.plan(pending, states, edge, None, None, now, cfg),
        "_checked_pending": lambda: sc._checked_pending(pending, states),
        "_ranks": lambda: sc._ranks([r.task_id for r in reqs]),
        "issued base": lambda: sc._issued_base([r.issued_at for r in reqs]),
        "pack_mapped": lambda: fl.pack_mapped(reqs, states, rank, 4 * (3 * n + 1)),
        "kr_plan_small launch + sync": launch_sync,
        "current_stream()": lambda: torch.cuda.current_stream(),
        "empty launch-less sync": lambda: st.synchronize(),
    }
    print(f"n={n}: " + ", ".join(f"{k} {med(f):.1f} us" for k, f in parts.items()), flush=True)
