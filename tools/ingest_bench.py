"""Trace-ingest throughput on this host: the native reader (kr_trace_parse ->
TraceColumns) vs the reference's load_traces (Python json + numpy objects),
on the reference-written fixture files replicated to N traces.  Run in the
build container (imports /root/reference):  python tools/ingest_bench.py [N]"""
import json
import os
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

from roboserve import workload  # noqa: E402

from paper_2605_11381_b200 import traces as tr  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
tr_threads = os.cpu_count()
lines = [l for f in sorted((ROOT / "tests/golden/traces").glob("*.jsonl"))
         for l in f.read_text().splitlines() if l.strip()]
with tempfile.TemporaryDirectory() as td:
    p = Path(td) / "big.jsonl"
    with p.open("w") as fh:
        for i in range(N):
            d = json.loads(lines[i % len(lines)])
            d["task_id"] = f"task-{i:06d}"
            fh.write(json.dumps(d, separators=(",", ":")) + "\n")
    mb = p.stat().st_size / 1e6
    tr.load_trace_columns(ROOT / "tests/golden/traces/c_mixed.jsonl")  # warm: library load
    t0 = time.perf_counter(); cols = tr.load_trace_columns(p); t1 = time.perf_counter()
    ref = workload.load_traces(p); t2 = time.perf_counter()
    t3 = time.perf_counter(); objs = tr.load_traces(p); t4 = time.perf_counter()
    assert len(ref) == cols.n_traces == len(objs)
    print(json.dumps({"traces": N, "rounds": cols.n_rounds, "file_mb": round(mb, 2),
                      "native_columns_s": round(t1 - t0, 3), "native_MBps": round(mb / (t1 - t0), 1),
                      "native_objects_s": round(t4 - t3, 3),
                      "reference_load_traces_s": round(t2 - t1, 3),
                      "reference_MBps": round(mb / (t2 - t1), 1),
                      "speedup_columns": round((t2 - t1) / (t1 - t0), 1),
                      "threads": tr_threads, "reference_threads": 1}))
