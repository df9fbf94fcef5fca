"""A/B the urgency kernel of two builds of the library on the same box:
    python tools/ab_urgency.py path/to/libA.so path/to/libB.so"""
import ctypes
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2605_11381_b200 import _lib, device as dev, fleet as fl, synthetic  # noqa: E402

R = 1 << 20
soa = synthetic.fleet_soa(R, seed=1)
fleet = fl.DeviceFleet.from_host(soa)
sched = fl.sched_struct("kairos", 10, 5, 150_000, 166_667, synthetic.NOW, 30,
                        synthetic.NOW - (1 << 39))
keys = fl.new_keys(R)
need = torch.empty(R, dtype=torch.int64, device="cuda")
stats = fl.new_key_stats()
fs = fleet.c_struct()
for path in sys.argv[1:] * 2:
    lib = _lib.load(path)
    def run():
        lib.kr_key_stats_init(stats.data_ptr(), dev.stream())
        lib.kr_urgency(ctypes.byref(fs), ctypes.byref(sched), keys.data_ptr(), need.data_ptr(),
                       None, None, None, None, None, stats.data_ptr(), None, dev.stream())
    for _ in range(5):
        run()
    # captured: 20 launches per graph, device time per launch (no host gaps)
    g = torch.cuda.CUDAGraph()
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        for _ in range(20):
            run()
    g.replay()
    ts = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); g.replay(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / 20)
    print(Path(path).name, "median ms per launch (graph)", round(statistics.median(ts), 4))
