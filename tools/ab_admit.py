"""A/B the admission (kr_select_admit: select + admit + ordered S_e) of two
library builds on the same box, on the keys of the bench fleet:
    python tools/ab_admit.py path/to/libA.so path/to/libB.so"""
import ctypes
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2605_11381_b200 import _lib, device as dev, fleet as fl, synthetic  # noqa: E402

R, k = 1 << 20, 8192
soa = synthetic.fleet_soa(R, seed=1)
fleet = fl.DeviceFleet.from_host(soa)
sched = fl.sched_struct("kairos", 10, 5, 150_000, 166_667, synthetic.NOW, 30,
                        synthetic.NOW - (1 << 39))
stats = fl.new_key_stats()
fl.key_stats_init(stats)
u = fl.urgency(fleet, sched, need_time=False, key_stats=stats)
ws = fl.Workspace(R)
adm = torch.empty(R, dtype=torch.uint8, device="cuda")
ref = torch.empty(R, dtype=torch.uint8, device="cuda")
eidx = torch.empty(k, dtype=torch.int32, device="cuda")
ekeys = fl.new_keys(k)
skipped0 = fleet.t["skipped"].clone()
fs = fleet.c_struct()
results = {}
for path in sys.argv[1:] * 3:
    lib = _lib.load(path)
    def run():
        lib.kr_select_admit(u.keys.data_ptr(), R, k, stats.data_ptr(), ctypes.byref(fs),
                            ctypes.byref(sched), adm.data_ptr(), ref.data_ptr(), eidx.data_ptr(),
                            ekeys.data_ptr(), None, ws.ptr(), ws.nbytes, dev.stream())
    for _ in range(3):
        run()
    ts = []
    for _ in range(20):
        fleet.t["skipped"].copy_(skipped0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); run(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    results.setdefault(Path(path).name, []).append(statistics.median(ts))
    results[Path(path).name + " S_e"] = eidx.cpu().numpy().tobytes().__hash__()
for k_, v in results.items():
    print(k_, v)
