"""A/B the full key sort (kr_sort_keys, 2^20 kairos keys) across library builds:
    python tools/ab_sort.py libA.so libB.so ..."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2605_11381_b200 import _lib, fleet as fl, synthetic  # noqa: E402

R = 1 << 20
soa = synthetic.fleet_soa(R, seed=20)
sched = fl.sched_struct("kairos", 10, 5, 150_000, 166_667, synthetic.NOW, 30, int(soa["issued_at"].min()))
for path in sys.argv[1:] * 2:
    _lib._LIB = _lib.load(path)
    fleet = fl.DeviceFleet.from_host(soa)
    keys = fl.urgency(fleet, sched, need_time=False).keys
    ws = fl.Workspace(R)
    order, sk = fl.sort_keys(keys, ws)
    ref = order.clone()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        fl.sort_keys(keys, ws, order=order, sorted_keys=sk)
    b.record()
    torch.cuda.synchronize()
    print(Path(path).name, round(a.elapsed_time(b) / 10, 3), "ms", int(ref[:100].sum()))
