"""Time the phases of the fleet-scale hybrid round at 2^20 robots
(HybridDecisionRound): urgency, full key sort, edge admission, offload scan."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import ctypes  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2605_11381_b200 import _lib, device as dev, engines as eng, fleet as fl, rounds, synthetic  # noqa: E402

R, k = 1 << 20, 8192
soa = synthetic.fleet_soa(R, seed=20)
fleet = fl.DeviceFleet.from_host(soa)
sched = fl.sched_struct("kairos", 10, 5, 150_000, 166_667, synthetic.NOW, 30, int(soa["issued_at"].min()))
edge = eng.EngineProfile(tier="edge", capacity=k, max_batch=256, points=((1, 150_000), (256, 400_000)))
cloud = eng.EngineProfile(tier="cloud", capacity=2048, max_batch=512, points=((1, 80_000), (512, 250_000)))
net = eng.NetworkModel(base_latency_us=20_000, uplink_bps=400_000_000, downlink_bps=1_000_000_000)
rnd = rounds.HybridDecisionRound(R, k, sched, cloud.capacity)
payload = torch.from_numpy(np.random.default_rng(22).choice(np.array([100_000, 300_000, 2_000_000], np.int64), R)).cuda()
up = eng.transfer_time_batch(net, payload, eng.UP)
thr = eng.cloud_thresholds(edge, cloud, net, 0, 0, k, rnd.cap)
rnd.set_cloud(up, thr)
print("T(c) first/last:", thr[0], thr[-1], "uplink values:", sorted(set(up.cpu().numpy().tolist())))


def t(fn, n=5):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n


print("urgency ms", t(lambda: rnd.urgency(fleet)))
print("admit (select k+window, edge admission, offload scan) ms", t(lambda: rnd.admit(fleet)),
      "n_cloud", int(rnd.n_cloud.item()), "full sorts", rnd.full_sorts)
order = rnd.full_order()
print("full key sort ms", t(lambda: rnd.full_order()))
fs = fleet.c_struct()


def place():
    _lib.check(rnd.lib.kr_place_cloud(order.data_ptr(), R, k, up.data_ptr(), rnd.thresholds.data_ptr(), rnd.cap,
                                      ctypes.byref(fs), ctypes.byref(sched), rnd.refetch.data_ptr(),
                                      rnd.cloud_idx.data_ptr(), rnd.n_cloud.data_ptr(), dev.stream()), "place")


print("offload scan over the full order ms", t(place), "n_cloud", int(rnd.n_cloud.item()))
rnd2 = rounds.HybridDecisionRound(R, k, sched, cloud.capacity)
rnd2.set_cloud(up, [min(x, 30_000) for x in thr])  # only the smallest payloads qualify
rnd2.urgency(fleet)
print("admit, sparse qualifiers ms", t(lambda: rnd2.admit(fleet)), "n_cloud", int(rnd2.n_cloud.item()),
      "full sorts", rnd2.full_sorts)
