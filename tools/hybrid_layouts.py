"""The cloud-tier fleet round (bench other_configs shape: 2^20 robots, k = 8192
edge, 2048 cloud slots) per overlapped layout and reserved-SM count, eager,
interleaved repeats:  python tools/hybrid_layouts.py"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2605_11381_b200 import engines as eng, fleet as fl, rounds, synthetic  # noqa: E402

R, k = 1 << 20, 8192
soa = synthetic.fleet_soa(R, seed=20)
fleet = fl.DeviceFleet.from_host(soa)
prev, cand, off = synthetic.chunks(R, seed=21)
edge = eng.EngineProfile(tier="edge", capacity=k, max_batch=256, points=((1, 150_000), (256, 400_000)))
cloud = eng.EngineProfile(tier="cloud", capacity=2048, max_batch=512, points=((1, 80_000), (512, 250_000)))
net = eng.NetworkModel(base_latency_us=20_000, uplink_bps=400_000_000, downlink_bps=1_000_000_000)
sched = fl.sched_struct("kairos", 10, 5, 150_000, 166_667, synthetic.NOW, 30, int(soa["issued_at"].min()))
rnd = rounds.HybridDecisionRound(R, k, sched, cloud.capacity)
payload = torch.from_numpy(np.random.default_rng(22).choice(
    np.array([100_000, 300_000, 2_000_000], np.int64), R)).cuda()
rnd.set_cloud(eng.transfer_time_batch(net, payload, eng.UP),
              eng.cloud_thresholds(edge, cloud, net, 0, 0, k, rnd.cap))
inp = rounds.DivergenceInputs(prev, cand, 0.9, offset=off)
LAYOUTS = [("urgency_first", 10), ("urgency_first", 4), ("urgency_first", 2), ("split", 2), ("split", 10)]
res = {x: [] for x in LAYOUTS}
for rep in range(3):
    for lay, r in LAYOUTS:
        step = lambda: rnd.run_overlapped(fleet, inp, reserve_sms=r, layout=lay)
        for _ in range(5):
            step()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(40):
            step()
        b.record()
        torch.cuda.synchronize()
        res[(lay, r)].append(round(1e3 * a.elapsed_time(b) / 40, 1))
for x, v in res.items():
    print(x, v, "median", sorted(v)[1])
