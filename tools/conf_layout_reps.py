"""Repeated confidence-round timings per (layout, reserved SMs), fp32 and fp64
magnitudes (configs[4] shape), interleaved so drifts hit every layout alike:
    python tools/conf_layout_reps.py"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2605_11381_b200 import HorizonPolicyConfig, fleet as fl, rounds, synthetic  # noqa: E402

LAYOUTS = [("split", 2), ("split", 16), ("urgency_first", 1), ("urgency_first", 4)]
if os.environ.get("CONF_LAYOUTS"):  # e.g. "split:12,split:20"
    LAYOUTS = [(x.split(":")[0], int(x.split(":")[1])) for x in os.environ["CONF_LAYOUTS"].split(",")]


def timed(rnd, reps=150):
    for _ in range(10):
        rnd.replay()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(reps):
        rnd.replay()
    b.record()
    torch.cuda.synchronize()
    return 1e3 * a.elapsed_time(b) / reps


R = 1 << 20
import os
DT = {"32": [torch.float32], "64": [torch.float64]}.get(os.environ.get("CONF_DT", ""), [torch.float32, torch.float64])
for dt in DT:
    soa = synthetic.fleet_soa(R, seed=18)
    fleet = fl.DeviceFleet.from_host(soa)
    sched = fl.sched_struct("kairos", 10, 5, 150_000, 166_667, synthetic.NOW, 30,
                            int(soa["issued_at"].min()))
    inp = rounds.ConfidenceInputs(synthetic.magnitudes(R, seed=19, dtype=dt),
                                  HorizonPolicyConfig.confidence(0.4, 5))
    res = {lr: [] for lr in LAYOUTS}
    for rep in range(4):
        for lay, r in LAYOUTS:
            rnd = rounds.DecisionRound(R, 8192, sched)
            rnd.capture(fleet, inp, reserve_sms=r, layout=lay)
            res[(lay, r)].append(round(timed(rnd), 1))
    for k, v in res.items():
        print(str(dt).split(".")[-1], k, v, "median", sorted(v)[len(v) // 2], flush=True)
