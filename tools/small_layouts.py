"""configs[1]-[3] rounds under each captured layout (sequential graph vs the
two concurrent layouts, reserved-SM variants): python tools/small_layouts.py
[--confidence: the 2^20-robot confidence-policy round instead]"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2605_11381_b200 import fleet as fl, rounds, synthetic  # noqa: E402

THR, REPS = 0.9, 300


def sched_for(soa):
    return fl.sched_struct("kairos", 10, 5, 150_000, 166_667, synthetic.NOW, 30,
                           int(soa["issued_at"].min()))


def timed_seq(rnd, fleet, inp):
    rnd.run(fleet, inp)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        rnd.run(fleet, inp)
    return bench(g.replay)


def bench(fn):
    for _ in range(10):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(REPS):
        fn()
    b.record()
    torch.cuda.synchronize()
    return 1e3 * a.elapsed_time(b) / REPS


def cases():
    if "--confidence" in sys.argv:  # the headline fleet under the confidence policy
        from paper_2605_11381_b200 import HorizonPolicyConfig
        R = 1 << 20
        soa = synthetic.fleet_soa(R, seed=18)
        yield "configs[4] confidence", R, 8192, soa, rounds.ConfidenceInputs(
            synthetic.magnitudes(R, seed=19), HorizonPolicyConfig.confidence(0.4, 5))
        return
    R = 1024
    soa = synthetic.fleet_soa(R, seed=11)
    prev, cand, off = synthetic.chunks(R, seed=12)
    yield "configs[1]", R, 64, soa, rounds.DivergenceInputs(prev, cand, THR, offset=off)
    R = 16384
    soa = synthetic.fleet_soa(R, seed=13)
    pa, ca, oa = synthetic.chunks(R // 2, seed=14, Lp=64, Lc=64, D=7)
    ph, chh, oh = synthetic.chunks(R // 2, seed=15, Lp=64, Lc=64, D=32)
    yield "configs[2]", R, 1024, soa, rounds.MixedInputs(
        [(0, rounds.DivergenceInputs(pa, ca, THR, offset=oa)),
         (R // 2, rounds.DivergenceInputs(ph, chh, THR, offset=oh))])
    R = 65536
    soa = synthetic.fleet_soa(R, seed=16)
    prev, cand, off = synthetic.chunks(R, seed=17, S=8)
    yield "configs[3]", R, 8192, soa, rounds.DivergenceInputs(prev, cand, THR, offset=off)


for name, R, k, soa, inp in cases():
    fleet = fl.DeviceFleet.from_host(soa)
    res = {"sequential": timed_seq(rounds.DecisionRound(R, k, sched_for(soa)), fleet, inp)}
    for layout in ("split", "urgency_first"):
        for reserve in ((-1, 4, 8, 16, 24, 32) if "--confidence" in sys.argv else (-1, 4, 8, 16)):
            rnd = rounds.DecisionRound(R, k, sched_for(soa))
            rnd.capture(fleet, inp, reserve_sms=reserve, layout=layout)
            res[f"{layout} reserve={reserve}"] = bench(rnd.replay)
    print(json.dumps({"config": name, "us_per_round": {k_: round(v, 2) for k_, v in res.items()}}))
