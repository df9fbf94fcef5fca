"""Round time per reserved-SM count for the bench's other configs (the split
layout's side-stream share during the horizon kernel):
    python tools/config_reserve_sweep.py [reserve ...]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2605_11381_b200 import HorizonPolicyConfig, fleet as fl, rounds, synthetic  # noqa: E402

THR = 0.9
RES = [int(x) for x in sys.argv[1:]] or [2, 4, 6, 8, 10, 12]


def timed(rnd, fleet, inp, reserve, reps=150):
    rnd.capture(fleet, inp, reserve_sms=reserve, layout="split")
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


def sched_for(soa):
    return fl.sched_struct("kairos", 10, 5, 150_000, 166_667, synthetic.NOW, 30,
                           int(soa["issued_at"].min()))


def case(name, R, k, make_inp, seed):
    soa = synthetic.fleet_soa(R, seed=seed)
    fleet = fl.DeviceFleet.from_host(soa)
    inp = make_inp()
    for rep in range(2):
        row = []
        for r in RES:
            rnd = rounds.DecisionRound(R, k, sched_for(soa))
            row.append(round(timed(rnd, fleet, inp, r), 1))
        print(name, "rep", rep, dict(zip(RES, row)), flush=True)


R = 1 << 20
case("configs[3]", 65536, 8192, lambda: rounds.DivergenceInputs(
    *synthetic.chunks(65536, seed=17, S=8)[:2], THR, offset=synthetic.chunks(65536, seed=17, S=8)[2]), 16)
case("conf fp32", R, 8192, lambda: rounds.ConfidenceInputs(
    synthetic.magnitudes(R, seed=19), HorizonPolicyConfig.confidence(0.4, 5)), 18)
case("conf fp64", R, 8192, lambda: rounds.ConfidenceInputs(
    synthetic.magnitudes(R, seed=25, dtype=torch.float64), HorizonPolicyConfig.confidence(0.4, 5)), 23)
case("div fp64", R, 8192, lambda: rounds.DivergenceInputs(
    *synthetic.chunks(R, seed=24, dtype=torch.float64)[:2], THR,
    offset=synthetic.chunks(R, seed=24, dtype=torch.float64)[2]), 23)
