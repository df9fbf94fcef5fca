"""Where the confidence-policy round's time goes (configs[4] shape: 2^20
robots, U 6x50 fp32, k = 8192): the horizon graph alone (all SMs / capped),
the urgency + admission graph alone, and the concurrent round per layout and
reserved-SM count with the side stream's own span.
    python tools/conf_round_diag.py [reserve ...]"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2605_11381_b200 import HorizonPolicyConfig, fleet as fl, rounds, synthetic  # noqa: E402

REPS = 100


def timed(fn, reps=REPS):
    for _ in range(5):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return 1e3 * a.elapsed_time(b) / reps


def main():
    reserves = [int(x) for x in sys.argv[1:]] or [-1, 8, 16, 24, 32]
    R = 1 << 20
    soa = synthetic.fleet_soa(R, seed=18)
    fleet = fl.DeviceFleet.from_host(soa)
    import os
    U = synthetic.magnitudes(R, seed=19, dtype=torch.float64 if os.environ.get("CONF_FP64") else torch.float32)
    sched = fl.sched_struct("kairos", 10, 5, 150_000, 166_667, synthetic.NOW, 30,
                            int(soa["issued_at"].min()))
    inp = rounds.ConfidenceInputs(U, HorizonPolicyConfig.confidence(0.4, 5))
    out = {}
    rnd = rounds.DecisionRound(R, 8192, sched)
    rnd.capture(fleet, inp, reserve_sms=0, layout="split")
    out["horizon_graph_all_sms_us"] = timed(rnd.g_horizon.replay)
    out["urgency_admission_graph_us"] = timed(rnd.g_decide.replay)
    out["sequential_round_us"] = timed(rnd.replay)
    for layout in ("split", "urgency_first"):
        for r in reserves:
            rnd = rounds.DecisionRound(R, 8192, sched)
            rnd.capture(fleet, inp, reserve_sms=r, layout=layout)
            h_only = timed(rnd.g_horizon.replay)
            ev = {}

            def mark(name):
                def f(stream):
                    e = torch.cuda.Event(enable_timing=True)
                    e.record(stream)
                    ev[name] = e
                return f
            t = timed(rnd.replay)
            rnd.replay_concurrent(before_horizon=mark("h0"), after_horizon=mark("h1"),
                                  before_side=mark("s0"), after_side=mark("s1"))
            torch.cuda.synchronize()
            side = ev["s0"].elapsed_time(ev["s1"]) * 1e3 if "s0" in ev else None
            hor = ev["h0"].elapsed_time(ev["h1"]) * 1e3
            out[f"{layout} reserve={r}"] = {"round_us": round(t, 1), "horizon_alone_us": round(h_only, 1),
                                            "horizon_in_round_us": round(hor, 1),
                                            "side_in_round_us": round(side, 1) if side else None}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
