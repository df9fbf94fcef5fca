"""The confidence round (fp64 magnitudes, split/16) on one evolving fleet: per
repeat the round time and the radix select's level-0 boundary-bin population
(SelState::hist[dstar0] in the round's workspace):
    python tools/conf_bin_diag.py"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2605_11381_b200 import HorizonPolicyConfig, fleet as fl, rounds, synthetic  # noqa: E402

R = 1 << 20
soa = synthetic.fleet_soa(R, seed=18)
fleet = fl.DeviceFleet.from_host(soa)
sched = fl.sched_struct("kairos", 10, 5, 150_000, 166_667, synthetic.NOW, 30,
                        int(soa["issued_at"].min()))
inp = rounds.ConfidenceInputs(synthetic.magnitudes(R, seed=19, dtype=torch.float64),
                              HorizonPolicyConfig.confidence(0.4, 5))
for rep in range(4):
    rnd = rounds.DecisionRound(R, 8192, sched)
    rnd.capture(fleet, inp, reserve_sms=16, layout="split")
    ts = []
    bins = []
    for it in range(20):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); rnd.replay(); b.record(); torch.cuda.synchronize()
        ts.append(1e3 * a.elapsed_time(b))
        raw = rnd.ws.buf[:276 + 4 * 2048].cpu().numpy().tobytes()
        d0 = int(np.frombuffer(raw[260:264], dtype=np.uint32)[0])
        bins.append(int(np.frombuffer(raw[276:276 + 4 * 2048], dtype=np.uint32)[d0]))
    print(f"rep {rep}: round us median {np.median(ts):.1f} (min {min(ts):.1f}, max {max(ts):.1f}); "
          f"boundary bin keys median {int(np.median(bins))} (min {min(bins)}, max {max(bins)})", flush=True)
