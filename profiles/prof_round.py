"""Profiling driver: a few decision rounds at the bench workload (2^20 robots,
50x7 fp32 chunks, k = 8192) for ncu.  Usage under gpurun:
  ncu --set full -k regex:k_horizon_divergence -s 2 -c 1 -o gpurun_out/div python profiles/prof_round.py
  (args: [R] [steps] [conf]: the confidence-policy round with U 2^20 x 6 x 50 fp32)
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2605_11381_b200 import fleet as fl, rounds, synthetic  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
soa = synthetic.fleet_soa(R, seed=1)
fleet = fl.DeviceFleet.from_host(soa)
prev, cand, off = synthetic.chunks(R, seed=2)
sched = fl.sched_struct("kairos", 10, 5, 150_000, 166_667, synthetic.NOW, 30,
                        synthetic.NOW - (1 << 39))
rnd = rounds.DecisionRound(R, 8192, sched)
inp = rounds.DivergenceInputs(prev, cand, 0.9, offset=off)
if len(sys.argv) > 3 and sys.argv[3] == "conf":  # the confidence-policy round instead
    from paper_2605_11381_b200 import HorizonPolicyConfig
    inp = rounds.ConfidenceInputs(synthetic.magnitudes(R, seed=19), HorizonPolicyConfig.confidence(0.4, 5))
for _ in range(steps):
    rnd.run(fleet, inp)
torch.cuda.synchronize()
print("done")
