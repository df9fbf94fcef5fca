"""Small-fleet round (BASELINE configs[1]: 1k robots, 50x7, k=64) for ncu
launch lists:  ncu --metrics gpu__time_duration.sum python profiles/prof_small.py [R] [k]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2605_11381_b200 import fleet as fl, rounds, synthetic  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
k = int(sys.argv[2]) if len(sys.argv) > 2 else 64
soa = synthetic.fleet_soa(R, seed=11)
fleet = fl.DeviceFleet.from_host(soa)
prev, cand, off = synthetic.chunks(R, seed=12)
sched = fl.sched_struct("kairos", 10, 5, 150_000, 166_667, synthetic.NOW, 30,
                        int(soa["issued_at"].min()))
rnd = rounds.DecisionRound(R, k, sched)
inp = rounds.DivergenceInputs(prev, cand, 0.9, offset=off)
for _ in range(3):
    rnd.run(fleet, inp)
torch.cuda.synchronize()
print("done")
