"""Diagnose the pipelined e2e: H2D of the next chunk on a copy stream while the
current round computes.  Variants: copy only / + compute / + D2H."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2605_11381_b200 import fleet as fl, rounds, synthetic  # noqa: E402

R = 1 << 20
soa = synthetic.fleet_soa(R, seed=1)
fleet = fl.DeviceFleet.from_host(soa)
prev, cand, off = synthetic.chunks(R, seed=2)
sched = fl.sched_struct("kairos", 10, 5, 150_000, 166_667, synthetic.NOW, 30, synthetic.NOW - (1 << 39))
rnd = rounds.DecisionRound(R, 8192, sched)
h = [cand[:, 0].cpu().pin_memory(), prev.cpu().pin_memory()]
ring = [torch.empty_like(prev) for _ in range(3)]
outH = torch.empty(R, dtype=torch.int32).pin_memory()
cs, xs = torch.cuda.current_stream(), torch.cuda.Stream()
inp = [rounds.DivergenceInputs(ring[(a + 2) % 3], ring[a], 0.9, offset=off) for a in range(3)]
rnd.run(fleet, inp[0]); torch.cuda.synchronize()

def go(steps, compute, d2h):
    h2d = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    h2s = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    done = [torch.cuda.Event() for _ in range(steps)]
    s0, e0 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record(cs)
    for i in range(steps):
        a = i % 3
        with torch.cuda.stream(xs):
            if i == 0: xs.wait_event(s0)
            if i >= 2: xs.wait_event(done[i - 2])
            h2s[i].record(xs)
            ring[a].copy_(h[i & 1], non_blocking=True)
            h2d[i].record(xs)
        cs.wait_event(h2d[i])
        if compute:
            o = rnd.run(fleet, inp[a])
            if d2h:
                outH.copy_(o.horizon, non_blocking=True)
        done[i].record(cs)
    e0.record(cs)
    torch.cuda.synchronize()
    per = [h2s[i].elapsed_time(h2d[i]) for i in range(steps)]
    print(f"compute={compute} d2h={d2h}: {s0.elapsed_time(e0)/steps:.2f} ms/step, h2d {[round(x,1) for x in per]}")

for c, d in ((False, False), (True, False), (True, True)):
    go(6, c, d)
