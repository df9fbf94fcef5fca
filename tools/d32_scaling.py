import sys, statistics
sys.path.insert(0, '/root/repo')
import torch
from paper_2605_11381_b200 import synthetic
from paper_2605_11381_b200.divergence import round_optimal_horizon_batch
for R in (4096, 8192, 16384, 65536, 262144):
    prev, cand, off = synthetic.chunks(R, seed=5, Lp=64, Lc=64, D=32)
    out = torch.empty(R, dtype=torch.int32, device="cuda")
    f = lambda: round_optimal_horizon_batch(prev, cand, 0.9, offset=off, out=out)
    for _ in range(3): f()
    ts = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); f(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    t = statistics.median(ts) / 1e3
    print(R, round(t * 1e6, 1), "us", round(R * 16392 / t / 1e9), "GB/s")
