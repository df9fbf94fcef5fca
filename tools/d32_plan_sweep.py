"""configs[2]'s humanoid group alone (8k robots, 64x32 fp32 chunks): the
divergence kernel's device time per launch (graph of 20), for plan knobs given
in the environment (KR_PLAN_FORCE_TR, KR_PLAN_MAX_STAGES):
    KR_TRACE_PLAN=1 python tools/d32_plan_sweep.py"""
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2605_11381_b200 import synthetic  # noqa: E402
from paper_2605_11381_b200.divergence import round_optimal_horizon_batch  # noqa: E402

R = 8192
prev, cand, off = synthetic.chunks(R, seed=15, Lp=64, Lc=64, D=32)
out = torch.empty(R, dtype=torch.int32, device="cuda")
for _ in range(3):
    round_optimal_horizon_batch(prev, cand, 0.9, off, out=out)
g = torch.cuda.CUDAGraph()
torch.cuda.synchronize()
with torch.cuda.graph(g):
    for _ in range(20):
        round_optimal_horizon_batch(prev, cand, 0.9, off, out=out)
g.replay()
ts = []
for _ in range(10):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); g.replay(); b.record(); torch.cuda.synchronize()
    ts.append(1e3 * a.elapsed_time(b) / 20)
print("us per launch", round(statistics.median(ts), 2), "GB/s", round(134.2e6 / statistics.median(ts) / 1e3, 0))
