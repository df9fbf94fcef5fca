"""One 2^20-robot divergence launch (bench workload shape) for ncu captures:
    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        -k regex:k_horizon_divergence python tools/div_once.py [S] [dtype]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2605_11381_b200 import synthetic  # noqa: E402
from paper_2605_11381_b200.divergence import round_optimal_horizon_batch  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 1
dt = torch.float64 if len(sys.argv) > 2 and sys.argv[2] == "f64" else torch.float32
R = (1 << 20) // (4 if S > 1 else 1)
prev, cand, off = synthetic.chunks(R, seed=2000, S=S, dtype=dt)
out = torch.empty(R, dtype=torch.int32, device="cuda")
for _ in range(2):
    round_optimal_horizon_batch(prev, cand, 0.9, offset=off, out=out)
torch.cuda.synchronize()
print("mean H", out.float().mean().item())
