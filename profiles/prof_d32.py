"""D=32 divergence at a small fleet (configs[2] humanoid half: 8k robots, 64x32)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2605_11381_b200 import synthetic  # noqa: E402
from paper_2605_11381_b200.divergence import round_optimal_horizon_batch  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
prev, cand, off = synthetic.chunks(R, seed=5, Lp=64, Lc=64, D=32)
for _ in range(3):
    round_optimal_horizon_batch(prev, cand, 0.9, offset=off)
torch.cuda.synchronize()
