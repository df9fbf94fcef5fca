"""Small driver for ncu captures of the non-headline horizon kernels:
    python profiles/prof_kernels.py conf|div32|ens|sweep16 [R]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2605_11381_b200 as kb  # noqa: E402
from paper_2605_11381_b200 import synthetic  # noqa: E402
from paper_2605_11381_b200.divergence import round_optimal_horizon_batch  # noqa: E402

which = sys.argv[1]
R = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 20
if which == "conf":
    U = synthetic.magnitudes(R, seed=3)
    for _ in range(3):
        kb.decide_horizon_batch(kb.HorizonPolicyConfig.confidence(0.4, 5), U, validate=False)
elif which.startswith("sweep"):
    C = int(which[5:])
    U = synthetic.magnitudes(R, seed=3)
    cfgs = [kb.HorizonPolicyConfig.confidence(0.013 + 0.947 * c / max(C - 1, 1), 1 + c % 8)
            for c in range(C)]
    for _ in range(3):
        kb.sweep_horizon_sums(cfgs, U, validate=False)
else:
    S, L, D = (1, 64, 32) if which == "div32" else (8, 50, 7)
    RR = R // 2 if which == "div32" else R // 4
    prev, cand, off = synthetic.chunks(RR, seed=5, Lp=L, Lc=L, D=D, S=S)
    for _ in range(3):
        round_optimal_horizon_batch(prev, cand, 0.9, offset=off)
torch.cuda.synchronize()
