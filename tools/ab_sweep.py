"""A/B the threshold-sweep kernel of two library builds (C = 16, K=6 N=50 fp32,
2^20 robots):  python tools/ab_sweep.py libA.so libB.so"""
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2605_11381_b200 import _lib, horizon, synthetic  # noqa: E402

U = synthetic.magnitudes(1 << 20, seed=3)
cfgs = [horizon.HorizonPolicyConfig.confidence(0.013 + 0.947 * c / 15, 1 + c % 8) for c in range(16)]
res = {}
for path in sys.argv[1:] * 3:
    _lib._LIB = _lib.load(path)  # the package's calls go to this build
    f = lambda: horizon.sweep_horizon_sums(cfgs, U, validate=False)
    ref = f().cpu()
    for _ in range(3):
        f()
    ts = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); f(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    res.setdefault(Path(path).name, []).append((round(statistics.median(ts), 4), int(ref.sum())))
for k, v in res.items():
    print(k, v)
