"""configs[2] round (8k arms 64x7 + 8k humanoids 64x32, k=1024) for ncu launch lists."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2605_11381_b200 import _lib, device as dev, fleet as fl, rounds, synthetic  # noqa: E402

R = 16384
lib = _lib.load()
soa = synthetic.fleet_soa(R, seed=13)
fleet = fl.DeviceFleet.from_host(soa)
pa, ca, oa = synthetic.chunks(R // 2, seed=14, Lp=64, Lc=64, D=7)
ph, chh, oh = synthetic.chunks(R // 2, seed=15, Lp=64, Lc=64, D=32)
sched = fl.sched_struct("kairos", 10, 5, 150_000, 166_667, synthetic.NOW, 30,
                        int(soa["issued_at"].min()))
rnd = rounds.DecisionRound(R, 1024, sched)


def div_into(H, prev, cand, off):
    n, Lp, D = prev.shape
    _lib.check(lib.kr_horizon_divergence(prev.data_ptr(), cand.data_ptr(), _lib.KR_F32, n, 1, Lp,
                                         cand.shape[2], D, off.data_ptr(), None, None, 0.9,
                                         H.data_ptr(), None, 0, dev.stream()), "div")


for _ in range(3):
    div_into(rnd.H[: R // 2], pa, ca, oa)
    div_into(rnd.H[R // 2:], ph, chh, oh)
    rnd.urgency(fleet)
    rnd.admit(fleet)
torch.cuda.synchronize()
