"""A/B the configs[1]-[3] rounds (captured, split layout) across library builds:
    python tools/ab_rounds.py libA.so libB.so ..."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2605_11381_b200 import _lib, fleet as fl, rounds, synthetic  # noqa: E402

sys.argv += []
import importlib.util  # noqa: E402
spec = importlib.util.spec_from_file_location("sl", Path(__file__).resolve().parent / "small_layouts.py")
for path in sys.argv[1:] * 2:
    _lib._LIB = _lib.load(path)
    res = []
    R = 16384
    soa = synthetic.fleet_soa(R, seed=13)
    pa, ca, oa = synthetic.chunks(R // 2, seed=14, Lp=64, Lc=64, D=7)
    ph, chh, oh = synthetic.chunks(R // 2, seed=15, Lp=64, Lc=64, D=32)
    inp = rounds.MixedInputs([(0, rounds.DivergenceInputs(pa, ca, 0.9, offset=oa)),
                              (R // 2, rounds.DivergenceInputs(ph, chh, 0.9, offset=oh))])
    fleet = fl.DeviceFleet.from_host(soa)
    sched = fl.sched_struct("kairos", 10, 5, 150_000, 166_667, synthetic.NOW, 30,
                            int(soa["issued_at"].min()))
    for reserve in (0, -1):
        rnd = rounds.DecisionRound(R, 1024, sched)
        rnd.capture(fleet, inp, reserve_sms=reserve, layout="split")
        for _ in range(10):
            rnd.replay()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        for _ in range(300):
            rnd.replay()
        b.record()
        torch.cuda.synchronize()
        res.append(round(1e3 * a.elapsed_time(b) / 300, 2))
    print(Path(path).name, "configs[2] us (sequential, concurrent):", res)
