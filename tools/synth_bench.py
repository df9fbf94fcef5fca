"""Device trace synthesis: throughput of synthesize_family_columns (device
columns, no host objects) and the distribution statistics next to the
reference's (tests/golden/synth_stats.json).  Run under gpurun:
    python tools/synth_bench.py [tasks]"""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import torch  # noqa: E402

import golden_io  # noqa: E402
import paper_2605_11381_b200 as kb  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
spec, pol = kb.SyntheticSpec(), kb.HorizonPolicyConfig.confidence()
kb.synthesize_family_columns(spec, pol, 100_000, 1000, seed=1)  # warm-up
torch.cuda.synchronize()
t0 = time.perf_counter()
cols = kb.synthesize_family_columns(spec, pol, 100_000, T, seed=2)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
print(json.dumps({"tasks": T, "rounds": cols.n_rounds, "s": dt, "tasks_per_s": T / dt,
                  "rounds_per_s": cols.n_rounds / dt}))
for s in golden_io.synth()["settings"]:
    sp = kb.SyntheticSpec(**s["spec"])
    kind, kw = s["policy"]
    p = kb.HorizonPolicyConfig.confidence(**kw) if kind == "confidence" else kb.HorizonPolicyConfig.static(**kw)
    got = golden_io.synth_stats(kb.synthesize_family(sp, p, s["gen_latency"], 3000, seed=5), s["spec"])
    keys = ["rounds_per_task", "horizon_mean", "horizon_std", "trigger_mean", "tail_mean", "u0_mean",
            "success_mean"]
    print(json.dumps({"setting": s["spec"], "policy": s["policy"],
                      "device": {k: round(got[k], 4) for k in keys},
                      "reference": {k: round(s["stats"][k], 4) for k in keys}}))
