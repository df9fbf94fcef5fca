"""Radix-select shape on the bench fleet's keys (2^20 robots, k = 8192): the
level-0 digit width, the boundary bin's population (the candidates the
single-CTA finish walks) and the histogram's concentration.
    python tools/sel_diag.py [R] [k]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2605_11381_b200 import fleet as fl, synthetic  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
k = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
soa = synthetic.fleet_soa(R, seed=1)
fleet = fl.DeviceFleet.from_host(soa)
sched = fl.sched_struct("kairos", 10, 5, 150_000, 166_667, synthetic.NOW, 30,
                        synthetic.NOW - (1 << 39))
stats = fl.new_key_stats()
fl.key_stats_init(stats)
u = fl.urgency(fleet, sched, need_time=False, key_stats=stats)
ws = fl.Workspace(R)
fl.select_admit(u.keys, k, ws, key_stats=stats)
torch.cuda.synchronize()
b = ws.buf[:276 + 4 * 2048].cpu().numpy().tobytes()
i32 = np.frombuffer(b[:276], dtype=np.int32)
W = int(np.frombuffer(b[160:164], dtype=np.int32)[0])
nrun = int(np.frombuffer(b[164:168], dtype=np.int32)[0])
run_pos = np.frombuffer(b[168:212], dtype=np.int32)[:nrun]
run_len = np.frombuffer(b[212:256], dtype=np.int32)[:nrun]
dstar0 = int(np.frombuffer(b[260:264], dtype=np.uint32)[0])
hist = np.frombuffer(b[276:276 + 4 * 2048], dtype=np.uint32)
nz = hist[hist > 0]
keys = u.keys.cpu().numpy().view(np.uint64).reshape(-1, 2)
print(f"R={R} k={k} digit W={W} runs={list(zip(run_pos.tolist(), run_len.tolist()))}")
print(f"boundary bin {dstar0}: {int(hist[dstar0])} keys; nonzero bins {nz.size}, max bin {int(hist.max())}")
print(f"distinct hi words {np.unique(keys[:, 0]).size}  (key.hi = bucket | aged)")
top = np.sort(hist)[::-1][:8]
print("largest bins", top.tolist())
