"""cProfile of the object-level plan() at 16 pending requests (per-call overhead)."""
import cProfile
import pstats
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent))
sys.argv = [sys.argv[0]]
import plan_latency as pl  # noqa: E402  (runs its own timing loop once on import)

kb = pl.kb
states, pending, now = pl.instance(16)
for _ in range(5):
    kb.plan(pending, states, pl.edge, None, None, now, pl.cfg)
pr = cProfile.Profile()
pr.enable()
for _ in range(200):
    kb.plan(pending, states, pl.edge, None, None, now, pl.cfg)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
