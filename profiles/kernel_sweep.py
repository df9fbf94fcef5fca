"""Per-kernel throughput sweep over the BASELINE configs (run under gpurun):
    python profiles/kernel_sweep.py [R]
Prints one JSON line per variant: median device time of 10 warm launches
(CUDA events on the launching stream) and algorithmic GB/s."""
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2605_11381_b200 as kb  # noqa: E402
from paper_2605_11381_b200 import synthetic  # noqa: E402
from paper_2605_11381_b200.divergence import round_optimal_horizon_batch  # noqa: E402

PEAK = json.loads((Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]


def timeit(fn, reps=10, batch=1):
    """Median device time per call; batch > 1 enqueues that many calls between
    the two events (the host's per-call table building then overlaps the
    previous call's kernel, so the figure is the device time per call)."""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(batch):
            fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / 1e3 / batch)
    return statistics.median(ts)


def report(name, R, bytes_per, t, needed=None):
    gbs = bytes_per * R / t / 1e9
    line = {"variant": name, "robots": R, "bytes_per_robot_round": bytes_per,
            "ms": t * 1e3, "GBps": round(gbs, 1), "frac_of_measured_peak": round(gbs / PEAK, 3),
            "robot_rounds_per_s": R / t}
    if needed is not None:  # bytes a decision can read (the compared rows only)
        line["needed_bytes_per_robot_round"] = round(needed, 1)
        line["needed_GBps"] = round(needed * R / t / 1e9, 1)
        line["needed_frac_of_measured_peak"] = round(needed * R / t / 1e9 / PEAK, 3)
    print(json.dumps(line), flush=True)


def main():
    R = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
    only = sys.argv[2] if len(sys.argv) > 2 else ""
    if only != "div":
        horizon_policy(R)
    divergence(R)


def horizon_policy(R):
    for K, N, dt, es in [(6, 50, torch.float32, 4), (6, 50, torch.float64, 8), (6, 64, torch.float32, 4)]:
        U = synthetic.magnitudes(R, seed=3, K=K, N=N, dtype=dt)
        cfg = kb.HorizonPolicyConfig.confidence(0.4, 5)
        out = torch.empty(R, dtype=torch.int32, device="cuda")
        t = timeit(lambda: kb.decide_horizon_batch(cfg, U, out=out, validate=False))
        report(f"confidence K={K} N={N} {str(dt)[6:]}", R, K * N * es + 4, t)
        del U
    U = synthetic.magnitudes(R, seed=3, K=6, N=50, dtype=torch.float32)
    # thresholds 0.013..0.96 avoid the synthetic bump 1.8x (a tie at t = 0.8
    # sends every uncertain-tail column down the exact fp64 path): "tie" adds it
    for C, tie in ((1, False), (16, False), (64, False), (16, True)):
        ts = [0.013 + 0.947 * c / max(C - 1, 1) for c in range(C)]
        if tie:
            ts[-1] = 0.8
        cfgs = [kb.HorizonPolicyConfig.confidence(t, 1 + c % 8) for c, t in enumerate(ts)]
        t = timeit(lambda: kb.sweep_horizon_sums(cfgs, U, validate=False))
        report(f"sweep C={C}{' tie@0.8' if tie else ''} K=6 N=50 float32 (sums, per call)", R, 6 * 50 * 4, t)
        t = timeit(lambda: kb.sweep_horizon_sums(cfgs, U, validate=False), batch=10)
        report(f"sweep C={C}{' tie@0.8' if tie else ''} K=6 N=50 float32 (sums, back to back)", R, 6 * 50 * 4, t)
    del U
    # the other layouts: fp64 storage, N = 49 (odd: warp per robot), N = 128 (VC = 4)
    cfgs = [kb.HorizonPolicyConfig.confidence(0.013 + 0.947 * c / 15, 1 + c % 8) for c in range(16)]
    for K, N, dt, es in [(6, 50, torch.float64, 8), (6, 49, torch.float32, 4),
                         (6, 128, torch.float32, 4)]:
        U = synthetic.magnitudes(R, seed=3, K=K, N=N, dtype=dt)
        t = timeit(lambda: kb.sweep_horizon_sums(cfgs, U, validate=False), batch=10)
        report(f"sweep C=16 K={K} N={N} {str(dt)[6:]} (sums, back to back)", R, K * N * es, t)
        del U


def divergence(R):
    for S, L, D, RR, dt in [(1, 50, 7, R, torch.float32), (1, 64, 32, R // 2, torch.float32),
                            (8, 50, 7, R // 4, torch.float32), (1, 50, 7, R, torch.float64)]:
        es = 4 if dt == torch.float32 else 8
        prev, cand, off = synthetic.chunks(RR, seed=5, Lp=L, Lc=L, D=D, S=S, dtype=dt)
        lim = (L - off.clamp(min=0)).clamp(min=0, max=L).double().mean().item()
        out = torch.empty(RR, dtype=torch.int32, device="cuda")
        t = timeit(lambda: round_optimal_horizon_batch(prev, cand, 0.9, offset=off, out=out))
        report(f"divergence S={S} L={L} D={D} {str(dt)[6:]}", RR, (1 + S) * L * D * es + 8, t,
               needed=(1 + S) * lim * D * es + 8)
        del prev, cand


if __name__ == "__main__":
    main()
