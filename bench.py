"""Benchmark: robot-rounds/s of the Kairos decision core (horizon + urgency +
top-k admission) on B200, per BASELINE.json.

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...   (one rank per GPU)

Workload (BASELINE.json configs[4], one GPU's share; weak scaling): each GPU
owns R = 2^20 pending robots.  A step is one decision round over the whole
fleet: divergence horizon of the new 50x7 fp32 chunk against the unexecuted
overlap of the previous chunk (offset U[0,10], threshold 0.9), urgency keys
from 0-5-round histories, and edge admission of the global top k = 8192 (NCCL
all-gather of per-shard candidates when N > 1).  Inputs (2.9 GB per GPU) are
larger than L2, so no flush is needed between steps.

`value` is device-timed (CUDA events, barrier + synchronize both sides, max
over ranks) with inputs resident in HBM; `e2e` runs the same round through the
C ABI from pinned host buffers with the host->device copies of every input and
the device->host read of every output inside the timed region.
`--impl reference` times the CPU restatement of the reference path
(oracle/, all host threads) on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "robot-rounds/sec for horizon+schedule decisions"
UNIT = "robot-rounds/s"
R_DEFAULT = 1 << 20
K_DEFAULT = 8192
LP = LC = 50
D = 7
THR = 0.9
# algorithmic bytes per robot-round of the dominant kernel (kr_horizon_divergence):
# prev row block + candidate row block (fp32) + offset (int32) in, horizon (int32) out
DIV_BYTES = (LP + LC) * D * 4 + 4 + 4


def workload_config(args, world):
    return {
        "workload": "configs[4] per-GPU share: 2^20 pending robots/GPU, divergence horizon "
                    "(prev/new chunk 50x7 fp32, overlap offset U[0,10], thr 0.9) + urgency "
                    "(0-5 round histories) + global top-k=8192 admission",
        "robots_per_gpu": args.robots, "global_k": args.k, "chunk": [LP, D], "samples": 1,
        "policy": "kairos B=10 A=5", "parallelism": f"robot-sharded x{world}",
        "l2": "inputs 2.9 GB/GPU > 126 MB L2 (no flush needed)",
        "timing": "CUDA events on the launching stream around K back-to-back rounds; a ~1 ms "
                  "blocking device spin precedes the start event so host enqueue gaps stay "
                  "out of the device time",
    }


# --------------------------------------------------------------------------
# clocks (NVML, sampled during the timed region)
# --------------------------------------------------------------------------
def _clock_poll(index, stop, ready, out):
    """Child process: poll NVML SM clock + throttle reasons until `stop` is set
    (`ready` is set once NVML answers, so the parent starts its timed region
    only after sampling has begun)."""
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(index)
    pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
    ready.set()
    samples, masks = [], 0
    while not stop.is_set():
        try:
            samples.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
            masks |= pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
        except Exception:
            pass
        time.sleep(0.0005)
    out.put((samples, masks, pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)))


class ClockSampler:
    """NVML clock / throttle-reason sampling in a forked process (no GIL
    contention with the launching thread) for the duration of a `with` block."""
    REASONS = {
        0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown",
    }

    def __init__(self, index: int):
        import multiprocessing as mp
        self.ctx = mp.get_context("fork")
        self.index = index
        self.result = ([], 0, None)

    def __enter__(self):
        try:
            import pynvml  # noqa: F401
            self.stop = self.ctx.Event()
            ready = self.ctx.Event()
            self.q = self.ctx.Queue()
            self.proc = self.ctx.Process(target=_clock_poll,
                                         args=(self.index, self.stop, ready, self.q), daemon=True)
            self.proc.start()
            ready.wait(timeout=30)  # NVML initialised and answering
            time.sleep(0.01)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.stop.set()
            try:
                self.result = self.q.get(timeout=10)
            except Exception:
                pass
            self.proc.join(timeout=10)

    def summary(self):
        samples, mask, max_mhz = self.result
        return {"sm_mhz": statistics.median(samples) if samples else None, "sm_max_mhz": max_mhz,
                "reasons": sorted(n for b, n in self.REASONS.items() if mask & b),
                "samples": len(samples)}


def hbm_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic():
    p = ROOT / "profiles" / "ncu_traffic.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d.get("kr_horizon_divergence_bytes_per_launch"), d.get("source")
    return None, None


# --------------------------------------------------------------------------
# CPU baseline / reference arm: the oracle port on the host cores
# --------------------------------------------------------------------------
def cpu_round(R: int, seed: int, nthreads: int):
    """One bounded CPU decision round of R robots with the oracle port:
    returns (seconds, nthreads)."""
    import torch
    from oracle import oracle as orc
    from paper_2605_11381_b200 import synthetic
    soa = synthetic.fleet_soa(R, seed=seed)
    prev, cand, off = synthetic.chunks(R, seed=seed + 1, device="cpu")
    prev, cand, off = prev.numpy(), cand.numpy(), off.numpy()
    t0 = time.perf_counter()
    orc.divergence_batch(prev, cand, THR, off, nthreads=nthreads)
    orc.plan_soa(soa, "kairos", 10, 5, 150_000, 166_667, synthetic.NOW, 30, min(K_DEFAULT, R))
    return time.perf_counter() - t0


def cpu_baseline(target_s: float = 10.0):
    from oracle import oracle as orc
    nthreads = orc.nthreads_default()
    t_small = cpu_round(8192, 5, nthreads)
    R = int(min(R_DEFAULT, max(8192, 8192 * target_s / max(t_small, 1e-6) / 3)))
    times = [cpu_round(R, 7 + i, nthreads) for i in range(3)]
    t = statistics.median(times)
    # the same port on one core (bounded sample)
    t1 = cpu_round(8192, 5, 1)
    R1 = int(min(R_DEFAULT, max(8192, 8192 * (target_s / 3) / max(t1, 1e-6) / 3)))
    t1 = statistics.median([cpu_round(R1, 9 + i, 1) for i in range(3)])
    out = {"value": R / t, "unit": UNIT, "cores": nthreads, "kind": "port",
           "sample": f"{R} robots x 3 rounds (median), oracle/ C port: OpenMP divergence "
                     f"horizon ({nthreads} threads) + serial plan() sort/admission",
           "port_1_thread": {"value": R1 / t1, "unit": UNIT, "cores": 1,
                             "sample": f"{R1} robots x 3 rounds (median), oracle/ C port, 1 thread"}}
    out.update(python_reference_baseline())
    return out


def _ref_objects(kb, soa, R):
    """Reference-package TaskState / PendingRequest objects of the first R
    robots of a synthetic fleet (setup, untimed): histories from the CSR
    slots, task ids whose string order is the robot order."""
    states, pending = {}, []
    for i in range(R):
        tid = f"task-{i:07d}"
        st = kb.TaskState(task_id=tid, t_start=int(soa["t_start"][i]))
        ne, ng, h = int(soa["n_exec"][i]), int(soa["n_gen"][i]), int(soa["hist_off"][i])
        for j in range(max(ne, ng)):
            gs, ge, es, ee = (int(x) for x in soa["slots"][h + j])
            if j < ng:
                st.begin_generation(j, gs)
            if j < ne:
                st.finish_generation(j, ge)
                st.record_execution(j, es, ee, 1)
        st.accumulated_generation = int(soa["accum_gen"][i])
        states[tid] = st
        pending.append(kb.PendingRequest(
            task_id=tid, round_id=ne, issued_at=int(soa["issued_at"][i]),
            obs_captured_at=int(soa["obs_captured_at"][i]),
            last_exec_info=kb.LastExecInfo(0, int(soa["remaining"][i])), payload_bytes=0,
            skipped=int(soa["skipped"][i])))
    return states, pending


_POOL_INPUTS = {}


def _pool_horizons(bounds):
    import roboserve
    lo, hi = bounds
    prev, cand, off = _POOL_INPUTS["prev"], _POOL_INPUTS["cand"], _POOL_INPUTS["off"]
    return [roboserve.round_optimal_horizon(prev[r, off[r]:], cand[r, 0], THR)
            for r in range(lo, hi)]


def python_reference_baseline():
    """the unmodified reference package (vendored under
    baseline/_ref by tools/vendor_reference.sh) on the host cores, on a
    bounded sample of the headline workload: per-robot round_optimal_horizon
    (workload.py:471-496) against the unexecuted overlap + one plan() over the
    sample's pending requests (scheduler.py:254-276).  Mode 1: one process,
    one core.  Mode 2: the horizon steps on a persistent fork pool of
    os.cpu_count() workers sharing the inputs copy-on-write (OPENBLAS 1
    thread), plan() single-process (one global decision).  Median of 3."""
    ref_root = ROOT / "baseline" / "_ref"
    if not (ref_root / "roboserve" / "__init__.py").exists():
        return {"reference_python": {"unavailable": "baseline/_ref not vendored "
                                                    "(tools/vendor_reference.sh)"}}
    import multiprocessing as mp
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    sys.path.insert(0, str(ref_root))
    import roboserve as kb
    from paper_2605_11381_b200 import synthetic
    res = {}
    for mode, R in (("reference_python_1core", 2048), ("reference_python_pool", 16384)):
        soa = synthetic.fleet_soa(R, seed=31)
        prev, cand, off = synthetic.chunks(R, seed=32, device="cpu")
        prev, cand = prev.double().numpy(), cand.double().numpy()
        off = off.numpy()
        states, pending = _ref_objects(kb, soa, R)
        edge = kb.EngineProfile(tier="edge", capacity=min(K_DEFAULT, R), max_batch=1,
                                points=((1, 100_000),))
        cfg = kb.SchedulerConfig()
        pool = None
        if mode.endswith("pool"):
            _POOL_INPUTS.update(prev=prev, cand=cand, off=off)
            workers = os.cpu_count() or 1
            pool = mp.get_context("fork").Pool(workers)
            step = (R + workers - 1) // workers
            chunks = [(lo, min(R, lo + step)) for lo in range(0, R, step)]
            pool.map(_pool_horizons, chunks)  # warm the workers
        times = []
        for _ in range(3):
            for st in states.values():
                st.skipped = 0
            t0 = time.perf_counter()
            if pool is None:
                for r in range(R):
                    kb.round_optimal_horizon(prev[r, off[r]:], cand[r, 0], THR)
            else:
                pool.map(_pool_horizons, chunks)
            kb.plan(pending, states, edge, None, None, synthetic.NOW, cfg)
            times.append(time.perf_counter() - t0)
        if pool is not None:
            pool.close()
            pool.join()
        t = statistics.median(times)
        res[mode] = {"value": R / t, "unit": UNIT, "cores": 1 if pool is None else workers,
                     "sample": f"{R} robots: round_optimal_horizon per robot + one plan() of "
                               f"{R} pending (k={min(K_DEFAULT, R)}), unmodified roboserve, "
                               f"median of 3"}
    return res


def run_reference(args, world, rank):
    if rank != 0:
        return
    from oracle import oracle as orc
    nthreads = orc.nthreads_default()
    R = args.ref_robots
    for i in range(args.warmup):
        cpu_round(R, 100 + i, nthreads)
    times = [cpu_round(R, 200 + i, nthreads) for i in range(args.steps)]
    total = sum(times)
    value = R * args.steps / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {**workload_config(args, world),
                   "reference_arm": f"oracle C port of the reference path (oracle/kairos_oracle.c, "
                                    f"{nthreads} host threads: OpenMP divergence + serial plan), "
                                    f"not the Python roboserve package; the unmodified package is "
                                    f"timed in our arm's cpu_baseline.reference_python_*"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": nthreads, "kind": "port",
                         "sample": f"{R} robots per step (bounded sample of the per-GPU "
                                   f"workload), oracle/ C restatement of the reference path"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------
# our arm
# --------------------------------------------------------------------------
def run_ours(args, world, rank, local_rank):
    import torch
    import torch.distributed as dist
    from paper_2605_11381_b200 import _lib, fleet as fl, rounds, synthetic

    torch.cuda.set_device(local_rank)
    lib = _lib.load()
    R = args.robots
    soa = synthetic.fleet_soa(R, seed=1000 + rank, rank_offset=rank * R)
    fleet = fl.DeviceFleet.from_host(soa)
    prev, cand, off = synthetic.chunks(R, seed=2000 + rank)
    base = synthetic.NOW - (1 << 39)
    sched = fl.sched_struct("kairos", 10, 5, 150_000, 166_667, synthetic.NOW, 30, base)
    if world > 1 or args.force_sharded:
        rnd = rounds.ShardedDecisionRound(R, args.k, sched)
    else:
        rnd = rounds.DecisionRound(R, args.k, sched)
    inputs = rounds.DivergenceInputs(prev, cand, THR, offset=off)
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # CUDA graphs at every N: the sharded round's NCCL all-gather is captured
    # inside the admission graph (rounds.ShardedDecisionRound.capture)
    graphs = not args.no_graph and not args.eager
    # --eager: the same overlap with eager launches
    overlap = not graphs and args.reserve_sms > 0 and not args.no_graph
    n_cap0 = lib.kr_launch_count()
    capture_error = None
    if graphs:
        # CUDA graphs: horizons | urgency + admission, the latter on a side
        # stream over `reserve_sms` SMs left free by the horizon kernel
        try:
            rnd.capture(fleet, inputs, reserve_sms=args.reserve_sms, layout=args.layout)
            per_round = (lib.kr_launch_count() - n_cap0) // 2  # warm-up run + capture
        except Exception as e:  # noqa: BLE001 -- a capture failure falls back to eager launches
            capture_error = f"{type(e).__name__}: {e}"[:200]
            torch.cuda.synchronize()
            graphs, overlap = False, args.reserve_sms > 0
    for _ in range(args.warmup):
        if graphs:
            rnd.replay()
        elif overlap:
            rnd.run_overlapped(fleet, inputs, args.reserve_sms, layout=args.layout)
        else:
            rnd.run(fleet, inputs)
    barrier()

    # timed region: K whole rounds; divergence kernel bracketed by events
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    sev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n0 = lib.kr_launch_count()
    with ClockSampler(local_rank) as clk:
        barrier()
        # nvbench-style blocking kernel: a ~1 ms device spin ahead of the start
        # event, so the host enqueues the first rounds while the GPU is busy and
        # the timed region holds the K rounds' device work back to back (without
        # it, K = 5 read 0.56 ms per round against 0.505 at K = 50: host launch
        # gaps, not device time)
        torch.cuda._sleep(2_000_000)  # on `stream` (the current stream)
        start.record(stream)
        for i in range(args.steps):
            if graphs:
                rnd.replay_concurrent(before_horizon=ev[i][0].record, after_horizon=ev[i][1].record,
                                      before_side=sev[i][0].record, after_side=sev[i][1].record)
            elif overlap:
                rnd.run_overlapped(fleet, inputs, args.reserve_sms, before_horizon=ev[i][0].record,
                                   after_horizon=ev[i][1].record, layout=args.layout)
            else:
                ev[i][0].record(stream)
                rnd.horizons(inputs)
                ev[i][1].record(stream)
                rnd.urgency(fleet)
                rnd.admit(fleet)
        end.record(stream)
        barrier()
    launches = per_round * args.steps if graphs else lib.kr_launch_count() - n0
    rnd.check()  # validation word of every timed round (key ranges, shard key uniqueness)
    elapsed = start.elapsed_time(end) / 1e3
    div_ms = [a.elapsed_time(b) for a, b in ev]
    t = torch.tensor([elapsed], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    elapsed = float(t.item())
    value = R * world * args.steps / elapsed

    # kernel breakdown of one extra round (events between the three steps)
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    e[0].record(stream); rnd.horizons(inputs); e[1].record(stream)
    rnd.urgency(fleet); e[2].record(stream); rnd.admit(fleet); e[3].record(stream)
    torch.cuda.synchronize()
    breakdown = {"horizon_divergence_ms": e[0].elapsed_time(e[1]),
                 "urgency_ms": e[1].elapsed_time(e[2]), "admission_ms": e[2].elapsed_time(e[3]),
                 "note": "one eager (non-graph) round; launch-rate bound for the small kernels"}
    if graphs:
        gd = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        gd[0].record(stream); rnd.g_decide.replay(); gd[1].record(stream)
        torch.cuda.synchronize()
        breakdown["urgency_plus_admission_graph_ms"] = gd[0].elapsed_time(gd[1])
        if args.reserve_sms != 0:  # the side stream inside the timed rounds (concurrent)
            breakdown["side_stream_ms_in_round"] = statistics.mean(
                a.elapsed_time(b) for a, b in sev)
        breakdown["reserve_sms"] = args.reserve_sms
        breakdown["layout"] = args.layout

    e2e, e2e_cold = run_e2e(args, world, soa, prev, cand, off, sched) if not args.no_e2e else (None, None)

    if rank != 0:
        return
    peak, peak_src = hbm_peak()
    div_avg_s = statistics.mean(div_ms) / 1e3
    achieved = DIV_BYTES * R / div_avg_s / 1e9
    traffic, traffic_src = ncu_traffic()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * elapsed / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded: fleet histories + N(0,1) action chunks, SURVEY.md 8d)",
        "config": workload_config(args, world),
        "roofline": {"bound": "hbm", "kernel": "kr_horizon_divergence", "achieved": achieved,
                     "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "peak_source": peak_src,
                     "algorithmic_bytes_per_robot_round": DIV_BYTES,
                     "launch_ms_mean": statistics.mean(div_ms),
                     "traffic_source": traffic_src},
        "round_roofline": round_roofline(soa, R, elapsed / args.steps, peak),
        "kernels": breakdown,
        "gpu_launches": int(launches),
        "cuda_graphs": bool(graphs) if capture_error is None else f"capture failed ({capture_error}); eager",
        "concurrency": ((f"urgency on the whole GPU, then " if args.layout == "urgency_first" else "")
                        + f"{'admission' if args.layout == 'urgency_first' else 'urgency + admission'}"
                        f"{' + NCCL candidate all-gather' if world > 1 else ''} on a side stream over "
                        f"{args.reserve_sms} SMs reserved from the horizon kernel"
                        if (graphs or overlap) and args.reserve_sms > 0 else None),
        "clocks": clk.summary(),
    }
    if e2e:
        line["e2e"] = e2e
        line["e2e_cold"] = e2e_cold
    if world == 1 and not args.no_configs:
        line["other_configs"] = other_configs()
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args.cpu_seconds)
    print(json.dumps(line), flush=True)


def _timed(step, steps, world):
    import torch
    import torch.distributed as dist
    for _ in range(2):
        step(0)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for i in range(steps):
        step(i)
    e.record()
    torch.cuda.synchronize()
    el = torch.tensor([s.elapsed_time(e) / 1e3], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(el, op=dist.ReduceOp.MAX)
    return float(el.item())


def round_roofline(soa, R, t_round, peak):
    """The whole round against HBM: algorithmic bytes of every step (horizon
    2,808 B + urgency's fleet fields, history slots and outputs + admission's
    key / observation / skip-counter / mask traffic) over the measured round
    time -- the horizon kernel shares HBM with the concurrent side stream, so
    its own fraction understates how busy the memory system is."""
    slots = int(np.maximum(soa["n_exec"], soa["n_gen"]).sum())
    urg = R * (8 * 3 + 4 * 5) + slots * 32 + R * (16 + 8)  # fields in, history, key + need out
    adm = R * (16 + 8 + 4 + 4 + 2)  # key, obs, skipped RMW, admitted + refetch masks
    total = R * DIV_BYTES + urg + adm
    gbs = total / t_round / 1e9
    return {"bytes_per_robot_round": total / R, "achieved": gbs, "peak": peak, "unit": "GB/s",
            "frac": gbs / peak,
            "note": "horizon + urgency + admission bytes of one round over the round time"}


def other_configs(reps: int = 200):
    """The other BASELINE.json configs on this GPU, each one whole decision
    round (horizons + urgency + top-k admission) replayed from CUDA graphs,
    in the concurrent "split" layout (horizons || urgency + admission) where
    it pays, with the reserved-SM count measured best per size
    (profiles/r1_small_layouts.jsonl, tools/small_layouts.py).
    configs[1] and [2] are L2-resident (labelled); configs[3] streams from HBM.
    configs[0] (the paper's Fig. 4 scenario) is a correctness case
    (tests/test_gpu_scheduler.py), configs[4] is the headline above."""
    import torch
    from paper_2605_11381_b200 import _lib, device as dev, fleet as fl, rounds, synthetic

    lib = _lib.load()
    out = {}

    def timed_captured(rnd, fleet, inp, reserve, layout="split"):
        rnd.capture(fleet, inp, reserve_sms=reserve, layout=layout)
        for _ in range(10):
            rnd.replay()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        for _ in range(reps):
            rnd.replay()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / 1e3 / reps

    def sched_for(soa):
        return fl.sched_struct("kairos", 10, 5, 150_000, 166_667, synthetic.NOW, 30,
                               int(soa["issued_at"].min()))

    # configs[1]: 1k robots, 50x7 @ 30 Hz, k = 64
    R = 1024
    soa = synthetic.fleet_soa(R, seed=11)
    fleet = fl.DeviceFleet.from_host(soa)
    prev, cand, off = synthetic.chunks(R, seed=12)
    rnd = rounds.DecisionRound(R, 64, sched_for(soa))
    inp = rounds.DivergenceInputs(prev, cand, THR, offset=off)
    t = timed_captured(rnd, fleet, inp, 0)
    out["configs[1] 1k robots 50x7 k=64"] = {
        "us_per_round": 1e6 * t, "robot_rounds_per_s": R / t, "l2": "resident (0.3 MB inputs)",
        "layout": "sequential, one graph per round with programmatic dependent launches "
                  "(at 1k robots a second stream costs more than it hides)"}
    # configs[2]: 16k mixed fleet, two homogeneous tensors, 64-step chunks, k = 1024
    R = 16384
    soa = synthetic.fleet_soa(R, seed=13)
    fleet = fl.DeviceFleet.from_host(soa)
    pa, ca, oa = synthetic.chunks(R // 2, seed=14, Lp=64, Lc=64, D=7)
    ph, chh, oh = synthetic.chunks(R // 2, seed=15, Lp=64, Lc=64, D=32)
    rnd = rounds.DecisionRound(R, 1024, sched_for(soa))
    inp = rounds.MixedInputs([(0, rounds.DivergenceInputs(pa, ca, THR, offset=oa)),
                              (R // 2, rounds.DivergenceInputs(ph, chh, THR, offset=oh))])
    t = timed_captured(rnd, fleet, inp, 8)
    out["configs[2] 16k mixed (8k arms 64x7 + 8k humanoids 64x32) k=1024"] = {
        "us_per_round": 1e6 * t, "robot_rounds_per_s": R / t,
        "l2": "163 MB of chunks (> 126 MB L2): mostly streamed from HBM",
        "layout": "split, 8 reserved SMs: the two groups' horizon kernels on forked streams || "
                  "urgency + admission"}
    # configs[3]: 64k robots, 8-sample ensembles 50x7, k = 8192 (one GPU's whole fleet)
    R = 65536
    soa = synthetic.fleet_soa(R, seed=16)
    fleet = fl.DeviceFleet.from_host(soa)
    prev, cand, off = synthetic.chunks(R, seed=17, S=8)
    rnd = rounds.DecisionRound(R, 8192, sched_for(soa))
    inp = rounds.DivergenceInputs(prev, cand, THR, offset=off)
    t = timed_captured(rnd, fleet, inp, 1)
    out["configs[3] 64k robots S=8 ensembles 50x7 k=8192"] = {
        "us_per_round": 1e6 * t, "robot_rounds_per_s": R / t,
        "l2": "streams from HBM (826 MB inputs)", "layout": "split, 1 reserved SM"}
    # the headline fleet with the confidence policy (paper default t=0.4, H_min=5)
    from paper_2605_11381_b200 import HorizonPolicyConfig
    R = 1 << 20
    soa = synthetic.fleet_soa(R, seed=18)
    fleet = fl.DeviceFleet.from_host(soa)
    U = synthetic.magnitudes(R, seed=19)
    rnd = rounds.DecisionRound(R, 8192, sched_for(soa))
    inp = rounds.ConfidenceInputs(U, HorizonPolicyConfig.confidence(0.4, 5))
    # horizons || urgency + admission, 8 reserved SMs (median of four
    # interleaved repeats per layout on two boxes: split/8 249.8-250.1 us,
    # split/16 257.0-260.5, urgency first/1 259.3-262.1; tools/conf_layout_reps.py)
    t = timed_captured(rnd, fleet, inp, 8)
    out["configs[4] per-GPU share, confidence policy (U 2^20 x 6 x 50 fp32), k=8192"] = {
        "us_per_round": 1e6 * t, "robot_rounds_per_s": R / t,
        "l2": "streams from HBM (1.26 GB of magnitudes)",
        "layout": "split: horizons || urgency + admission (8 reserved SMs)"}
    # fp64 storage (the reference's native dtype, workload.py:485-486): the
    # headline divergence round and the confidence round, same layouts
    R = 1 << 20
    soa = synthetic.fleet_soa(R, seed=23)
    fleet = fl.DeviceFleet.from_host(soa)
    prev, cand, off = synthetic.chunks(R, seed=24, dtype=torch.float64)
    rnd = rounds.DecisionRound(R, 8192, sched_for(soa))
    t = timed_captured(rnd, fleet, rounds.DivergenceInputs(prev, cand, THR, offset=off), 2)
    out["configs[4] per-GPU share, fp64 chunks (50x7 fp64), k=8192"] = {
        "us_per_round": 1e6 * t, "robot_rounds_per_s": R / t,
        "l2": "streams from HBM (5.9 GB of chunks)", "layout": "split, 2 reserved SMs",
        "round_GBps": (DIV_BYTES * 2 - 8) * R / t / 1e9}
    del prev, cand
    U = synthetic.magnitudes(R, seed=25, dtype=torch.float64)
    rnd = rounds.DecisionRound(R, 8192, sched_for(soa))
    # horizons || urgency + admission, 16 reserved SMs (median of four
    # interleaved repeats: split/16 398 us, urgency first/4 442 us, split/2
    # 498 us; tools/conf_layout_reps.py CONF_DT=64)
    t = timed_captured(rnd, fleet, rounds.ConfidenceInputs(
        U, HorizonPolicyConfig.confidence(0.4, 5)), 16)
    out["configs[4] per-GPU share, confidence policy fp64 (U 2^20 x 6 x 50 fp64), k=8192"] = {
        "us_per_round": 1e6 * t, "robot_rounds_per_s": R / t,
        "l2": "streams from HBM (2.5 GB of magnitudes)",
        "layout": "split: horizons || urgency + admission (16 reserved SMs)"}
    del U
    # the headline fleet with a cloud tier (phase 3 at fleet scale, §8(f)1):
    # full key order + edge admission + the ordered offload scan
    import numpy as np
    from paper_2605_11381_b200 import engines as eng
    R, k = 1 << 20, 8192
    soa = synthetic.fleet_soa(R, seed=20)
    fleet = fl.DeviceFleet.from_host(soa)
    prev, cand, off = synthetic.chunks(R, seed=21)
    edge = eng.EngineProfile(tier="edge", capacity=k, max_batch=256,
                             points=((1, 150_000), (256, 400_000)))
    cloud = eng.EngineProfile(tier="cloud", capacity=2048, max_batch=512,
                              points=((1, 80_000), (512, 250_000)))
    net = eng.NetworkModel(base_latency_us=20_000, uplink_bps=400_000_000,
                           downlink_bps=1_000_000_000)
    rnd = rounds.HybridDecisionRound(R, k, sched_for(soa), cloud.capacity)
    payload = torch.from_numpy(np.random.default_rng(22).choice(
        np.array([100_000, 300_000, 2_000_000], np.int64), R)).cuda()
    rnd.set_cloud(eng.transfer_time_batch(net, payload, eng.UP),
                  eng.cloud_thresholds(edge, cloud, net, 0, 0, k, rnd.cap))
    inp = rounds.DivergenceInputs(prev, cand, THR, offset=off)
    # eager (the offload scan reads its slot count back: one sync), overlapped
    # like the graph rounds: urgency, then horizons || the admission side stream
    # (tests/test_gpu_hybrid_round.py: identical decisions to the sequential round)
    step = lambda: rnd.run_overlapped(fleet, inp, reserve_sms=10, layout="urgency_first")
    for _ in range(5):
        step()
    torch.cuda.synchronize()
    n_cloud = int(rnd.n_cloud.item())
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps // 4):
        step()
    b.record()
    torch.cuda.synchronize()
    t = a.elapsed_time(b) / 1e3 / (reps // 4)
    out["configs[4] per-GPU share with a cloud tier (k=8192 edge, 2048 cloud slots)"] = {
        "us_per_round": 1e6 * t, "robot_rounds_per_s": R / t, "cloud_placed": n_cloud,
        "full_sorts": rnd.full_sorts,
        "layout": "eager, overlapped: urgency, then horizons (138 SMs) || ordered top k + 4096 "
                  "(fused select), edge admission, ordered offload scan, one 4-byte read of the "
                  "slot count (rounds.HybridDecisionRound.run_overlapped)"}
    return out


def run_e2e(args, world, soa, prev, cand, off, sched):
    """The round through the C ABI from pinned host buffers, copies timed.

    Streaming (the headline `e2e`): in a serving loop a round's host inputs are
    the new action chunk and the per-request scalars that change every round
    (issued_at, obs_captured_at, remaining actions, overlap offset); the
    previous chunk is the last round's new chunk and the fleet history are
    already device-resident.  Each step copies one new chunk (alternating two
    host chunk sets, so the compared trajectories differ) and those scalars,
    runs the round, and reads back horizons, need times, admitted / refetch
    masks, skip counters and the ordered S_e.
    Cold (`e2e_cold`): every input of the round, history included, is copied."""
    import torch
    from paper_2605_11381_b200 import fleet as fl, rounds

    R = args.robots
    graphs = not args.no_graph  # the sharded round's NCCL all-gather is captured too
    rnd = (rounds.ShardedDecisionRound(R, args.k, sched) if world > 1
           else rounds.DecisionRound(R, args.k, sched))
    outs = {"H": torch.empty(R, dtype=torch.int32).pin_memory(),
            "need": torch.empty(R, dtype=torch.int64).pin_memory(),
            "adm": torch.empty(R, dtype=torch.uint8).pin_memory(),
            "ref": torch.empty(R, dtype=torch.uint8).pin_memory(),
            "skip": torch.empty(R, dtype=torch.int32).pin_memory(),
            "edge": torch.empty((max(rnd.k, 1), 2), dtype=torch.int64).pin_memory()}
    d2h = sum(t.numel() * t.element_size() for t in outs.values())

    def read_back(o, fleet):
        outs["H"].copy_(o.horizon, non_blocking=True)
        outs["need"].copy_(o.need_time, non_blocking=True)
        outs["adm"].copy_(o.admitted, non_blocking=True)
        outs["ref"].copy_(o.refetch, non_blocking=True)
        outs["skip"].copy_(fleet.t["skipped"], non_blocking=True)
        outs["edge"][: o.edge_keys.shape[0]].copy_(o.edge_keys, non_blocking=True)

    # ---- streaming rounds (pipelined) ----
    # The next step's H2D runs on a copy stream while this step computes and
    # reads back: device chunks rotate through a ring of three (new, prev, and
    # the one being filled) and the per-request scalars through two staging
    # sets, each with its own fleet view (history and skip counters shared) and
    # its own captured graphs, so no device-to-device copy queues behind the
    # next step's transfer.  Every step still moves its own inputs in and its
    # results out inside the timed region.
    h_chunks = [cand[:, 0].cpu().pin_memory(), prev.cpu().pin_memory()]  # alternate A, B
    ring = [torch.empty_like(prev) for _ in range(3)]
    fleet = fl.DeviceFleet.from_host(soa)
    per_round = ("issued_at", "obs_captured_at", "remaining")
    h_sc = {k: torch.from_numpy(np.ascontiguousarray(soa[k])).pin_memory() for k in per_round}
    h_off = off.cpu().pin_memory()
    d_off = torch.empty_like(off)
    stage = [{k: fleet.t[k] if si == 0 else torch.empty_like(fleet.t[k]) for k in per_round}
             for si in range(2)]
    stage_off = [d_off, torch.empty_like(off)]
    views = [fl.DeviceFleet.from_tensors({**fleet.t, **stage[si]}) for si in range(2)]
    inp6 = [[rounds.DivergenceInputs(ring[(a + 2) % 3], ring[a], THR, offset=stage_off[si])
             for si in range(2)] for a in range(3)]
    if graphs:
        rnd.run(views[0], inp6[0][0])
        torch.cuda.synchronize()
        try:
            g_h = [[torch.cuda.CUDAGraph() for _ in range(2)] for _ in range(3)]
            for a in range(3):
                for si in range(2):
                    with torch.cuda.graph(g_h[a][si]):
                        rnd.horizons(inp6[a][si])
            g_d = [torch.cuda.CUDAGraph() for _ in range(2)]
            for si in range(2):
                with torch.cuda.graph(g_d[si]):
                    rnd.urgency(views[si])
                    rnd.admit(views[si])
        except Exception:  # noqa: BLE001 -- capture failure: eager launches
            torch.cuda.synchronize()
            graphs = False
    cs = torch.cuda.current_stream()
    xs = torch.cuda.Stream()

    def run_steps(steps, start_evt):
        h2d = [torch.cuda.Event() for _ in range(steps)]
        done = [torch.cuda.Event() for _ in range(steps)]
        for i in range(steps):
            a, si = i % 3, i % 2
            with torch.cuda.stream(xs):
                if i == 0:
                    xs.wait_event(start_evt)
                if i >= 2:  # ring slot / staging set last read by step i - 2
                    xs.wait_event(done[i - 2])
                ring[a].copy_(h_chunks[i & 1], non_blocking=True)
                stage_off[si].copy_(h_off, non_blocking=True)
                for k, v in h_sc.items():
                    stage[si][k].copy_(v, non_blocking=True)
                h2d[i].record(xs)
            cs.wait_event(h2d[i])
            if graphs:
                g_h[a][si].replay()
                g_d[si].replay()
                o = rnd.outputs()
            else:
                o = rnd.run(views[si], inp6[a][si])
            read_back(o, views[si])
            done[i].record(cs)

    h2d_stream = h_chunks[0].numel() * 4 + h_off.numel() * 4 + sum(
        v.numel() * v.element_size() for v in h_sc.values())
    steps = max(2, min(args.steps, args.e2e_steps))
    ring[2].copy_(h_chunks[1])  # the previous chunk of step 0 (last round's, resident)
    w0 = torch.cuda.Event()
    w0.record(cs)
    run_steps(2, w0)  # warm-up
    ring[2].copy_(h_chunks[1])
    torch.cuda.synchronize()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    s0, e0 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record(cs)
    run_steps(steps, s0)
    e0.record(cs)
    torch.cuda.synchronize()
    el = torch.tensor([s0.elapsed_time(e0) / 1e3], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(el, op=dist.ReduceOp.MAX)
    t = float(el.item())
    stream = {"value": R * world * steps / t, "unit": UNIT, "h2d_bytes_per_step": int(h2d_stream),
              "d2h_bytes_per_step": int(d2h), "steps": steps, "ms_per_step": 1e3 * t / steps,
              "path": "streaming round through the C ABI: pinned host -> H2D of the new chunk "
                      "[R,50,7] fp32 + per-request scalars (issued_at, obs_captured_at, remaining, "
                      "offset); previous chunk (last round's) and fleet history device-resident; "
                      "D2H of horizons, need times, masks, skip counters, ordered S_e; the next "
                      "step's H2D (copy stream) overlaps this step's compute and D2H"}

    # ---- cold rounds: every input copied ----
    h_prev, h_cand = prev.cpu().pin_memory(), cand.cpu().pin_memory()
    h_soa = {k: torch.from_numpy(np.ascontiguousarray(soa[k])).pin_memory()
             for k in fl.INT_FIELDS64 + fl.INT_FIELDS32 + ("slots",)}
    d_prev, d_cand = torch.empty_like(prev), torch.empty_like(cand)
    d_soa = {k: torch.empty(v.shape, dtype=v.dtype, device="cuda") for k, v in h_soa.items()}
    cfleet = fl.DeviceFleet.from_tensors(d_soa)
    cinp = rounds.DivergenceInputs(d_prev, d_cand, THR, offset=d_off)

    def cold_step(i):
        d_prev.copy_(h_prev, non_blocking=True)
        d_cand.copy_(h_cand, non_blocking=True)
        d_off.copy_(h_off, non_blocking=True)
        for k, v in h_soa.items():
            d_soa[k].copy_(v, non_blocking=True)
        read_back(rnd.run(cfleet, cinp), cfleet)

    h2d_cold = sum(t_.numel() * t_.element_size() for t_ in [h_prev, h_cand, h_off, *h_soa.values()])
    t = _timed(cold_step, steps, world)
    cold = {"value": R * world * steps / t, "unit": UNIT, "h2d_bytes_per_step": int(h2d_cold),
            "d2h_bytes_per_step": int(d2h), "steps": steps, "ms_per_step": 1e3 * t / steps,
            "path": "every input of the round (both chunks, all fleet state and history) copied "
                    "from pinned host each step; eager launches"}
    return stream, cold


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--robots", type=int, default=R_DEFAULT)
    ap.add_argument("--k", type=int, default=K_DEFAULT)
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--eager", action="store_true",
                    help="N=1: the N>1 path (eager launches, side-stream overlap) instead of graphs")
    ap.add_argument("--reserve-sms", type=int, default=2,
                    help="SMs left to urgency + admission (side stream) during the horizon "
                         "kernel (tools/reserve_sweep.sh; the sharded round with its NCCL "
                         "all-gather on the side stream: --force-sharded 0.467 ms at 2, "
                         "0.480 ms at 10)")
    ap.add_argument("--layout", choices=["split", "urgency_first"], default="split",
                    help="graph layout of the round (see rounds.DecisionRound.capture)")
    ap.add_argument("--force-sharded", action="store_true",
                    help="diagnostic: the N>1 sharded round (local select, all-gather, global "
                         "select) on a one-rank process group")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-configs", action="store_true",
                    help="skip the other BASELINE configs' round latencies")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--ref-robots", type=int, default=16384)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, world, rank)
        return
    if world > 1 or args.force_sharded:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29531")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, world, rank, local_rank)
    finally:
        if world > 1 or args.force_sharded:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
