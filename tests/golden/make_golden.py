"""Generate the golden parity fixtures by running the REFERENCE itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the unmodified reference package `roboserve` from
/root/reference/pkg/src, feeds it seeded synthetic inputs for every hot-path
function (horizon.py:108-132, workload.py:461-496, core.py:31-47/157-166,
waiting.py:46-100, scheduler.py:79-276, pkg/scratch_fig4.py) and stores the
inputs together with the reference's outputs under tests/golden/.  The
fixtures are what pins both the CPU oracle (oracle/) and the CUDA path; the
GPU box never needs /root/reference.
"""

from __future__ import annotations

import contextlib
import io
import json
import os
import runpy
import sys
from pathlib import Path

import numpy as np

sys.dont_write_bytecode = True
REF_SRC = "/root/reference/pkg/src"
REF_PKG = "/root/reference/pkg"
sys.path.insert(0, REF_SRC)

from roboserve import core, horizon, scheduler, waiting, workload  # noqa: E402
from roboserve.core import Interval, LastExecInfo, PendingRequest, TaskState  # noqa: E402
from roboserve.engines import EngineProfile, NetworkModel  # noqa: E402

OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(OUT.parent))
import golden_io  # noqa: E402  (tests/golden_io.py: shared fixture helpers)


# --- step 1a: confidence horizon -------------------------------------------

def gen_confidence(rng: np.random.Generator):
    cases = []

    def add(u, t, hmin):
        mags = horizon.UpdateMagnitudes(u)
        cfg = horizon.HorizonPolicyConfig.confidence(threshold=float(t), min_horizon=int(hmin))
        cases.append((mags.u.copy(), float(t), int(hmin), horizon.decide_horizon(cfg, mags)))

    # synthesized rounds: the reference's own magnitude model (workload.py:341-359)
    for _ in range(700):
        K = int(rng.integers(2, 11))
        N = int(rng.choice([1, 2, 3, 7, 16, 31, 50, 64]))
        spec = workload.SyntheticSpec(chunk_size=N, diffusion_steps=K,
                                      uncertain_fraction=float(rng.uniform(0, 0.5)))
        u = workload._synth_round_magnitudes(spec, rng).u
        if rng.random() < 0.5:
            u = u.astype(np.float32).astype(np.float64)   # fp32-storable
        t = float(rng.choice([0.0, 0.2, 0.4, 0.8, 1.0, rng.uniform(0, 2)]))
        add(u, t, int(rng.integers(1, 9)))
    # bump == (1 + t) exactly: f = 1.8 * mean vs 1.8 * mean -> bit-level tie
    for _ in range(100):
        N = int(rng.integers(8, 65))
        spec = workload.SyntheticSpec(chunk_size=N, diffusion_steps=6, uncertain_fraction=0.4)
        add(workload._synth_round_magnitudes(spec, rng).u, 0.8, 1)
    # wide dynamic range, zeros, ties, N == 1 with long pairwise sums
    for _ in range(300):
        K = int(rng.integers(2, 8))
        N = int(rng.integers(1, 40))
        u = rng.uniform(0, 1, (K, N)) * 10.0 ** rng.uniform(-6, 6, (K, N))
        u[rng.random((K, N)) < 0.15] = 0.0
        if rng.random() < 0.3:
            u[-1] = u[:-1].mean(axis=0) * rng.choice([1.0, 1.4, 1.5])
        add(u.astype(np.float32).astype(np.float64), float(rng.choice([0.0, 0.4, 0.5])),
            int(rng.integers(1, 4)))
    for K in list(range(2, 40)) + [64, 129, 130, 200, 300]:
        u = rng.uniform(0, 1, (K, 1)) * 10.0 ** rng.uniform(-5, 5, (K, 1))
        add(u, float(rng.uniform(0, 1)), 1)
    return cases


def save_confidence(cases):
    shapes = np.array([c[0].shape for c in cases], np.int64)
    offs = np.concatenate([[0], np.cumsum(shapes[:, 0] * shapes[:, 1])]).astype(np.int64)
    np.savez_compressed(
        OUT / "horizon_confidence.npz",
        u=np.concatenate([c[0].ravel() for c in cases]), shapes=shapes, offsets=offs,
        threshold=np.array([c[1] for c in cases]), min_horizon=np.array([c[2] for c in cases]),
        expected=np.array([c[3] for c in cases], np.int64))


# --- step 1a': threshold sweep (horizon.py:135-151) --------------------------

def gen_sweep(rng: np.random.Generator):
    """Sequences of rounds (mixed shapes within a sequence) x configuration
    lists (static and confidence, duplicates, more than 64 configurations),
    with the reference's sweep_thresholds means."""
    cases = []
    for i in range(48):
        n = int(rng.integers(1, 41))
        shapes = [(int(rng.integers(2, 9)), int(rng.choice([1, 7, 50, 64])))]
        if rng.random() < 0.4:
            shapes.append((6, 50))
        seq = []
        for _ in range(n):
            K, N = shapes[int(rng.integers(0, len(shapes)))]
            spec = workload.SyntheticSpec(chunk_size=N, diffusion_steps=K,
                                          uncertain_fraction=float(rng.uniform(0, 0.5)))
            u = workload._synth_round_magnitudes(spec, rng).u
            if rng.random() < 0.5:
                u = u.astype(np.float32).astype(np.float64)
            seq.append(horizon.UpdateMagnitudes(u))
        C = int(rng.choice([1, 3, 8, 17, 64, 70]))
        cfgs = []
        for _ in range(C):
            if rng.random() < 0.2:
                cfgs.append(horizon.HorizonPolicyConfig.static(int(rng.integers(1, 80))))
            else:
                t = float(rng.choice([0.0, 0.2, 0.4, 0.8, 1.0, rng.uniform(0, 2)]))
                cfgs.append(horizon.HorizonPolicyConfig.confidence(t, int(rng.integers(1, 9))))
        cases.append((seq, cfgs, horizon.sweep_thresholds(cfgs, seq)))
    return cases


def save_sweep(cases):
    us, shapes, seq_off, kinds, sh, thr, hmin, cfg_off, exp = [], [], [0], [], [], [], [], [0], []
    for seq, cfgs, means in cases:
        for m in seq:
            us.append(m.u.ravel())
            shapes.append(m.u.shape)
        seq_off.append(len(shapes))
        for c in cfgs:
            kinds.append(int(c.kind == horizon.CONFIDENCE_THRESHOLD))
            sh.append(c.static_h)
            thr.append(c.threshold)
            hmin.append(c.min_horizon)
        cfg_off.append(len(kinds))
        exp.extend(means)
    shapes = np.array(shapes, np.int64)
    offs = np.concatenate([[0], np.cumsum(shapes[:, 0] * shapes[:, 1])]).astype(np.int64)
    np.savez_compressed(OUT / "sweep.npz", u=np.concatenate(us), shapes=shapes, offsets=offs,
                        seq_off=np.array(seq_off, np.int64), kind=np.array(kinds, np.int64),
                        static_h=np.array(sh, np.int64), threshold=np.array(thr),
                        min_horizon=np.array(hmin, np.int64),
                        cfg_off=np.array(cfg_off, np.int64), expected=np.array(exp))


# --- step 1b: divergence horizon + cosine scores ----------------------------

def gen_divergence(rng: np.random.Generator):
    cases = []
    for ci in range(420):
        D = int(rng.choice([1, 2, 3, 4, 7, 8, 12, 15, 16, 17, 20, 24, 31, 32, 33, 40, 48, 64]))
        Lr = int(rng.integers(1, 41))
        Lc = Lr if rng.random() < 0.7 else int(rng.integers(1, 41))
        ref = rng.normal(0, 1, (Lr, D)) * 10.0 ** rng.uniform(-3, 3)
        L = max(Lr, Lc)
        noise = rng.normal(0, 1, (L, D)) * (0.3 * np.arange(1, L + 1)[:, None] / L)
        cand = np.zeros((Lc, D))
        m = min(Lr, Lc)
        cand[:m] = ref[:m] + noise[:m] * np.abs(ref[:m]).mean()
        if Lc > m:
            cand[m:] = rng.normal(0, 1, (Lc - m, D))
        if rng.random() < 0.1:
            ref[rng.integers(0, Lr)] = 0.0
        if rng.random() < 0.1:
            cand[rng.integers(0, Lc)] = 0.0
        if rng.random() < 0.5:
            ref = ref.astype(np.float32).astype(np.float64)
            cand = cand.astype(np.float32).astype(np.float64)
        cos = np.array([workload._cosine(cand[i], ref[i]) for i in range(m)])
        if ci % 5 == 0 and m > 1:
            thr = float(cos[int(rng.integers(0, m))])     # exact tie: cos == thr passes
            thr = min(1.0, max(thr, 1e-3)) if thr > 0 else 0.5
        else:
            thr = float(rng.choice([0.9, 0.95, 0.99, rng.uniform(0.05, 1.0), 1.0]))
        h = workload.round_optimal_horizon(ref, cand, thr)
        cases.append((ref, cand, thr, h, cos))
    # reference test-suite shapes (tests/test_workload.py:211-229)
    return cases


def save_divergence(cases, name="divergence.npz"):
    rs = np.array([c[0].shape for c in cases], np.int64)
    cs = np.array([c[1].shape for c in cases], np.int64)
    np.savez_compressed(
        OUT / name,
        ref=np.concatenate([c[0].ravel() for c in cases]),
        cand=np.concatenate([c[1].ravel() for c in cases]),
        ref_shapes=rs, cand_shapes=cs,
        ref_off=np.concatenate([[0], np.cumsum(rs[:, 0] * rs[:, 1])]).astype(np.int64),
        cand_off=np.concatenate([[0], np.cumsum(cs[:, 0] * cs[:, 1])]).astype(np.int64),
        thr=np.array([c[2] for c in cases]), expected=np.array([c[3] for c in cases], np.int64),
        cos=np.concatenate([c[4] for c in cases]),
        cos_off=np.concatenate([[0], np.cumsum([len(c[4]) for c in cases])]).astype(np.int64))


# --- step 2: time, ledger, ratio, bucket ------------------------------------

def gen_time(rng):
    rows = []
    hzs = [1, 2, 3, 7.5, 10, 29.97, 30, 30.0, 50, 59.94, 100, 1000.0, 1 / 3, 0.1, 12.5, 240]
    for hz in hzs:
        for c in [0, 1, 2, 3, 9, 10, 29, 30, 48, 50, 64, 99, 1000, 12345, 10**6]:
            rows.append({"count": c, "hz": hz, "us": core.us_from_actions(c, hz)})
    for _ in range(300):
        hz = float(rng.choice(hzs))
        c = int(rng.integers(0, 5000))
        rows.append({"count": c, "hz": hz, "us": core.us_from_actions(c, hz)})
    return rows


def random_state(rng, tid: str, now: int, max_rounds: int = 6, p_inflight: float = 0.4):
    """A TaskState built through its own mutators (core.py:192-219)."""
    t = int(now - rng.integers(500_000, 20_000_000))
    st = TaskState(task_id=tid, t_start=t, accumulated_generation=int(rng.integers(0, 5_000_000)))
    n = int(rng.integers(0, max_rounds + 1))
    cur = t
    for j in range(n):
        gs = cur + int(rng.integers(0, 200_000))
        ge = gs + int(rng.integers(100_000, 400_000))
        es = ge + int(rng.integers(0, 50_000))
        ee = es + core.exec_duration(int(rng.integers(10, 51)), 30)
        st.begin_generation(j, gs)
        st.finish_generation(j, ge)
        st.record_execution(j, es, ee, 1)
        cur = ee - int(rng.integers(0, 300_000))
    if rng.random() < p_inflight:
        st.begin_generation(n, cur + int(rng.integers(0, 200_000)))
    return st


def state_json(st: TaskState):
    return {"task_id": st.task_id, "t_start": st.t_start, "skipped": st.skipped,
            "accumulated_generation": st.accumulated_generation,
            "gen_starts": list(st.gen_starts), "gen_ends": list(st.gen_ends),
            "exec_intervals": [[iv.start, iv.end] for iv in st.exec_intervals],
            "horizons": list(st.horizons)}


def req_json(r: PendingRequest):
    return {"task_id": r.task_id, "round_id": r.round_id, "issued_at": r.issued_at,
            "obs_captured_at": r.obs_captured_at,
            "last_exec_info": [r.last_exec_info.exec_start, r.last_exec_info.remaining_actions],
            "payload_bytes": r.payload_bytes, "skipped": r.skipped}


def gen_plan(rng):
    instances = []
    for ii in range(140):
        now = 100_000_000
        P = int(rng.choice([1, 2, 3, 5, 17, 64, 120]))
        tie_heavy = ii % 4 == 0
        id_style = rng.integers(0, 3)
        if id_style == 0:
            ids = [f"task-{i:04d}" for i in rng.choice(20000, P, replace=False)]
        elif id_style == 1:
            ids = [str(i) for i in rng.choice(100000, P, replace=False)]
        else:
            ids = ["".join(rng.choice(list("abAB09-_z"), int(rng.integers(1, 6)))) + f"#{i}"
                   for i in range(P)]
        states, pending = {}, []
        for tid in ids:
            st = random_state(rng, tid, now, max_rounds=2 if tie_heavy else 6)
            if tie_heavy:
                st.t_start = now - 1_000_000
            states[tid] = st
            skipped = int(rng.integers(0, 3 if tie_heavy else 13))
            st.skipped = skipped
            issued = now - int(rng.integers(0, 3 if tie_heavy else 1_000_000))
            pending.append(PendingRequest(
                task_id=tid, round_id=len(st.exec_intervals), issued_at=issued,
                obs_captured_at=issued - int(rng.integers(0, 300_000)),
                last_exec_info=LastExecInfo(issued - 1000, int(rng.integers(0, 40))),
                payload_bytes=int(rng.integers(0, 400_000)), skipped=skipped))
        policy = ["kairos", "fifo", "las"][ii % 3] if ii % 7 else "kairos"
        B = int(rng.choice([1, 2, 5, 10, 16]))
        A = int(rng.choice([1, 3, 5, 7]))
        cfg = scheduler.SchedulerConfig(policy=policy, buckets=B, aging_interval=A,
                                        stale_threshold=int(rng.choice([0, 150_000, 10**9])),
                                        default_exec_estimate=int(rng.choice([166_667, 0, 10**6])))
        cap = int(rng.integers(1, max(2, P + 3)))
        in_flight = int(rng.integers(0, 3))
        edge = EngineProfile(tier="edge", capacity=cap, max_batch=1, points=((1, 1000),))
        before = {t: state_json(s) for t, s in states.items()}
        # per-request intermediates through the reference functions
        inter = {}
        for r in pending:
            s = states[r.task_id]
            wr = waiting.current_wait_ratio(s, now)
            inter[r.task_id] = {
                "total_wait": waiting.ledger_from_history(s).total_wait, "wr": wr,
                "bucket": scheduler.assign_bucket(wr, r.skipped, cfg),
                "est": scheduler.estimate_exec_latency(s, cfg.default_exec_estimate),
                "need_time": core.exec_end_from_piggyback(r, 30)}
        order_in = list(pending)
        rng.shuffle(order_in)
        plan = scheduler.plan(order_in, states, edge, None, None, now, cfg,
                              edge_in_flight=in_flight)
        instances.append({
            "now": now, "policy": policy, "buckets": B, "aging_interval": A,
            "stale_threshold": cfg.stale_threshold,
            "default_exec_estimate": cfg.default_exec_estimate,
            "capacity": cap, "edge_in_flight": in_flight, "control_hz": 30,
            "states": list(before.values()), "pending": [req_json(r) for r in order_in],
            "intermediates": inter,
            "expected": {
                "edge": [r.task_id for r in plan.edge],
                "deferred": [[r.task_id, r.skipped] for r in plan.deferred],
                "refetch": sorted(plan.refetch_task_ids),
                "skipped_after": {t: s.skipped for t, s in states.items()}}})
    return instances


def random_profile(rng, tier):
    """A valid saturating profile: lat(b) = base + slope * b (throughput rises to max_batch)."""
    nb = int(rng.integers(1, 6))
    batches = sorted(set(int(b) for b in rng.choice([1, 2, 3, 4, 6, 8, 12, 16, 32], nb, replace=False)))
    base = int(rng.integers(20_000, 400_000))
    slope = int(rng.integers(1_000, 60_000))
    pts = tuple((b, base + slope * b) for b in batches)
    return EngineProfile(tier=tier, capacity=int(rng.integers(1, 40)), max_batch=batches[-1],
                         points=pts)


def gen_plan_cloud(rng):
    """plan() with a cloud tier and network model (scheduler.py:160-221)."""
    instances = []
    for ii in range(80):
        now = 100_000_000
        P = int(rng.choice([1, 3, 8, 30, 90, 200]))
        ids = [f"task-{i:04d}" for i in rng.choice(20000, P, replace=False)]
        states, pending = {}, []
        for tid in ids:
            st = random_state(rng, tid, now)
            skipped = int(rng.integers(0, 13))
            st.skipped = skipped
            states[tid] = st
            issued = now - int(rng.integers(0, 1_000_000))
            pending.append(PendingRequest(
                task_id=tid, round_id=len(st.exec_intervals), issued_at=issued,
                obs_captured_at=issued - int(rng.integers(0, 300_000)),
                last_exec_info=LastExecInfo(issued - 1000, int(rng.integers(0, 40))),
                payload_bytes=int(rng.choice([0, 1_000, 50_000, 300_000, int(rng.integers(0, 2_000_000))])),
                skipped=skipped))
        policy = ["kairos", "fifo", "las"][ii % 3]
        cfg = scheduler.SchedulerConfig(policy=policy, buckets=10, aging_interval=5,
                                        stale_threshold=int(rng.choice([0, 150_000, 10**9])))
        edge = None if ii % 9 == 0 else random_profile(rng, "edge")
        cloud = random_profile(rng, "cloud")
        net = NetworkModel(base_latency_us=int(rng.integers(1_000, 120_000)),
                           uplink_bps=int(rng.choice([10**6, 10**7, 10**8, int(rng.integers(10**5, 10**9))])),
                           downlink_bps=int(rng.choice([10**7, 10**8, int(rng.integers(10**5, 10**9))])))
        eif = int(rng.integers(0, 12))
        cif = int(rng.integers(0, 12))
        before = {t: state_json(s) for t, s in states.items()}
        order_in = list(pending)
        rng.shuffle(order_in)
        plan = scheduler.plan(order_in, states, edge, cloud, net, now, cfg,
                              edge_in_flight=eif, cloud_in_flight=cif)
        prof = lambda e: None if e is None else {"tier": e.tier, "capacity": e.capacity,
                                                  "max_batch": e.max_batch, "points": list(e.points)}
        instances.append({
            "now": now, "policy": policy, "buckets": 10, "aging_interval": 5,
            "stale_threshold": cfg.stale_threshold,
            "default_exec_estimate": cfg.default_exec_estimate,
            "edge": prof(edge), "cloud": prof(cloud),
            "net": {"base_latency_us": net.base_latency_us, "uplink_bps": net.uplink_bps,
                    "downlink_bps": net.downlink_bps},
            "edge_in_flight": eif, "cloud_in_flight": cif, "control_hz": 30,
            "states": list(before.values()), "pending": [req_json(r) for r in order_in],
            "expected": {
                "edge": [r.task_id for r in plan.edge],
                "cloud": [r.task_id for r in plan.cloud],
                "deferred": [[r.task_id, r.skipped] for r in plan.deferred],
                "refetch": sorted(plan.refetch_task_ids),
                "skipped_after": {t: s.skipped for t, s in states.items()}}})
    return instances


def gen_fig4():
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        g = runpy.run_path(os.path.join(REF_PKG, "scratch_fig4.py"), run_name="scratch_fig4")
    out = []
    for durs, gen in g["candidates"]:
        durs_us = [[d * g["MS"] for d in task] for task in durs]
        kai = g["policy_order"](durs_us, gen * g["MS"], g["kairos_choose_factory"](durs_us, gen * g["MS"]))
        fifo = g["policy_order"](durs_us, gen * g["MS"], g["fifo_choose"])
        las = g["policy_order"](durs_us, gen * g["MS"], g["las_choose_factory"](gen * g["MS"]))
        w_kai, w_fifo, w_las, w_opt = g["evaluate"](durs_us, gen * g["MS"])
        out.append({"durs": durs, "gen": gen, "kairos": list(kai), "fifo": list(fifo),
                    "las": list(las), "w_kai": w_kai, "w_fifo": w_fifo, "w_las": w_las,
                    "w_opt": w_opt})
    return {"stdout": buf.getvalue(), "candidates": out}


# --- simulator planning loop (sim.py:285-311, 358-385, 424-440) ----------

def gen_sim():
    """Run the reference discrete-event simulator and record, in order, every
    TaskState mutation it makes (creation, begin/finish generation with the
    accumulated-generation increment, record_execution) and every plan() call
    with its inputs and decision.  Replaying the log against an incremental
    device ledger must reproduce every decision."""
    from roboserve import sim as rsim
    from roboserve.workload import SyntheticSpec, synthesize_family

    log: list = []

    class RecState(TaskState):
        def __init__(self, *args, **kwargs):
            super().__init__(*args, **kwargs)
            log.append({"k": "new", "t": self.task_id, "a": self.t_start})

        def begin_generation(self, round_id, at):
            super().begin_generation(round_id, at)
            log.append({"k": "bg", "t": self.task_id, "j": round_id, "a": at})

        def finish_generation(self, round_id, at):
            super().finish_generation(round_id, at)
            log.append({"k": "fg", "t": self.task_id, "j": round_id, "a": at,
                        "g0": self.accumulated_generation})

        def record_execution(self, round_id, start, end, horizon):
            super().record_execution(round_id, start, end, horizon)
            log.append({"k": "rx", "t": self.task_id, "j": round_id, "a": start, "b": end,
                        "h": horizon})

    ref_plan = rsim.plan

    def rec_plan(pending, states, edge, cloud, net, now, cfg, *, edge_in_flight=0,
                 cloud_in_flight=0):
        # accumulated_generation of the finished round is added right after
        # finish_generation: fold the pending increments into the log first
        open_fg: dict = {}
        for e in log:
            if e["k"] == "fg" and "c" not in e:
                open_fg.setdefault(e["t"], []).append(e)
        for tid, es in open_fg.items():
            nxt = [x["g0"] for x in es[1:]] + [states[tid].accumulated_generation]
            for e, g1 in zip(es, nxt):
                e["c"] = g1 - e.pop("g0")
        pending = list(pending)
        entry = {"k": "plan", "now": now, "eif": edge_in_flight, "cif": cloud_in_flight,
                 "pending": [req_json(r) for r in pending]}
        d = ref_plan(pending, states, edge, cloud, net, now, cfg, edge_in_flight=edge_in_flight,
                     cloud_in_flight=cloud_in_flight)
        entry["exp"] = {"edge": [r.task_id for r in d.edge], "cloud": [r.task_id for r in d.cloud],
                        "deferred": [[r.task_id, r.skipped] for r in d.deferred],
                        "refetch": sorted(d.refetch_task_ids)}
        log.append(entry)
        return d

    prof = lambda e: None if e is None else {"tier": e.tier, "capacity": e.capacity,
                                              "max_batch": e.max_batch, "points": list(e.points)}
    netj = lambda n: None if n is None else {"base_latency_us": n.base_latency_us,
                                             "uplink_bps": n.uplink_bps,
                                             "downlink_bps": n.downlink_bps}
    edge = EngineProfile(tier="edge", capacity=4, max_batch=4,
                         points=((1, 120_000), (2, 150_000), (4, 210_000)))
    cloud = EngineProfile(tier="cloud", capacity=8, max_batch=8,
                          points=((1, 60_000), (4, 80_000), (8, 110_000)))
    wan = NetworkModel(base_latency_us=40_000, uplink_bps=50_000_000, downlink_bps=200_000_000)
    lan = NetworkModel(base_latency_us=2_000, uplink_bps=400_000_000, downlink_bps=800_000_000)
    scenarios = [
        ("kairos-edge", scheduler.SchedulerConfig(), edge, None, None, None, 36, 12, "event"),
        ("kairos-hybrid", scheduler.SchedulerConfig(stale_threshold=100_000), edge, cloud, wan,
         lan, 48, 16, "event"),
        ("fifo-edge", scheduler.SchedulerConfig(policy="fifo"), edge, None, None, None, 30, 10,
         "event"),
        ("las-hybrid", scheduler.SchedulerConfig(policy="las", buckets=4, aging_interval=2),
         edge, cloud, wan, None, 30, 10, "event"),
        ("kairos-interval", scheduler.SchedulerConfig(buckets=16, aging_interval=3), edge, None,
         None, None, 30, 12, "interval"),
    ]
    out = []
    old_state, old_plan = rsim.TaskState, rsim.plan
    rsim.TaskState, rsim.plan = RecState, rec_plan
    try:
        for i, (name, scfg, e, c, net, enet, ntr, slots, mode) in enumerate(scenarios):
            log.clear()
            spec = SyntheticSpec(action_budget=160, uncertain_fraction=0.3)
            traces = synthesize_family(spec, horizon.HorizonPolicyConfig.confidence(0.4, 5),
                                       gen_latency=150_000, count=ntr, seed=100 + i)
            cfg = rsim.SimConfig(scheduler=scfg, edge=e, cloud=c, network=net, edge_network=enet,
                                 plan_mode=mode, plan_interval_us=40_000)
            rsim.run_fleet(traces, slots, cfg)
            for ev in log:  # increments after the last plan() never reach a decision
                if ev.pop("g0", None) is not None:
                    ev["c"] = 0
            out.append({"name": name, "policy": scfg.policy, "buckets": scfg.buckets,
                        "aging_interval": scfg.aging_interval,
                        "stale_threshold": scfg.stale_threshold,
                        "default_exec_estimate": scfg.default_exec_estimate,
                        "edge": prof(e), "cloud": prof(c), "net": netj(net),
                        "log": list(log)})
    finally:
        rsim.TaskState, rsim.plan = old_state, old_plan
    return out


# --- trace ingest + pareto (workload.py:163-262, cli.py:104-140) ------------

def gen_traces():
    """Trace files written by the reference's store_traces, the reference's
    `roboserve pareto` CSV over them, and malformed variants with the
    reference load_traces' TraceFormatError fields."""
    import copy
    import tempfile

    from roboserve import cli
    from roboserve.workload import SyntheticSpec, synthesize_family

    tdir = OUT / "traces"
    tdir.mkdir(exist_ok=True)
    conf = horizon.HorizonPolicyConfig.confidence(0.4, 5)
    fams = [
        ("a_arms.jsonl", SyntheticSpec(chunk_size=16, diffusion_steps=6, action_budget=60,
                                       success_rate=0.7), 6, True),
        ("b_humanoid.jsonl", SyntheticSpec(chunk_size=32, diffusion_steps=10, control_hz=50.0,
                                           action_budget=80, uncertain_fraction=0.35), 5, False),
        ("c_mixed.jsonl", SyntheticSpec(chunk_size=16, diffusion_steps=6, action_budget=40,
                                        control_hz=29.97, bump_factor=2.5), 4, True),
    ]
    for i, (name, spec, count, traj) in enumerate(fams):
        fam = synthesize_family(spec, conf, gen_latency=80_000, count=count, seed=300 + i,
                                id_prefix=name[0], with_trajectories=traj, trajectory_dim=3)
        workload.store_traces(fam, tdir / name)
    pareto = {}
    with tempfile.TemporaryDirectory() as td:
        for key, args in (("default", []),
                          ("custom", ["--static-grid", "1,7,16,40", "--threshold-grid",
                                      "0,0.05,0.4,0.8,1.5,2.5", "--h-min", "3"])):
            out = Path(td) / f"{key}.csv"
            with contextlib.redirect_stdout(io.StringIO()):
                rc = cli.main(["pareto", "--traces", str(tdir), "--out", str(out), *args])
            assert rc == 0
            pareto[key] = {"args": args, "csv": out.read_text()}
    # malformed variants of one valid trace line
    base = workload.trace_to_dict(workload.load_traces(tdir / "a_arms.jsonl")[0])
    def mut(f):
        d = copy.deepcopy(base)
        f(d)
        return json.dumps(d, separators=(",", ":"))
    good = json.dumps(base, separators=(",", ":"))
    texts = {
        "broken_json": good + "\n{broken\n",
        "not_object": "\n\n[1, 2]\n",
        "extra_data": good + " 7\n",
        "missing_control_hz": mut(lambda d: d.pop("control_hz")),
        "missing_rounds": mut(lambda d: d.pop("rounds")),
        "missing_round_field": mut(lambda d: d["rounds"][1].pop("horizon")),
        "horizon_bounds": mut(lambda d: d["rounds"][0].__setitem__("horizon", 99)),
        "horizon_zero": mut(lambda d: d["rounds"][1].__setitem__("horizon", 0)),
        "neg_round_id": mut(lambda d: d["rounds"][0].__setitem__("round_id", -1)),
        "neg_trigger": mut(lambda d: d["rounds"][1].__setitem__("trigger_action_index", -2)),
        "noncontiguous": mut(lambda d: d["rounds"][1].__setitem__("round_id", 5)),
        "trigger_bound": mut(lambda d: d["rounds"][1].__setitem__(
            "trigger_action_index", d["rounds"][0]["horizon"])),
        "no_rounds": mut(lambda d: d.__setitem__("rounds", [])),
        "zero_hz": mut(lambda d: d.__setitem__("control_hz", 0)),
        "neg_payload": mut(lambda d: d.__setitem__("obs_payload_bytes", -1)),
        "empty_task": mut(lambda d: d.__setitem__("task_id", "")),
        "neg_magnitude": mut(lambda d: d["rounds"][0]["update_magnitudes"][1].__setitem__(2, -0.5)),
        "nan_magnitude": mut(lambda d: d["rounds"][1]["update_magnitudes"][0].__setitem__(
            0, float("nan"))),
        "one_d_magnitudes": mut(lambda d: d["rounds"][0].__setitem__("update_magnitudes", [1.0, 2.0])),
        "k1_magnitudes": mut(lambda d: d["rounds"][0].__setitem__("update_magnitudes", [[1.0, 2.0]])),
        "empty_magnitudes": mut(lambda d: d["rounds"][0].__setitem__("update_magnitudes", [])),
        "three_d": mut(lambda d: d["rounds"][0].__setitem__("update_magnitudes", [[[1.0]], [[2.0]]])),
        "blank_lines_ok": "\n  \n" + good + "\n\n" + good.replace('"a-0000"', '"a-9999"') + "\n",
        "second_line_bad": good + "\n" + mut(lambda d: d.__setitem__("success", None)).replace(
            '"round_id":0', '"round_id":3', 1) + "\n",
    }
    errors = []
    with tempfile.TemporaryDirectory() as td:
        for name, text in texts.items():
            f = Path(td) / "x.jsonl"
            f.write_text(text)
            try:
                loaded = workload.load_traces(f)
                errors.append({"name": name, "text": text, "ok": [workload.trace_to_dict(t) for t in loaded]})
            except workload.TraceFormatError as e:
                errors.append({"name": name, "text": text, "error": str(e), "raw": e.raw_message,
                               "line": e.line, "task_id": e.task_id, "round_id": e.round_id})
    (OUT / "traces_expected.json").write_text(json.dumps({"pareto": pareto, "cases": errors},
                                                         indent=0))


# --- synthetic traces: the reference's distributions (§8(f)4) ---------------

SYNTH_INVALID = [{"chunk_size": 0}, {"diffusion_steps": 1}, {"control_hz": 0.0},
                 {"action_budget": 0}, {"uncertain_fraction": 1.5}, {"decay": 1.0},
                 {"noise_scale": 0.5}, {"bump_factor": 1.0}, {"success_rate": -0.1},
                 {"chunk_sizes": 3, "zeta": 1}]

SYNTH_SETTINGS = [
    ({}, ("confidence", {}), 100_000),
    ({"chunk_size": 32, "diffusion_steps": 8, "action_budget": 120, "uncertain_fraction": 0.5,
      "decay": 0.4, "noise_scale": 0.2, "bump_factor": 2.5, "success_rate": 0.6},
     ("confidence", {"threshold": 0.3, "min_horizon": 4}), 50_000),
    ({"uncertain_fraction": 0.05, "control_hz": 15.0}, ("static", {"horizon": 20}), 100_000),
]


def gen_synth():
    out = []
    for spec_kw, (kind, pol_kw), gen_latency in SYNTH_SETTINGS:
        spec = workload.SyntheticSpec(**spec_kw)
        pol = (horizon.HorizonPolicyConfig.confidence(**pol_kw) if kind == "confidence"
               else horizon.HorizonPolicyConfig.static(**pol_kw))
        fam = workload.synthesize_family(spec, pol, gen_latency, 3000, seed=17)
        out.append({"spec": spec_kw, "policy": [kind, pol_kw], "gen_latency": gen_latency,
                    "stats": golden_io.synth_stats(fam, spec_kw)})
    # the reference's validation message (workload.py:386-391)
    try:
        workload.synthesize_trace(workload.SyntheticSpec(), horizon.HorizonPolicyConfig.static(2),
                                  100_000, 0)
    except ValueError as e:
        err = str(e)
    spec_errors = []
    for kw in SYNTH_INVALID:
        try:
            workload.SyntheticSpec.from_dict(kw)
        except ValueError as e:
            spec_errors.append([kw, str(e)])
    return {"settings": out, "too_slow_error": err, "spec_errors": spec_errors}


def gen_divergence_haswell():
    """The divergence cases with the reference's cosines computed by numpy's
    OpenBLAS running its Haswell core (OPENBLAS_CORETYPE=Haswell, which the
    library also selects on Zen hosts): pins the second ddot order."""
    if os.environ.get("OPENBLAS_CORETYPE") != "Haswell":
        import subprocess
        env = dict(os.environ, OPENBLAS_CORETYPE="Haswell")
        subprocess.run([sys.executable, __file__, "haswell"], env=env, check=True)
        return
    import threadpoolctl
    cores = {i["architecture"] for i in threadpoolctl.threadpool_info()
             if i.get("internal_api") == "openblas"}
    assert cores == {"Haswell"}, cores
    save_divergence(gen_divergence(np.random.default_rng(31)), "divergence_haswell.npz")


def main():
    if sys.argv[1:] == ["synth"]:  # only the synthesis-distribution fixture
        (OUT / "synth_stats.json").write_text(json.dumps(gen_synth(), indent=0))
        return
    if sys.argv[1:] == ["haswell"]:  # only the Haswell-order divergence fixture
        gen_divergence_haswell()
        return
    if sys.argv[1:] == ["traces"]:  # only the trace-ingest fixtures
        gen_traces()
        return
    if sys.argv[1:] == ["sweep"]:  # only the threshold-sweep fixture
        save_sweep(gen_sweep(np.random.default_rng(11)))
        return
    if sys.argv[1:] == ["sim"]:  # only the simulator replay fixture
        (OUT / "sim_replay.json").write_text(json.dumps(gen_sim(), separators=(",", ":")))
        return
    rng = np.random.default_rng(20260517)
    save_confidence(gen_confidence(rng))
    save_divergence(gen_divergence(rng))
    gen_divergence_haswell()
    (OUT / "time.json").write_text(json.dumps(gen_time(rng)))
    (OUT / "plan.json").write_text(json.dumps(gen_plan(rng), separators=(",", ":")))
    (OUT / "plan_cloud.json").write_text(json.dumps(gen_plan_cloud(np.random.default_rng(7)),
                                                    separators=(",", ":")))
    (OUT / "fig4.json").write_text(json.dumps(gen_fig4(), indent=1))
    save_sweep(gen_sweep(np.random.default_rng(11)))
    (OUT / "sim_replay.json").write_text(json.dumps(gen_sim(), separators=(",", ":")))
    gen_traces()
    (OUT / "synth_stats.json").write_text(json.dumps(gen_synth(), indent=0))
    for p in sorted(OUT.iterdir()):
        if p.suffix in (".npz", ".json"):
            print(f"{p.name:28s} {p.stat().st_size:>9d} B")


if __name__ == "__main__":
    main()
