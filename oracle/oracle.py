"""TEST INFRASTRUCTURE ONLY -- ctypes front end of the CPU oracle.

`oracle/kairos_oracle.c` restates the reference's hot path
(/root/reference/pkg/src/roboserve/{horizon,waiting,scheduler,core}.py and
workload.py:461-496) in plain C; this module loads it and converts numpy
arrays / reference-shaped objects into its structure-of-arrays form.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
--impl reference) import this module, and only as the checker or the timed
CPU baseline.  The product package never imports it.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from fractions import Fraction
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_SO = _HERE / "build" / "liboracle.so"
_LIB = None

KAIROS, FIFO, LAS = 0, 1, 2
POLICY_CODES = {"kairos": KAIROS, "fifo": FIFO, "las": LAS}

_i64p = ctypes.POINTER(ctypes.c_int64)
_i32p = ctypes.POINTER(ctypes.c_int32)
_u8p = ctypes.POINTER(ctypes.c_uint8)
_f64p = ctypes.POINTER(ctypes.c_double)


class _Profile(ctypes.Structure):
    _fields_ = [("capacity", ctypes.c_int64), ("max_batch", ctypes.c_int64),
                ("npts", ctypes.c_int32), ("batch", ctypes.POINTER(ctypes.c_int64)),
                ("latency", ctypes.POINTER(ctypes.c_int64))]


class _Net(ctypes.Structure):
    _fields_ = [("base_latency_us", ctypes.c_int64), ("uplink_bps", ctypes.c_int64),
                ("downlink_bps", ctypes.c_int64)]


class _Fleet(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int64),
        ("t_start", _i64p),
        ("issued_at", _i64p),
        ("obs_captured_at", _i64p),
        ("accum_gen", _i64p),
        ("remaining", _i32p),
        ("lexrank", _i32p),
        ("skipped", _i32p),
        ("hist_off", _i64p),
        ("n_exec", _i32p),
        ("n_gen", _i32p),
        ("slots", _i64p),
    ]


def build() -> Path:
    """Compile the oracle (gcc, -ffp-contract=off) if it is missing or stale."""
    src = [_HERE / "kairos_oracle.c", _HERE / "kairos_oracle.h"]
    if not _SO.exists() or any(s.stat().st_mtime > _SO.stat().st_mtime for s in src):
        subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _SO


def lib():
    global _LIB
    if _LIB is None:
        build()
        L = ctypes.CDLL(str(_SO))
        vp = ctypes.c_void_p
        L.orc_np_mean_col.restype = ctypes.c_double
        L.orc_np_mean_col.argtypes = [_f64p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64]
        L.orc_ddot.restype = ctypes.c_double
        L.orc_ddot.argtypes = [_f64p, _f64p, ctypes.c_int64]
        L.orc_set_dot_order.restype = ctypes.c_int
        L.orc_set_dot_order.argtypes = [ctypes.c_int]
        L.orc_get_dot_order.restype = ctypes.c_int
        L.orc_get_dot_order.argtypes = []
        L.orc_cosine.restype = ctypes.c_double
        L.orc_cosine.argtypes = [_f64p, _f64p, ctypes.c_int64]
        L.orc_decide_horizon_conf.restype = ctypes.c_int32
        L.orc_decide_horizon_conf.argtypes = [_f64p, ctypes.c_int64, ctypes.c_int64,
                                              ctypes.c_double, ctypes.c_int64]
        L.orc_round_optimal_horizon.restype = ctypes.c_int64
        L.orc_round_optimal_horizon.argtypes = [_f64p, ctypes.c_int64, _f64p, ctypes.c_int64,
                                                ctypes.c_int64, ctypes.c_double]
        L.orc_horizon_conf_batch.restype = None
        L.orc_horizon_conf_batch.argtypes = [vp, ctypes.c_int, ctypes.c_int64, ctypes.c_int64,
                                             ctypes.c_int64, ctypes.c_double, ctypes.c_int64,
                                             _i32p, ctypes.c_int]
        L.orc_divergence_batch.restype = None
        L.orc_divergence_batch.argtypes = [vp, vp, ctypes.c_int, ctypes.c_int64, ctypes.c_int64,
                                           ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                           _i32p, _i32p, _i32p, ctypes.c_double, _i32p, _f64p,
                                           ctypes.c_int]
        L.orc_us_from_actions.restype = ctypes.c_int64
        L.orc_us_from_actions.argtypes = [ctypes.c_int64] * 3
        L.orc_total_wait.restype = ctypes.c_int64
        L.orc_total_wait.argtypes = [_i64p, ctypes.c_int32, ctypes.c_int32]
        L.orc_current_wait_ratio.restype = ctypes.c_double
        L.orc_current_wait_ratio.argtypes = [ctypes.c_int64] * 3
        L.orc_assign_bucket.restype = ctypes.c_int32
        L.orc_assign_bucket.argtypes = [ctypes.c_double, ctypes.c_int64, ctypes.c_int64,
                                        ctypes.c_int64]
        L.orc_batch_latency.restype = ctypes.c_int64
        L.orc_batch_latency.argtypes = [ctypes.POINTER(_Profile), ctypes.c_int64]
        L.orc_transfer_time.restype = ctypes.c_int64
        L.orc_transfer_time.argtypes = [ctypes.POINTER(_Net), ctypes.c_int64, ctypes.c_int]
        L.orc_plan_tiers.restype = ctypes.c_int64
        L.orc_plan_tiers.argtypes = [ctypes.POINTER(_Fleet), _i64p, ctypes.c_int] + \
            [ctypes.c_int64] * 5 + [ctypes.POINTER(_Profile), ctypes.POINTER(_Profile),
                                    ctypes.POINTER(_Net), ctypes.c_int64, ctypes.c_int64,
                                    _i32p, _u8p, _i32p, _u8p, _i32p, _i64p]
        L.orc_plan.restype = ctypes.c_int64
        L.orc_plan.argtypes = [ctypes.POINTER(_Fleet), ctypes.c_int] + [ctypes.c_int64] * 8 + [
            _i32p, _i64p, _f64p, _i32p, _i64p, _i64p, _u8p, _u8p, _i32p]
        _LIB = L
    return _LIB


def _p(a, t):
    return None if a is None else a.ctypes.data_as(t)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def hz_ratio(control_hz) -> tuple[int, int]:
    """Exact (numerator, denominator) of control_hz, as core.py:42 takes it."""
    fr = Fraction(control_hz)
    return fr.numerator, fr.denominator


# --- step 1 -----------------------------------------------------------------

def np_mean_col(u, n: int) -> float:
    u = _f64(u)
    return lib().orc_np_mean_col(_p(u, _f64p), u.shape[0], u.shape[1], n)


DOT_ORDERS = {"skylakex": 0, "haswell": 1}


def set_dot_order(name: str) -> str:
    """Select the OpenBLAS core whose ddot order the oracle reproduces
    (process-wide); returns the previous one."""
    prev = get_dot_order()
    if lib().orc_set_dot_order(DOT_ORDERS[name]) != 0:
        raise ValueError(name)
    return prev


def get_dot_order() -> str:
    code = lib().orc_get_dot_order()
    return next(k for k, v in DOT_ORDERS.items() if v == code)


def ddot(x, y) -> float:
    x, y = _f64(x), _f64(y)
    return lib().orc_ddot(_p(x, _f64p), _p(y, _f64p), x.size)


def cosine(a, b) -> float:
    a, b = _f64(a), _f64(b)
    return lib().orc_cosine(_p(a, _f64p), _p(b, _f64p), a.size)


def decide_horizon_conf(u, threshold: float, min_horizon: int) -> int:
    u = _f64(u)
    return int(lib().orc_decide_horizon_conf(_p(u, _f64p), u.shape[0], u.shape[1],
                                             1.0 + threshold, min_horizon))


def round_optimal_horizon(reference, candidate, thr: float) -> int:
    ref, cand = _f64(reference), _f64(candidate)
    return int(lib().orc_round_optimal_horizon(_p(ref, _f64p), ref.shape[0], _p(cand, _f64p),
                                               cand.shape[0], ref.shape[1], thr))


def horizon_conf_batch(U: np.ndarray, threshold: float, min_horizon: int,
                       nthreads: int = 0) -> np.ndarray:
    assert U.dtype in (np.float32, np.float64) and U.ndim == 3
    U = np.ascontiguousarray(U)
    R, K, N = U.shape
    H = np.empty(R, np.int32)
    lib().orc_horizon_conf_batch(U.ctypes.data, int(U.dtype == np.float64), R, K, N,
                                 1.0 + threshold, min_horizon, _p(H, _i32p), nthreads)
    return H


def sweep_sums(U: np.ndarray, cfgs) -> np.ndarray:
    """sum_r decide_horizon(cfg, U[r]) per configuration (horizon.py:135-151 is
    sum(decide_horizon(...)) / len(seq)).  cfgs: (kind, static_h, threshold,
    min_horizon) tuples, kind 1 = confidence, 0 = static (horizon.py:121-122)."""
    R, _, N = U.shape
    out = np.empty(len(cfgs), np.int64)
    for c, (kind, static_h, t, hmin) in enumerate(cfgs):
        if kind == 0:
            out[c] = R * min(static_h, N)
        else:
            out[c] = int(horizon_conf_batch(U, t, hmin).astype(np.int64).sum())
    return out


def divergence_batch(prev, cand, thr: float, offset=None, len_prev=None, len_cand=None,
                     want_cos: bool = False, nthreads: int = 0):
    """prev [R,Lp,D]; cand [R,Lc,D] or [R,S,Lc,D] (same float dtype)."""
    prev = np.ascontiguousarray(prev)
    cand = np.ascontiguousarray(cand)
    assert prev.dtype == cand.dtype and prev.dtype in (np.float32, np.float64)
    if cand.ndim == 3:
        cand = cand[:, None]
    R, Lp, D = prev.shape
    _, S, Lc, D2 = cand.shape
    assert D == D2 and cand.shape[0] == R
    conv = lambda a: None if a is None else np.ascontiguousarray(a, np.int32)
    offset, len_prev, len_cand = conv(offset), conv(len_prev), conv(len_cand)
    H = np.empty(R, np.int32)
    cos = np.empty((R, S, Lc), np.float64) if want_cos else None
    lib().orc_divergence_batch(prev.ctypes.data, cand.ctypes.data,
                               int(prev.dtype == np.float64), R, S, Lp, Lc, D,
                               _p(offset, _i32p), _p(len_prev, _i32p), _p(len_cand, _i32p),
                               thr, _p(H, _i32p), _p(cos, _f64p), nthreads)
    return (H, cos) if want_cos else H


# --- step 2 -----------------------------------------------------------------

def us_from_actions(count: int, control_hz) -> int:
    p, q = hz_ratio(control_hz)
    return int(lib().orc_us_from_actions(count, p, q))


def total_wait(slots: np.ndarray, n_exec: int, n_gen: int) -> int:
    slots = np.ascontiguousarray(slots, np.int64).reshape(-1)
    if slots.size == 0:
        slots = np.zeros(4, np.int64)
    return int(lib().orc_total_wait(_p(slots, _i64p), n_exec, n_gen))


def current_wait_ratio(total: int, t_start: int, now: int) -> float:
    return float(lib().orc_current_wait_ratio(total, t_start, now))


def assign_bucket(wr: float, skipped: int, buckets: int, aging_interval: int) -> int:
    return int(lib().orc_assign_bucket(wr, skipped, buckets, aging_interval))


# --- fleet SoA --------------------------------------------------------------

FLEET_FIELDS = {
    "t_start": np.int64, "issued_at": np.int64, "obs_captured_at": np.int64,
    "accum_gen": np.int64, "remaining": np.int32, "lexrank": np.int32,
    "skipped": np.int32, "hist_off": np.int64, "n_exec": np.int32, "n_gen": np.int32,
    "slots": np.int64,
}


def fleet_from_objects(pending, states, all_task_ids=None) -> dict:
    """Reference-shaped PendingRequest / TaskState objects -> SoA arrays.

    `lexrank` is each request's task_id position in Python string order over
    `all_task_ids` (default: the pending ids), so integer comparison of ranks
    reproduces the reference's `task_id` tiebreak (scheduler.py:115).
    """
    pending = list(pending)
    ids = sorted(all_task_ids if all_task_ids is not None else [r.task_id for r in pending])
    rank = {t: i for i, t in enumerate(ids)}
    n = len(pending)
    out = {k: np.zeros(n, v) for k, v in FLEET_FIELDS.items() if k != "slots"}
    slots = []
    for i, req in enumerate(pending):
        st = states[req.task_id]
        out["t_start"][i] = st.t_start
        out["issued_at"][i] = req.issued_at
        out["obs_captured_at"][i] = req.obs_captured_at
        out["accum_gen"][i] = st.accumulated_generation
        out["remaining"][i] = req.last_exec_info.remaining_actions
        out["lexrank"][i] = rank[req.task_id]
        out["skipped"][i] = req.skipped
        ne, ng = len(st.exec_intervals), len(st.gen_starts)
        out["n_exec"][i], out["n_gen"][i] = ne, ng
        out["hist_off"][i] = len(slots)
        for j in range(max(ne, ng)):
            gs = st.gen_starts[j] if j < ng else 0
            ge = st.gen_ends[j] if j < ng and st.gen_ends[j] is not None else 0
            es, ee = (st.exec_intervals[j].start, st.exec_intervals[j].end) if j < ne else (0, 0)
            slots.append((gs, ge, es, ee))
    out["slots"] = np.array(slots if slots else [(0, 0, 0, 0)], np.int64).reshape(-1, 4)
    out["n"] = n
    return out


def plan_soa(fleet: dict, policy: str, buckets: int, aging_interval: int,
             stale_threshold: int, default_exec_estimate: int, now: int,
             control_hz, edge_avail: int) -> dict:
    """scheduler.py:254-276 plan() on SoA input (edge tier only)."""
    n = int(fleet["n"])
    arrs = {k: np.ascontiguousarray(fleet[k], v) for k, v in FLEET_FIELDS.items()}
    f = _Fleet(n, *[_p(arrs[k], _i64p if arrs[k].dtype == np.int64 else _i32p)
                    for k in ["t_start", "issued_at", "obs_captured_at", "accum_gen", "remaining",
                              "lexrank", "skipped", "hist_off", "n_exec", "n_gen", "slots"]])
    p, q = hz_ratio(control_hz)
    res = {
        "order": np.empty(n, np.int32), "total_wait": np.empty(n, np.int64),
        "wr": np.empty(n, np.float64), "bucket": np.empty(n, np.int32),
        "est": np.empty(n, np.int64), "need_time": np.empty(n, np.int64),
        "admitted": np.empty(n, np.uint8), "refetch": np.empty(n, np.uint8),
        "skipped_out": np.empty(n, np.int32),
    }
    res["n_edge"] = int(lib().orc_plan(
        ctypes.byref(f), POLICY_CODES[policy], buckets, aging_interval, stale_threshold,
        default_exec_estimate, now, p, q, edge_avail,
        _p(res["order"], _i32p), _p(res["total_wait"], _i64p), _p(res["wr"], _f64p),
        _p(res["bucket"], _i32p), _p(res["est"], _i64p), _p(res["need_time"], _i64p),
        _p(res["admitted"], _u8p), _p(res["refetch"], _u8p), _p(res["skipped_out"], _i32p)))
    return res


def nthreads_default() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()


# --- phase 3 (hybrid placement) ----------------------------------------------

def _profile(d):
    """Profile mapping (tier, capacity, max_batch, points) -> (struct, keepalive)."""
    if d is None:
        return None, None
    pts = np.asarray(d["points"], np.int64).reshape(-1, 2)
    b, lat = np.ascontiguousarray(pts[:, 0]), np.ascontiguousarray(pts[:, 1])
    st = _Profile(int(d["capacity"]), int(d["max_batch"]), len(pts), _p(b, _i64p), _p(lat, _i64p))
    return st, (b, lat)


def batch_latency(profile: dict, batch: int) -> int:
    st, keep = _profile(profile)
    return int(lib().orc_batch_latency(ctypes.byref(st), batch))


def transfer_time(net: dict, payload: int, up: bool) -> int:
    n = _Net(int(net["base_latency_us"]), int(net["uplink_bps"]), int(net["downlink_bps"]))
    return int(lib().orc_transfer_time(ctypes.byref(n), payload, int(up)))


def plan_tiers(fleet: dict, payload, policy: str, buckets: int, aging_interval: int,
               stale_threshold: int, default_exec_estimate: int, now: int, edge, cloud, net,
               edge_in_flight: int, cloud_in_flight: int) -> dict:
    """scheduler.py:254-276 plan() with edge / cloud profiles and network (dicts)."""
    n = int(fleet["n"])
    arrs = {k: np.ascontiguousarray(fleet[k], v) for k, v in FLEET_FIELDS.items()}
    f = _Fleet(n, *[_p(arrs[k], _i64p if arrs[k].dtype == np.int64 else _i32p)
                    for k in ["t_start", "issued_at", "obs_captured_at", "accum_gen", "remaining",
                              "lexrank", "skipped", "hist_off", "n_exec", "n_gen", "slots"]])
    pay = np.ascontiguousarray(payload, np.int64)
    e, ek = _profile(edge)
    c, ck = _profile(cloud)
    nt = None if net is None else _Net(int(net["base_latency_us"]), int(net["uplink_bps"]),
                                       int(net["downlink_bps"]))
    res = {"order": np.empty(n, np.int32), "tier": np.empty(n, np.uint8),
           "cloud_order": np.empty(max(n, 1), np.int32), "refetch": np.empty(n, np.uint8),
           "skipped_out": np.empty(n, np.int32)}
    n_edge = ctypes.c_int64(0)
    nc = lib().orc_plan_tiers(
        ctypes.byref(f), _p(pay, _i64p), POLICY_CODES[policy], buckets, aging_interval,
        stale_threshold, default_exec_estimate, now,
        ctypes.byref(e) if e is not None else None, ctypes.byref(c) if c is not None else None,
        ctypes.byref(nt) if nt is not None else None, edge_in_flight, cloud_in_flight,
        _p(res["order"], _i32p), _p(res["tier"], _u8p), _p(res["cloud_order"], _i32p),
        _p(res["refetch"], _u8p), _p(res["skipped_out"], _i32p), ctypes.byref(n_edge))
    res["n_cloud"] = int(nc)
    res["n_edge"] = int(n_edge.value)
    res["cloud_order"] = res["cloud_order"][:nc]
    return res
