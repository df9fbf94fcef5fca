"""Step 3: execution-aware priority ordering and top-k edge admission.

Drop-in for `roboserve.scheduler` (reference scheduler.py:1-284).  Config and
plan types keep the reference's fields and validation.  `plan` packs the
pending set into the fleet layout, and three CUDA kernels make every decision:

  kr_urgency    ledger -> wait ratio -> bucket (+aging) -> exec estimate ->
                aged estimate -> one unique 128-bit key per request whose
                ascending order is the reference's order (buckets high to low,
                then (-aged, issued_at, task_id); FIFO / LAS keys likewise)
  kr_sort_keys  the total order (needed for the ordered `deferred` tuple)
  kr_admit      edge prefix of k = capacity - in_flight, stale-observation
                refetch mask and the skip-counter side effect

  kr_place_cloud the phase-3 cloud offload scan over the rest of the order
                (scheduler.py:160-221): per-round thresholds T(c) are host
                scalars from the engine profiles; per-request uplink times
                (kr_transfer_time) and the ordered scan run on the device

The host only builds the result objects and mirrors the skip counters into
`states` as the reference does (scheduler.py:229-234).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, replace
from typing import Iterable, Mapping, Optional, Sequence

import numpy as np
import torch

from . import _lib
from . import device as dev
from . import engines as eng
from . import fleet as fl
from .core import Duration, PendingRequest, TaskState, TimePoint
from .waiting import _state_fleet
from . import ledger as _ledger

KAIROS = "kairos"
FIFO = "fifo"
LAS = "las"
POLICIES = (KAIROS, FIFO, LAS)

AGED_MAX = (1 << 56) - 1


@dataclass(frozen=True)
class SchedulerConfig:
    """Scheduler knobs (scheduler.py:38-56)."""

    policy: str = KAIROS
    buckets: int = 10
    aging_interval: int = 5
    stale_threshold: Duration = 150_000
    default_exec_estimate: Duration = 166_667

    def __post_init__(self) -> None:
        if self.policy not in POLICIES:
            raise ValueError(f"policy must be one of {POLICIES}, got {self.policy!r}")
        if self.buckets < 1:
            raise ValueError(f"buckets must be >= 1, got {self.buckets}")
        if self.aging_interval < 1:
            raise ValueError(f"aging_interval must be >= 1, got {self.aging_interval}")
        if self.stale_threshold < 0:
            raise ValueError("stale_threshold must be >= 0")
        if self.default_exec_estimate < 0:
            raise ValueError("default_exec_estimate must be >= 0")


@dataclass(frozen=True)
class DispatchPlan:
    """Per-tier dispatch lists plus deferred requests (scheduler.py:59-76)."""

    edge: tuple
    cloud: tuple
    deferred: tuple
    refetch_task_ids: frozenset

    @property
    def dispatched(self) -> tuple:
        return self.edge + self.cloud


def assign_bucket(wr: float, skipped: int, cfg: SchedulerConfig) -> int:
    """Equal-width wait-ratio bucket with skip promotion (scheduler.py:79-88)."""
    if not 0.0 <= wr <= 1.0:
        raise ValueError(f"wait ratio must be in [0, 1], got {wr}")
    if skipped < 0:
        raise ValueError(f"skipped must be >= 0, got {skipped}")
    if cfg.buckets > 256 or skipped >= (1 << 31):
        raise ValueError("buckets must be <= 256 and skipped < 2^31 on the device path")
    w = dev.tensor([float(wr)], torch.float64)
    s = dev.tensor([int(skipped)], torch.int32)
    b = torch.empty(1, dtype=torch.int32, device=w.device)
    _lib.check(_lib.load().kr_assign_bucket(w.data_ptr(), s.data_ptr(), 1, cfg.buckets,
                                            cfg.aging_interval, b.data_ptr(), dev.stream()),
               "kr_assign_bucket")
    return int(b.item())


def estimate_exec_latency(state: TaskState, default: Optional[Duration] = None) -> Duration:
    """Last execution length, else the default (scheduler.py:91-104)."""
    sched = fl.sched_struct(FIFO, 1, 1, 0, default if default is not None else 0, 0, 1, 0)
    out = fl.urgency(_state_fleet(state), sched, need_time=False, intermediates=True)
    return int(out.est.item())


def _issued_base(issued) -> int:
    if len(issued) == 0:
        return 0
    lo, hi = int(min(issued)), int(max(issued))
    if hi - lo >= fl.ISSUED_SPAN:
        raise ValueError("pending issue times span more than 2^40 µs; the packed sort key "
                         "cannot order them")
    return lo


def _ranks(ids: Sequence[str]) -> dict:
    if len(ids) >= fl.RANK_SPAN:
        raise ValueError("more than 2^24 pending requests in one planning round")
    rank = {t: i for i, t in enumerate(sorted(ids))}
    if len(rank) != len(ids):  # a repeated id collapsed into one entry
        raise ValueError("pending set holds more than one request for a task")
    return rank


def order_within_bucket(requests: Sequence[PendingRequest], exec_estimates: Mapping[str, Duration],
                        cfg: SchedulerConfig) -> list[PendingRequest]:
    """Descending aged estimate, then arrival, then task id (scheduler.py:107-117).

    Keys are packed on the host (hi = AGED_MAX - aged, lo = issued/rank word)
    and ordered by the device sort."""
    reqs = list(requests)
    if not reqs:
        return []
    rank = _ranks([r.task_id for r in reqs])
    issued = np.array([r.issued_at for r in reqs], np.int64)
    base = _issued_base(issued)
    keys = np.empty((len(reqs), 2), np.uint64)
    for i, r in enumerate(reqs):
        aged = exec_estimates[r.task_id] * (1 + r.skipped)
        if not 0 <= aged <= AGED_MAX:
            raise ValueError("aged execution estimate outside the packed key range")
        keys[i, 0] = AGED_MAX - aged
        keys[i, 1] = ((r.issued_at - base) << 24) | rank[r.task_id]
    kt = dev.tensor(keys.view(np.int64), torch.int64)
    ws = fl.Workspace(len(reqs))
    order, _ = fl.sort_keys(kt, ws)
    return [reqs[i] for i in order.cpu().tolist()]


def _checked_pending(pending: Iterable[PendingRequest],
                     states: Mapping[str, TaskState]) -> list[PendingRequest]:
    """The pending requests, validated (scheduler.py:245-251).  The reference
    sorts them by (issued_at, task_id) first; every result here is ordered by
    the unique packed keys, so the sort only decides which unknown task the
    error names -- it runs only when there is one."""
    reqs = list(pending)
    if not all(r.task_id in states for r in reqs):
        for req in sorted(reqs, key=lambda r: (r.issued_at, r.task_id)):
            if req.task_id not in states:
                raise ValueError(f"pending request references unknown task {req.task_id!r}")
    return reqs


def plan(pending: Iterable[PendingRequest], states: Mapping[str, TaskState], edge, cloud, net,
         now: TimePoint, cfg: SchedulerConfig, *, edge_in_flight: int = 0,
         cloud_in_flight: int = 0) -> DispatchPlan:
    """One planning round under the configured policy (scheduler.py:254-276).

    With `states` a `ledger.LedgerStates` (the simulator's task-state mapping
    backed by the device-resident incremental ledger), task histories are not
    re-packed: only the pending requests' scalars travel and the urgency pass
    reads each task's running wait total in O(1) (kr_urgency_ledger)."""
    reqs = _checked_pending(pending, states)
    edge_avail = max(0, edge.capacity - edge_in_flight) if edge is not None else 0
    cloud_avail = max(0, cloud.capacity - cloud_in_flight) if cloud is not None else 0
    n = len(reqs)
    if n == 0:
        return DispatchPlan(edge=(), cloud=(), deferred=(), refetch_task_ids=frozenset())
    if cfg.buckets > 256:
        raise ValueError("the packed sort key supports at most 256 buckets")
    rank = _ranks([r.task_id for r in reqs])
    base = _issued_base([r.issued_at for r in reqs])
    # the plan's keys need no control rate (need times are not part of it): hz = 1/1
    sched = _lib.KrSched(fl.POLICY_CODE[cfg.policy], cfg.buckets, cfg.aging_interval, 0,
                         cfg.stale_threshold, cfg.default_exec_estimate, int(now), 1, 1, base)
    ledger_backed = isinstance(states, _ledger.LedgerStates)
    no_cloud = cloud is None or net is None or cloud_avail == 0 or edge_avail >= n
    if not ledger_backed and no_cloud and n <= SMALL_PLAN_MAX:
        return _plan_small(reqs, states, rank, sched, min(edge_avail, n))
    flags = dev.flags()
    if ledger_backed:
        keys, view = states.ledger.urgency(reqs, states, rank, sched, flags)
    else:
        view = fl.DeviceFleet.from_host(fl.host_soa(reqs, states, rank))
        keys = fl.urgency(view, sched, need_time=False, flags=flags).keys
    return _place(reqs, states, keys, view, sched, flags, edge, cloud, net, edge_avail,
                  cloud_avail, edge_in_flight, cloud_in_flight)


# ---------------------------------------------------------------------------
# Small planning rounds: one launch, zero-copy staging (kr_plan_small)
# ---------------------------------------------------------------------------
SMALL_PLAN_MAX = 4096  # kr_plan_small's one-CTA bitonic sort


def _bumped(req, skipped: int):
    """dataclasses.replace(req, skipped=skipped) for an already validated
    request (scheduler.py:232-234): the copy's fields are the original's."""
    d = getattr(req, "__dict__", None)
    if d is None or not hasattr(type(req), "__dataclass_fields__"):
        return replace(req, skipped=skipped)
    new = object.__new__(type(req))
    new.__dict__.update(d)
    new.__dict__["skipped"] = skipped
    return new


def _plan_small(reqs, states, rank_of, sched, k) -> DispatchPlan:
    """Edge-tier plan() for n <= SMALL_PLAN_MAX in one launch + one sync."""
    n = len(reqs)
    fs, out, out_dev = fl.pack_mapped(reqs, states, rank_of, 4 * (3 * n + 1))
    out = out.view(np.int32)
    st = dev.raw_stream()
    _lib.check(_lib.load().kr_plan_small(ctypes.byref(fs), ctypes.byref(sched), k, out_dev,
                                         st), "kr_plan_small")
    dev.sync(st)
    f = int(out[3 * n]) & 0xFFFFFFFF
    if f & (_lib.FLAG_KEY_RANGE | _lib.FLAG_RATIO):
        raise ValueError("a pending request falls outside the packed sort-key range "
                         "(aged estimate >= 2^56 µs or lifetime >= 2^53 µs)")
    from . import _kr_pack
    a = out.ctypes.data  # order [n], refetch [n], skipped [n] (int32, mapped host memory)
    s_edge, deferred, refetch_ids = _kr_pack.finish(reqs, states, a, a + 4 * n, a + 8 * n, n, k,
                                                    0, _bumped)
    return DispatchPlan(edge=s_edge, cloud=(), deferred=deferred, refetch_task_ids=refetch_ids)


def _place(reqs, states, keys, fleet, sched, flags, edge, cloud, net, edge_avail, cloud_avail,
           edge_in_flight, cloud_in_flight) -> DispatchPlan:
    """Order, edge admission, cloud offload and the result objects, from the
    packed keys (scheduler.py:193-241)."""
    n = len(reqs)
    ws = fl.Workspace(n)
    order, sorted_keys = fl.sort_keys(keys, ws)
    k = min(edge_avail, n)
    kth_ptr = sorted_keys.data_ptr() + (k - 1) * 16 if 0 < k < n else None
    refetch = torch.empty(n, dtype=torch.uint8, device=keys.device)
    fl.admit(keys, k, kth_ptr, fleet, sched, None, refetch=refetch)
    n_cloud = 0
    cloud_idx = None
    if cloud is not None and net is not None and cloud_avail > 0 and k < n:
        # phase 3 (scheduler.py:210-221): per-round thresholds on the host,
        # per-request uplink times and the ordered offload scan on the device
        cap = min(cloud_avail, n - k)
        thr = eng.cloud_thresholds(edge, cloud, net, edge_in_flight, cloud_in_flight, k, cap)
        payload = dev.tensor(np.array([r.payload_bytes for r in reqs], np.int64), torch.int64)
        up = eng.transfer_time_batch(net, payload, eng.UP)
        thr_t = dev.tensor(np.array(thr, np.int64), torch.int64)
        cloud_idx = torch.empty(cap, dtype=torch.int32, device=keys.device)
        n_cloud_t = torch.zeros(1, dtype=torch.int32, device=keys.device)
        fs = fleet.c_struct()
        _lib.check(_lib.load().kr_place_cloud(
            order.data_ptr(), n, k, up.data_ptr(), thr_t.data_ptr(), cap, ctypes.byref(fs),
            ctypes.byref(sched), refetch.data_ptr(), cloud_idx.data_ptr(), n_cloud_t.data_ptr(),
            dev.stream()), "kr_place_cloud")
        n_cloud = int(n_cloud_t.item())
    # one device->host read of everything the result objects need
    out = torch.empty(3 * n + 1, dtype=torch.int32, device=keys.device)
    out[:n] = order
    out[n:2 * n] = refetch
    out[2 * n:3 * n] = fleet.t["skipped"]
    out[3 * n:] = flags
    host = out.cpu().numpy()
    f = int(host[3 * n]) & 0xFFFFFFFF
    if f & (_lib.FLAG_KEY_RANGE | _lib.FLAG_RATIO):
        raise ValueError("a pending request falls outside the packed sort-key range "
                         "(aged estimate >= 2^56 µs or lifetime >= 2^53 µs)")
    cloud_h = cloud_idx[:n_cloud].cpu().numpy() if n_cloud else np.zeros(0, np.int32)
    in_cloud = np.zeros(n, np.int32)
    in_cloud[cloud_h] = 1
    from . import _kr_pack
    host = np.ascontiguousarray(host)
    a = host.ctypes.data
    s_edge, deferred, refetch_ids = _kr_pack.finish(reqs, states, a, a + 4 * n, a + 8 * n, n, k,
                                                    in_cloud.ctypes.data if n_cloud else 0,
                                                    _bumped)
    s_cloud = tuple(reqs[i] for i in cloud_h)
    return DispatchPlan(edge=s_edge, cloud=s_cloud, deferred=deferred,
                        refetch_task_ids=refetch_ids)


def plan_fifo(pending, states, edge, cloud, net, now, cfg, **kw) -> DispatchPlan:
    return plan(pending, states, edge, cloud, net, now, replace(cfg, policy=FIFO), **kw)


def plan_las(pending, states, edge, cloud, net, now, cfg, **kw) -> DispatchPlan:
    return plan(pending, states, edge, cloud, net, now, replace(cfg, policy=LAS), **kw)
