"""Fleet-scale decision round: the production hot path.

One round = for every pending robot-round of the fleet
  (1) divergence horizon of the new chunk against the unexecuted overlap of
      the previous one (kr_horizon_divergence) -- or the confidence policy
      over update magnitudes (kr_horizon_confidence);
  (2) execution-aware urgency: next-need time and the packed priority key
      (kr_urgency);
  (3) top-k admission under the edge budget: device radix select of the k-th
      key, the admission pass (masks + skip counters) and the ordered S_e
      (kr_topk_select, kr_admit).
Everything is stream-ordered on the current CUDA stream with no host sync, so
a round can be captured in a CUDA graph.

Sharding (`ShardedDecisionRound`): one process per GPU owns a contiguous
range of robots.  Steps (1)-(2) are local.  Each rank selects its local top
k' = min(k, R_local) keys, the k'-key candidate lists are exchanged with one
NCCL all-gather over NVLink (the only cross-GPU traffic), and every rank runs
the same device select over the gathered keys.  The global k-th key decides
admission locally (key <= kth), which is exact because the global top k is a
subset of the union of local top-k' sets and keys are unique.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import _lib
from . import device as dev
from . import fleet as fl

ALL_ONES = -1  # int64 view of 0xFFFF...FFFF
SMALL_ADMIT_MAX = 16384  # kr_select.cu kSmallAdmit: admission sorts every key up to here


@dataclass
class RoundOutputs:
    horizon: torch.Tensor      # int32 [R]
    need_time: torch.Tensor    # int64 [R]
    keys: torch.Tensor         # int64 [R, 2] (kr_key)
    admitted: torch.Tensor     # uint8 [R]
    refetch: torch.Tensor      # uint8 [R]
    edge_keys: torch.Tensor    # int64 [k, 2] S_e keys in order (global when sharded)
    edge_idx: torch.Tensor | None = None  # int32 [k] local indices (single GPU)
    kth: torch.Tensor | None = None       # the k-th key (None when k == 0)
    flags: torch.Tensor | None = None     # int32 [1] validation word (DecisionRound.check)


@dataclass
class DivergenceInputs:
    prev: torch.Tensor                 # [R, Lp, D]
    cand: torch.Tensor                 # [R, Lc, D] or [R, S, Lc, D]
    threshold: float
    offset: torch.Tensor | None = None
    len_prev: torch.Tensor | None = None
    len_cand: torch.Tensor | None = None


@dataclass
class ConfidenceInputs:
    """The confidence-threshold (or static) policy over update magnitudes."""
    U: torch.Tensor                    # [R, K, N] fp32 / fp64
    cfg: object                        # horizon.HorizonPolicyConfig


@dataclass
class MixedInputs:
    """A heterogeneous fleet: horizon inputs per contiguous robot group, e.g.
    arms (64x7) and humanoids (64x32) as two homogeneous tensors (configs[2]).
    groups: [(first robot, DivergenceInputs | ConfidenceInputs)], covering
    the fleet.  The groups' horizon kernels run concurrently on forked streams."""
    groups: list


def raise_round_flags(f: int) -> None:
    """The validation bits of a fleet round -> the drop-in's ValueErrors."""
    if f & _lib.FLAG_DUP_KEY:
        raise ValueError("two shards produced the same priority key: sharded rounds need "
                         "global robot ranks (lexrank) and one issued base on every rank")
    if f & (_lib.FLAG_KEY_RANGE | _lib.FLAG_RATIO):
        raise ValueError("a pending request falls outside the packed sort-key range "
                         "(aged estimate >= 2^56 µs, issue-time span >= 2^40 µs, "
                         ">= 2^24 requests or lifetime >= 2^53 µs)")
    if f & _lib.FLAG_TIME_RANGE:
        raise ValueError("remaining actions must be >= 0 (or the need time overflows int64)")


class DecisionRound:
    """Preallocated single-GPU decision round over R robots, budget k."""

    one_graph_sequential = True  # sequential layout also captured as one graph

    def __init__(self, R: int, k: int, sched: _lib.KrSched):
        self.R = R
        self.k = min(k, R)
        self.sched = sched
        d = dev.device()
        self.H = torch.empty(R, dtype=torch.int32, device=d)
        self.need_time = torch.empty(R, dtype=torch.int64, device=d)
        self.keys = fl.new_keys(R, d)
        self.admitted = torch.empty(R, dtype=torch.uint8, device=d)
        self.refetch = torch.empty(R, dtype=torch.uint8, device=d)
        self.kth = fl.new_keys(1, d)
        self.edge_idx = torch.empty(max(self.k, 1), dtype=torch.int32, device=d)
        self.edge_keys = fl.new_keys(max(self.k, 1), d)
        self.ws = fl.Workspace(R)
        self.key_stats = fl.new_key_stats(d)
        # validation word: the urgency pass ORs KR_FLAG_KEY_RANGE / _RATIO /
        # _TIME_RANGE into it when a request falls outside the packed key's
        # range (plan() raises there); sticky across rounds until check()
        self.flags = dev.flags()
        self.lib = _lib.load()
        self.max_sms = 0  # divergence grid SM cap (0: all); see capture(concurrent=...)
        # the keys' OR / AND statistics feed only the radix select; rounds whose
        # admission sorts everything (R <= 16,384: kr_select.cu kSmallAdmit) or
        # selects nothing skip them (one launch less per round; a select that
        # gets no statistics computes its own, so a wrong guess costs only time)
        self.stats_needed = not (type(self) is DecisionRound and
                                 (R <= SMALL_ADMIT_MAX or self.k == 0 or self.k >= R))
        # rounds that run the radix select: the urgency pass's last CTA prepares
        # the select state from per-CTA statistics (kr_urgency_prep /
        # kr_select_admit_prepared: two launches fewer)
        self.prepared = (type(self) is DecisionRound and self.stats_needed
                         and not os.environ.get("KR_ROUND_NO_PREP"))
        if self.prepared:
            self.ws.buf.zero_()  # the state's last-CTA counter starts at 0

    def horizons(self, h) -> None:
        if isinstance(h, MixedInputs):
            self._horizons_mixed(h)
            return
        self._horizon_into(self.H, h)

    def _horizons_mixed(self, h: MixedInputs) -> None:
        main = torch.cuda.current_stream()
        if len(h.groups) == 1:
            start, g = h.groups[0]
            self._horizon_into(self.H[start:], g)
            return
        if not hasattr(self, "group_streams"):
            self.group_streams = []
        while len(self.group_streams) < len(h.groups):
            self.group_streams.append(torch.cuda.Stream(device=self.H.device))
        fork = torch.cuda.Event()
        fork.record(main)
        for (start, g), st in zip(h.groups, self.group_streams):
            st.wait_event(fork)
            with torch.cuda.stream(st):
                self._horizon_into(self.H[start:], g)
        for st in self.group_streams[: len(h.groups)]:
            main.wait_stream(st)

    def _horizon_into(self, H: torch.Tensor, h) -> None:
        if isinstance(h, ConfidenceInputs):
            from .horizon import decide_horizon_batch
            decide_horizon_batch(h.cfg, h.U, out=H[: h.U.shape[0]], validate=False,
                                 max_sms=self.max_sms)
            return
        prev, cand = h.prev, h.cand
        if cand.dim() == 3:
            cand = cand.unsqueeze(1)
        R, Lp, D = prev.shape
        S, Lc = cand.shape[1], cand.shape[2]
        dtype = _lib.KR_F64 if prev.dtype == torch.float64 else _lib.KR_F32
        _lib.check(self.lib.kr_horizon_divergence(
            prev.data_ptr(), cand.data_ptr(), dtype, R, S, Lp, Lc, D, _lib.ptr(h.offset),
            _lib.ptr(h.len_prev), _lib.ptr(h.len_cand), float(h.threshold), H.data_ptr(),
            None, self.max_sms, dev.stream()), "kr_horizon_divergence")

    def urgency(self, fleet: fl.DeviceFleet) -> None:
        st = dev.stream()
        fs = fleet.c_struct()
        if self.prepared:
            _lib.check(self.lib.kr_urgency_prep(
                ctypes.byref(fs), ctypes.byref(self.sched), self.keys.data_ptr(),
                self.need_time.data_ptr(), self.flags.data_ptr(), self.k, self.ws.ptr(),
                self.ws.nbytes, st), "kr_urgency_prep")
            return
        if self.stats_needed:
            _lib.check(self.lib.kr_key_stats_init(self.key_stats.data_ptr(), st),
                       "kr_key_stats_init")
        _lib.check(self.lib.kr_urgency(
            ctypes.byref(fs), ctypes.byref(self.sched), self.keys.data_ptr(),
            self.need_time.data_ptr(), None, None, None, None, None,
            self.key_stats.data_ptr() if self.stats_needed else None, self.flags.data_ptr(), st),
            "kr_urgency")

    def check(self, reset: bool = True) -> None:
        """Raise the reference's ValueError if any round since the last check
        met an input outside the packed sort key's range (one 4-byte read;
        call it outside graph capture, e.g. every N rounds or at the end of a
        replay).  The decisions of such a round are not the reference's."""
        f = dev.read_flags(self.flags)
        if reset and f:
            self.flags.zero_()
        raise_round_flags(f)

    def admit(self, fleet: fl.DeviceFleet) -> None:
        if self.prepared:
            fs = fleet.c_struct()
            _lib.check(self.lib.kr_select_admit_prepared(
                self.keys.data_ptr(), self.R, self.k, ctypes.byref(fs), ctypes.byref(self.sched),
                self.admitted.data_ptr(), self.refetch.data_ptr(), self.edge_idx.data_ptr(),
                self.edge_keys.data_ptr(), self.kth.data_ptr(), self.ws.ptr(), self.ws.nbytes,
                dev.stream()), "kr_select_admit_prepared")
            return
        fl.select_admit(self.keys, self.k, self.ws,
                        key_stats=self.key_stats if self.stats_needed else None, fleet=fleet,
                        sched=self.sched, admitted=self.admitted, refetch=self.refetch,
                        edge_idx=self.edge_idx, edge_keys=self.edge_keys, kth=self.kth)

    def outputs(self) -> RoundOutputs:
        return RoundOutputs(self.H, self.need_time, self.keys, self.admitted, self.refetch,
                            self.edge_keys[: self.k], self.edge_idx[: self.k],
                            self.kth if self.k else None, self.flags)

    def run(self, fleet: fl.DeviceFleet, h: DivergenceInputs) -> RoundOutputs:
        self.horizons(h)
        self.urgency(fleet)
        self.admit(fleet)
        return self.outputs()

    def capture(self, fleet: fl.DeviceFleet, h: DivergenceInputs, reserve_sms: int = 0,
                layout: str = "split") -> None:
        """Record the round as CUDA graphs over these fixed device buffers.

        layout "split": horizons | urgency + admission.  With `reserve_sms` > 0
        the divergence grid leaves that many SMs free and `replay()` runs the
        two graphs on two streams: urgency and admission do not depend on this
        round's horizons (the reference's order uses history, not H), so they
        overlap the HBM-bound horizon kernel on the reserved SMs.
        layout "urgency_first": the HBM-streaming urgency pass first on the
        whole GPU, then the horizon kernel on all but `reserve_sms` SMs while
        the latency-bound admission (select, admit, sort of S_e) runs on the
        side stream."""
        if layout not in ("split", "urgency_first"):
            raise ValueError(f"unknown round layout {layout!r}")
        self.layout = layout
        # reserve_sms < 0: concurrent without an SM cap (side kernels co-reside
        # wherever the horizon kernel leaves room)
        self.max_sms = 0 if reserve_sms <= 0 else max(1, torch.cuda.get_device_properties(
            self.H.device).multi_processor_count - reserve_sms)
        self.run(fleet, h)  # warm-up: attribute / occupancy caches, lazy loading
        torch.cuda.synchronize()
        self.g_horizon, self.g_decide = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        self.g_urgency = None
        with torch.cuda.graph(self.g_horizon):
            self.horizons(h)
        if layout == "urgency_first":
            self.g_urgency = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.g_urgency):
                self.urgency(fleet)
            with torch.cuda.graph(self.g_decide):
                self.admit(fleet)
        else:
            with torch.cuda.graph(self.g_decide):
                self.urgency(fleet)
                self.admit(fleet)
        self.side = torch.cuda.Stream(device=self.H.device) if reserve_sms != 0 else None
        # sequential rounds (no side stream) also as one graph: one launch per
        # round, and the urgency pass's programmatic launch overlaps the horizon
        # kernel's tail (configs[1]: 20.7 -> see DESIGN "The round")
        self.g_seq = None
        if self.side is None and layout == "split" and self.one_graph_sequential:
            self.g_seq = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.g_seq):
                self.horizons(h)
                self.urgency(fleet)
                self.admit(fleet)

    def replay_concurrent(self, before_horizon=None, after_horizon=None, before_side=None,
                          after_side=None) -> None:
        """One round from the captured graphs.  With reserved SMs the horizon
        graph is launched first on the current stream and the urgency +
        admission graph on the side stream (ordered after all prior work of the
        current stream, not after the horizons); the current stream joins the
        side stream at the end.  `before_horizon` / `after_horizon` (callables)
        may record events around the horizon graph."""
        main = torch.cuda.current_stream()
        if getattr(self, "g_seq", None) is not None and not (before_horizon or after_horizon):
            self.g_seq.replay()
            return
        if self.g_urgency is not None:
            self.g_urgency.replay()  # the side stream forks after it
        if self.side is None:
            if before_horizon:
                before_horizon(main)
            self.g_horizon.replay()
            if after_horizon:
                after_horizon(main)
            self.g_decide.replay()
            return
        fork = torch.cuda.Event()
        fork.record(main)
        if before_horizon:
            before_horizon(main)
        self.g_horizon.replay()
        if after_horizon:
            after_horizon(main)
        self.side.wait_event(fork)
        with torch.cuda.stream(self.side):
            if before_side:
                before_side(self.side)
            self.g_decide.replay()
            if after_side:
                after_side(self.side)
        main.wait_stream(self.side)

    def replay(self) -> RoundOutputs:
        self.replay_concurrent()
        return self.outputs()

    def run_overlapped(self, fleet: fl.DeviceFleet, h: DivergenceInputs, reserve_sms: int = 8,
                       before_horizon=None, after_horizon=None,
                       layout: str = "split") -> RoundOutputs:
        """One eager round with the graph path's overlap (see `capture`): the
        horizon kernel on the current stream over all but `reserve_sms` SMs and
        the admission (for a sharded round: local select, the NCCL all-gather
        of candidates, global select, local admission) on a side stream
        concurrently -- preceded on the current stream by the urgency pass
        ("urgency_first") or running it on the side stream too ("split"); the
        current stream joins the side stream at the end.  (A sharded round over
        NCCL is captured too -- `capture` -- with the all-gather inside the
        admission graph; over gloo it runs here.)"""
        n_sm = torch.cuda.get_device_properties(self.H.device).multi_processor_count
        self.max_sms = 0 if reserve_sms <= 0 else max(1, n_sm - reserve_sms)
        if getattr(self, "side", None) is None:
            self.side = torch.cuda.Stream(device=self.H.device)
        main = torch.cuda.current_stream()
        if layout == "urgency_first":
            self.urgency(fleet)
        fork = torch.cuda.Event()
        fork.record(main)
        if before_horizon:
            before_horizon(main)
        self.horizons(h)
        if after_horizon:
            after_horizon(main)
        self.side.wait_event(fork)
        with torch.cuda.stream(self.side):
            if layout != "urgency_first":
                self.urgency(fleet)
            self.admit(fleet)
        main.wait_stream(self.side)
        return self.outputs()


class HybridDecisionRound(DecisionRound):
    """Single-GPU fleet round with the phase-3 cloud tier (scheduler.py:193-234,
    §8(f)1 at fleet scale): edge admission of the first k in key order
    (kr_admit), then the ordered offload scan over the following ranks
    (kr_place_cloud) against the round's per-count thresholds
    T(c) = edge_est - (drain(c) + batch(c+1) + down) (engines.cloud_thresholds,
    host integers) and the requests' uplink times.

    The scan usually fills the cloud slots within a few thousand ranks, so the
    order is only materialised for the first k + window ranks (the fused
    select, no side effects); when the scan reaches the end of that window
    with slots left (one 4-byte read back), the full key order is sorted and
    the scan re-run over it (the placement is idempotent).  Outputs: the
    round's `outputs()` (edge = order[:k]) plus `cloud()` in offload order;
    deferred = everything else."""

    def __init__(self, R: int, k: int, sched: _lib.KrSched, cloud_cap: int,
                 window: int | None = None):
        super().__init__(R, k, sched)
        d = dev.device()
        self.cap = max(0, min(int(cloud_cap), R - self.k))
        self.kp = min(R, self.k + (window if window is not None else max(2 * self.cap, 4096)))
        self.cand_idx = torch.empty(max(self.kp, 1), dtype=torch.int32, device=d)
        self.cand_keys = fl.new_keys(max(self.kp, 1), d)
        self.order = None  # full order (fallback only)
        self.sorted_keys = None
        self.cloud_idx = torch.empty(max(self.cap, 1), dtype=torch.int32, device=d)
        self.n_cloud = torch.zeros(1, dtype=torch.int32, device=d)
        self.up_us = None
        self.thresholds = None
        self.full_sorts = 0  # rounds that needed the full order (diagnostic)

    def set_cloud(self, up_us: torch.Tensor, thresholds) -> None:
        """up_us [R] int64 (engines.transfer_time_batch of each request's
        payload); thresholds: T(c) for c < cap (engines.cloud_thresholds)."""
        if up_us.shape[0] != self.R or up_us.dtype != torch.int64:
            raise ValueError("up_us must be an int64 tensor of R uplink times")
        thr = torch.as_tensor(list(thresholds)[: self.cap], dtype=torch.int64)
        if thr.numel() < self.cap:
            raise ValueError("need a threshold for every cloud slot")
        self.up_us = up_us
        self.thresholds = thr.to(up_us.device)

    def _place(self, fleet, order: torch.Tensor, n: int) -> None:
        fs = fleet.c_struct()
        _lib.check(self.lib.kr_place_cloud(
            order.data_ptr(), n, self.k, self.up_us.data_ptr(), self.thresholds.data_ptr(),
            self.cap, ctypes.byref(fs), ctypes.byref(self.sched), self.refetch.data_ptr(),
            self.cloud_idx.data_ptr(), self.n_cloud.data_ptr(), dev.stream()), "kr_place_cloud")

    def admit(self, fleet: fl.DeviceFleet) -> None:
        k, R = self.k, self.R
        if self.cap > 0 and self.up_us is None:
            raise RuntimeError("set_cloud() first: the round has a cloud tier")
        # the ordered first kp ranks, no side effects
        fl.select_admit(self.keys, self.kp, self.ws, key_stats=self.key_stats,
                        edge_idx=self.cand_idx, edge_keys=self.cand_keys)
        kth_ptr = self.cand_keys.data_ptr() + (k - 1) * 16 if 0 < k < R else None
        if 0 < k < R:
            self.kth.copy_(self.cand_keys[k - 1: k])
        else:  # k >= R: every key is admitted (kr_topk_select's convention)
            self.kth.fill_(ALL_ONES)
        fl.admit(self.keys, k, kth_ptr, fleet, self.sched, None, admitted=self.admitted,
                 refetch=self.refetch)
        if self.cap == 0:
            self.n_cloud.zero_()
            return
        self._place(fleet, self.cand_idx, self.kp)
        if self.kp < R and int(self.n_cloud.item()) < self.cap:
            if self.order is None:
                self.order = torch.empty(R, dtype=torch.int32, device=self.keys.device)
                self.sorted_keys = fl.new_keys(R, self.keys.device)
            fl.sort_keys(self.keys, self.ws, order=self.order, sorted_keys=self.sorted_keys)
            self._place(fleet, self.order, R)
            self.full_sorts += 1

    def outputs(self) -> RoundOutputs:
        return RoundOutputs(self.H, self.need_time, self.keys, self.admitted, self.refetch,
                            self.cand_keys[: self.k], self.cand_idx[: self.k],
                            self.kth if self.k else None, self.flags)

    def cloud(self) -> torch.Tensor:
        """The offloaded robots in offload order (one device->host read)."""
        return self.cloud_idx[: int(self.n_cloud.item())]

    def full_order(self) -> torch.Tensor:
        """The complete key order (sorted on demand when the round did not)."""
        if self.order is None:
            self.order = torch.empty(self.R, dtype=torch.int32, device=self.keys.device)
            self.sorted_keys = fl.new_keys(self.R, self.keys.device)
        fl.sort_keys(self.keys, self.ws, order=self.order, sorted_keys=self.sorted_keys)
        return self.order


def sharded_topk(keys, n_local: int, k: int, sizes: list, ops, group=None):
    """Exact global top-k admission over robot-sharded keys (host protocol).

    `ops` supplies the device primitives (product: `CudaShardOps`; the CPU
    tests plug in a numpy twin to exercise this protocol under gloo):
      local_candidates(keys, kl, kg) -> [kg, 2] local top-kl keys ascending,
                                        sentinel-padded
      all_gather(cand)               -> [W * kg, 2] (W sorted runs)
      merge(runs, W, kg, want_kth)   -> (global S_e keys [kg, 2] in order,
                                         the kg-th key or None)
      apply(keys, k, kth)            -> local admission (masks, skip counters)
    Exact: the global top-kg is a subset of the union of the local top-kl
    lists, so merging the sorted runs and keeping ranks < kg gives it in order.
    Returns (k_global, global ordered S_e keys).
    """
    world = len(sizes)
    total = sum(sizes)
    kg = min(k, total)
    kl = min(kg, n_local)
    cand = ops.local_candidates(keys, kl, kg)
    gathered = ops.all_gather(cand)
    edge, kth = None, None
    if kg > 0:
        edge, kth = ops.merge(gathered, world, kg, kg < total)
    ops.apply(keys, kg, kth)
    return kg, edge


class CudaShardOps:
    """sharded_topk primitives as C-ABI calls on preallocated device buffers."""

    def __init__(self, rnd: "ShardedDecisionRound", fleet: fl.DeviceFleet):
        self.r = rnd
        self.fleet = fleet

    def local_candidates(self, keys, kl, kg):
        # fused select + gather + sort of the local top-kl (no side effects:
        # no fleet / masks), sentinel padding beyond kl
        r, st = self.r, dev.stream()
        r.cand.fill_(ALL_ONES)
        if kl > 0:
            _lib.check(r.lib.kr_select_admit(keys.data_ptr(), r.R, kl, r.key_stats.data_ptr(),
                                             None, None, None, None, None, r.cand.data_ptr(),
                                             None, r.ws.ptr(), r.ws.nbytes, st),
                       "kr_select_admit(local candidates)")
        return r.cand

    def all_gather(self, cand):
        # the only cross-GPU traffic of a round: W x k' x 16 B over NVLink (NCCL)
        if dist.get_backend(self.r.group) == "nccl":
            dist.all_gather_into_tensor(self.r.gathered, cand, group=self.r.group)
        else:  # gloo (tests: several ranks sharing one device)
            parts = list(self.r.gathered.chunk(self.r.world))
            dist.all_gather(parts, cand, group=self.r.group)
        return self.r.gathered

    def merge(self, runs, W, kg, want_kth):
        r = self.r
        _lib.check(r.lib.kr_merge_runs(runs.data_ptr(), W, kg, kg, r.global_edge.data_ptr(),
                                       r.kth_global.data_ptr() if want_kth else None,
                                       r.flags.data_ptr(), dev.stream()), "kr_merge_runs")
        return r.global_edge[:kg], (r.kth_global if want_kth else None)

    def apply(self, keys, k, kth):
        r = self.r
        fs = self.fleet.c_struct()
        _lib.check(r.lib.kr_admit(keys.data_ptr(), r.R, k, _lib.ptr(kth), ctypes.byref(fs),
                                  ctypes.byref(r.sched), r.admitted.data_ptr(),
                                  r.refetch.data_ptr(), None, None, None, 0, dev.stream()),
                   "kr_admit(apply)")


class ShardedDecisionRound(DecisionRound):
    """Robot-sharded round: local steps + one all-gather of top-k' candidates.

    `k` is the global edge budget.  Requires torch.distributed (NCCL on GPUs)."""

    def __init__(self, R_local: int, k: int, sched: _lib.KrSched, group=None):
        super().__init__(R_local, k, sched)
        self.k_request = k  # the global budget (self.k is clamped to the local shard)
        self.group = group
        self.world = dist.get_world_size(group)
        sizes = torch.tensor([R_local], dtype=torch.int64, device=self.H.device)
        allsz = [torch.zeros_like(sizes) for _ in range(self.world)]
        dist.all_gather(allsz, sizes, group=group)
        self.sizes = [int(s.item()) for s in allsz]
        # keys are comparable across shards only if every rank packs them
        # against the same round scalars (issued base, now, policy)
        mine = torch.tensor([sched.issued_base, sched.now, sched.policy, sched.buckets,
                             sched.aging_interval], dtype=torch.int64, device=self.H.device)
        every = [torch.zeros_like(mine) for _ in range(self.world)]
        dist.all_gather(every, mine, group=group)
        if any(not torch.equal(e, every[0]) for e in every):
            raise ValueError("sharded round: every rank needs the same kr_sched issued_base, now "
                             "and policy (keys are compared across shards)")
        self.k_global = min(k, sum(self.sizes))
        kg = max(self.k_global, 1)
        d = self.H.device
        self.cand = fl.new_keys(kg, d)
        self.gathered = fl.new_keys(kg * self.world, d)
        self.kth_global = fl.new_keys(1, d)
        self.global_edge = fl.new_keys(kg, d)

    def admit(self, fleet: fl.DeviceFleet) -> None:
        sharded_topk(self.keys, self.R, self.k_request, self.sizes, CudaShardOps(self, fleet),
                     self.group)

    one_graph_sequential = False  # one capture of the NCCL all-gather per round graph

    def capture(self, fleet: fl.DeviceFleet, h, reserve_sms: int = 0,
                layout: str = "split") -> None:
        """CUDA graphs of the sharded round (see DecisionRound.capture): the
        NCCL all-gather of the candidates is captured inside the admission
        graph -- every op of the protocol works on preallocated buffers with
        no host synchronisation -- so a replay is one enqueue per graph.  The
        warm-up round inside DecisionRound.capture initialises the
        communicator before capture.  NCCL only: gloo collectives run on the
        host (use run / run_overlapped)."""
        if dist.get_backend(self.group) != "nccl":
            raise RuntimeError("a sharded round is captured only over NCCL (gloo runs eagerly)")
        super().capture(fleet, h, reserve_sms=reserve_sms, layout=layout)

    def outputs(self) -> RoundOutputs:
        return RoundOutputs(self.H, self.need_time, self.keys, self.admitted, self.refetch,
                            self.global_edge[: self.k_global], None, self.kth_global)


class ShardedHybridRound(ShardedDecisionRound):
    """Robot-sharded round with the phase-3 cloud tier (SURVEY §8(e) extension).

    Every rank contributes its ordered local top k + window candidates with
    their uplink times; one all-gather, the same merge on every rank (keeping
    each candidate's position so its uplink time follows it): the merged first
    k ranks are the global S_e (edge admission by the k-th key, exactly as the
    edge-only protocol), and the same ordered offload scan runs over the
    following ranks (kr_place_cloud) -- identical on every rank.  If the scan
    runs out of ranks with slots left, every rank widens the window 4x and
    repeats the cloud part (the decision is the same everywhere).  Each rank
    then applies the placements of its own robots (skip counter reset,
    stale-observation refetch).  up_us: this shard's uplink times;
    thresholds: the global T(c)."""

    def __init__(self, R_local: int, k: int, sched: _lib.KrSched, cloud_cap: int, group=None,
                 window: int | None = None):
        super().__init__(R_local, k, sched, group)
        self.rank = dist.get_rank(group)
        self.total = sum(self.sizes)
        self.cap = max(0, min(int(cloud_cap), self.total - self.k_global))
        self.window = window if window is not None else max(2 * self.cap, 4096)
        self.up_us = None
        self.thresholds = None
        self.widened = 0
        self.cloud_keys = fl.new_keys(max(self.cap, 1), self.H.device)
        self.n_cloud = 0

    def set_cloud(self, up_us: torch.Tensor, thresholds) -> None:
        if up_us.shape[0] != self.R or up_us.dtype != torch.int64:
            raise ValueError("up_us must be an int64 tensor of this shard's uplink times")
        thr = torch.as_tensor(list(thresholds)[: self.cap], dtype=torch.int64)
        if thr.numel() < self.cap:
            raise ValueError("need a threshold for every cloud slot")
        self.up_us = up_us
        self.thresholds = thr.to(up_us.device)

    def _gather(self, t: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
        if dist.get_backend(self.group) == "nccl":
            dist.all_gather_into_tensor(out, t, group=self.group)
        else:  # gloo (tests: several ranks sharing one device)
            dist.all_gather(list(out.chunk(self.world)), t, group=self.group)
        return out

    def _buffers(self, kg2: int) -> dict:
        """Per-window device buffers, allocated once per window size (the
        steady state never allocates: the window only widens, rarely)."""
        if getattr(self, "_buf_kg2", None) != kg2:
            d, n = self.H.device, max(kg2, 1)
            self._buf = {
                "cand_keys": fl.new_keys(n, d),
                "cand_idx": torch.zeros(n, dtype=torch.int32, device=d),
                "cand_up": torch.zeros(n, dtype=torch.int64, device=d),
                "g_keys": fl.new_keys(n * self.world, d),
                "g_up": torch.zeros(n * self.world, dtype=torch.int64, device=d),
                "merged": fl.new_keys(n, d),
                "pos": torch.empty(n, dtype=torch.int32, device=d),
                "cloud_pos": torch.zeros(max(self.cap, 1), dtype=torch.int32, device=d),
                "n_cloud": torch.zeros(1, dtype=torch.int32, device=d),
            }
            self._buf_kg2 = kg2
        return self._buf

    def _candidates(self, kg2: int, b: dict) -> None:
        """This shard's ordered top min(kg2, R) keys (sentinel-padded to kg2),
        their local indices and uplink times; no side effects."""
        kl2 = min(kg2, self.R)
        b["cand_keys"].fill_(ALL_ONES)
        if kl2 > 0:
            fl.select_admit(self.keys, kl2, self.ws, key_stats=self.key_stats,
                            edge_idx=b["cand_idx"], edge_keys=b["cand_keys"])
            if self.cap > 0:
                torch.index_select(self.up_us, 0, b["cand_idx"][:kl2], out=b["cand_up"][:kl2])

    def admit(self, fleet: fl.DeviceFleet) -> None:
        """One select, one all-gather of (key, uplink) candidates and one merge
        serve both tiers: the merged first k_global ranks are the global S_e
        (edge admission by the k-th key, as in the edge-only protocol), the
        following ranks feed the offload scan.  Preallocated buffers; the one
        host read is the offload count, deciding whether the window must widen
        (the same decision on every rank)."""
        if self.cap > 0 and self.up_us is None:
            raise RuntimeError("set_cloud() first: the round has a cloud tier")
        st = dev.stream()
        kg = self.k_global
        window = self.window if self.cap > 0 else 0
        edge_done = False
        self.n_cloud = 0
        while True:
            kg2 = min(kg + window, self.total)
            b = self._buffers(kg2)
            self._candidates(kg2, b)
            g_keys = self._gather(b["cand_keys"][:max(kg2, 1)], b["g_keys"])
            g_up = self._gather(b["cand_up"][:max(kg2, 1)], b["g_up"]) if self.cap > 0 else None
            if kg2 > 0:
                _lib.check(self.lib.kr_merge_runs_pos(g_keys.data_ptr(), self.world, kg2, kg2,
                                                      b["merged"].data_ptr(), b["pos"].data_ptr(),
                                                      None, self.flags.data_ptr(), st),
                           "kr_merge_runs_pos")
            if not edge_done:  # global S_e and the local edge admission
                if kg > 0:
                    self.global_edge[:kg].copy_(b["merged"][:kg])
                    self.kth_global.copy_(b["merged"][kg - 1: kg])
                kth = self.kth_global if 0 < kg < self.total else None
                CudaShardOps(self, fleet).apply(self.keys, kg, kth)
                edge_done = True
            if self.cap == 0:
                return
            _lib.check(self.lib.kr_place_cloud(
                b["pos"].data_ptr(), kg2, kg, g_up.data_ptr(), self.thresholds.data_ptr(),
                self.cap, None, None, None, b["cloud_pos"].data_ptr(), b["n_cloud"].data_ptr(),
                st), "kr_place_cloud")
            n = int(b["n_cloud"].item())
            if n == self.cap or kg2 == self.total:
                break
            window *= 4
            self.widened += 1
        self.n_cloud = n
        # offload order as keys (entries past n are never read), and this
        # shard's placements applied on the device (skip reset + refetch)
        torch.index_select(g_keys, 0, b["cloud_pos"].long(), out=self.cloud_keys)
        fs = fleet.c_struct()
        _lib.check(self.lib.kr_apply_placements(
            b["cloud_pos"].data_ptr(), b["n_cloud"].data_ptr(), self.cap, kg2, self.rank,
            b["cand_idx"].data_ptr(), ctypes.byref(fs), ctypes.byref(self.sched),
            self.refetch.data_ptr(), st), "kr_apply_placements")

    def cloud(self) -> torch.Tensor:
        """The global offload set as keys, in offload order (same on every rank)."""
        return self.cloud_keys[: self.n_cloud]
