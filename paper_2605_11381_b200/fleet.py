"""Device-resident fleet state and the batched decision round.

Layout in HBM (structure-of-arrays, one entry per pending request; see
DESIGN.md "Data layout"):

    t_start, issued_at, obs_captured_at, accum_gen, hist_off : int64 [R]
    remaining, lexrank, skipped, n_exec, n_gen               : int32 [R]
    slots                                                    : int64 [S, 4]
        (gen_start, gen_end, exec_start, exec_end) per recorded round, CSR by
        hist_off; a robot has max(n_exec, n_gen) slots, the last one holding
        only the start of an in-flight successor generation.
    keys                                                     : kr_key [R] (16 B)

`DeviceFleet.from_objects` packs reference-shaped TaskState / PendingRequest
objects (any object with the reference's attribute names) into that layout;
`urgency` and `admit` are the step-2 / step-3 kernels over it.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Mapping, Sequence

import numpy as np
import torch

from . import _lib
from . import device as dev

INT_FIELDS64 = ("t_start", "issued_at", "obs_captured_at", "accum_gen", "hist_off")
INT_FIELDS32 = ("remaining", "lexrank", "skipped", "n_exec", "n_gen")
POLICY_CODE = {"kairos": _lib.KR_KAIROS, "fifo": _lib.KR_FIFO, "las": _lib.KR_LAS}
ISSUED_SPAN = 1 << 40
RANK_SPAN = 1 << 24


def host_soa(pending: Sequence, states: Mapping, rank_of: Mapping[str, int]) -> dict:
    """Reference-shaped objects -> numpy structure-of-arrays (host packing by
    the native packer, _kr_pack: one pass over the objects in C)."""
    from . import _kr_pack
    n = len(pending)
    cap = 1024 + 60 * n + 128 * n
    while True:
        buf = np.empty(cap, np.uint8)
        offs = _kr_pack.pack(pending, states, rank_of, buf.ctypes.data, cap, 0)
        if offs is not None:
            break
        cap *= 2
    osl, o32, _, nsl = offs
    c64 = buf[:40 * n].view(np.int64).reshape(5, n)
    c32 = buf[o32:o32 + 20 * n].view(np.int32).reshape(5, n)
    a = {k: c64[j] for j, k in enumerate(("t_start", "issued_at", "obs_captured_at", "accum_gen",
                                           "hist_off"))}
    a.update({k: c32[j] for j, k in enumerate(INT_FIELDS32)})
    a["slots"] = buf[osl:osl + 32 * nsl].view(np.int64).reshape(nsl, 4)
    a["n"] = n
    return a


def pack_mapped(reqs, states, rank_of, out_bytes: int) -> tuple:
    """host_soa's columns written straight into the mapped arena
    (device.MappedArena) by the native packer (_kr_pack, csrc/kr_pack.c: one
    pass over the objects in C), plus `out_bytes` of output space: returns
    (kr_fleet over the mapped device addresses, the output region as a uint8
    host view, its device address).  The arena is reused by the next call on
    this thread."""
    from . import _kr_pack
    n = len(reqs)
    a = dev.arena()
    while True:
        offs = _kr_pack.pack(reqs, states, rank_of, a.blob.data_ptr(), a.nbytes, out_bytes)
        if offs is not None:
            break
        a = dev.arena(2 * a.nbytes)
    osl, o32, oout, _ = offs
    d, d32 = a.dbase, a.dbase + o32
    fs = _lib.KrFleet(n, d, d + 8 * n, d + 16 * n, d + 24 * n, d32, d32 + 4 * n, d32 + 8 * n,
                      d + 32 * n, d32 + 12 * n, d32 + 16 * n, d + osl)
    return fs, a.host[oout:oout + out_bytes], d + oout


@dataclass
class DeviceFleet:
    """Fleet SoA resident on one GPU (tensors are owned by this object)."""

    n: int
    t: dict  # name -> CUDA tensor

    @classmethod
    def from_host(cls, soa: Mapping) -> "DeviceFleet":
        """One host->device copy of every column (packed into one pinned blob,
        each field 256-byte aligned like its own allocation, then viewed per
        field on the device): a planning call with a few requests pays one
        transfer, not eleven."""
        d = dev.device()
        n = int(soa["n"])
        slots = np.ascontiguousarray(np.asarray(soa["slots"], np.int64).reshape(-1))
        fields = [(k, np.int64, n) for k in INT_FIELDS64] + [("slots", np.int64, slots.size)] + \
                 [(k, np.int32, n) for k in INT_FIELDS32]
        offs, off = [], 0
        for _, dt, cnt in fields:
            offs.append(off)
            off += (np.dtype(dt).itemsize * cnt + 255) // 256 * 256
        blob = torch.empty(max(off, 256), dtype=torch.uint8, pin_memory=True)
        hb = blob.numpy()
        for (k, dt, cnt), o in zip(fields, offs):
            src = slots if k == "slots" else np.asarray(soa[k], dt)
            hb[o:o + np.dtype(dt).itemsize * cnt].view(dt)[:] = src
        g = blob.to(d, non_blocking=True)
        tdt = {np.int64: torch.int64, np.int32: torch.int32}
        t = {}
        for (k, dt, cnt), o in zip(fields, offs):
            t[k] = g[o:o + np.dtype(dt).itemsize * cnt].view(tdt[dt])
        t["slots"] = t["slots"].view(-1, 4)
        torch.cuda.current_stream(d).synchronize()  # the pinned blob is released on return
        return cls(n, t)

    @classmethod
    def from_tensors(cls, tensors: Mapping[str, torch.Tensor]) -> "DeviceFleet":
        t = dict(tensors)
        return cls(int(t["issued_at"].numel()), t)

    @classmethod
    def from_objects(cls, pending: Sequence, states: Mapping,
                     rank_of: Mapping[str, int] | None = None) -> "DeviceFleet":
        if rank_of is None:
            rank_of = {tid: i for i, tid in enumerate(sorted(r.task_id for r in pending))}
        return cls.from_host(host_soa(pending, states, rank_of))

    def c_struct(self) -> _lib.KrFleet:
        t = self.t
        return _lib.KrFleet(self.n, *[t[k].data_ptr() for k in (
            "t_start", "issued_at", "obs_captured_at", "accum_gen", "remaining", "lexrank",
            "skipped", "hist_off", "n_exec", "n_gen", "slots")])


def sched_struct(policy: str, buckets: int, aging_interval: int, stale_threshold: int,
                 default_exec_estimate: int, now: int, control_hz, issued_base: int) -> _lib.KrSched:
    num, den = dev.hz_ratio(control_hz)
    return _lib.KrSched(POLICY_CODE[policy], buckets, aging_interval, 0, stale_threshold,
                        default_exec_estimate, now, num, den, issued_base)


@dataclass
class UrgencyOut:
    keys: torch.Tensor            # uint8 view of kr_key [R] (int64 [R, 2])
    need_time: torch.Tensor | None = None
    total_wait: torch.Tensor | None = None
    wr: torch.Tensor | None = None
    bucket: torch.Tensor | None = None
    est: torch.Tensor | None = None
    slot_wait: torch.Tensor | None = None


def new_keys(n: int, device=None) -> torch.Tensor:
    """Storage for n kr_key (16-byte) keys: int64 [n, 2] = (hi, lo)."""
    return torch.empty((max(n, 0), 2), dtype=torch.int64, device=device or dev.device())


def urgency(fleet: DeviceFleet, sched: _lib.KrSched, *, need_time=True, intermediates=False,
            slot_waits=False, keys: torch.Tensor | None = None, flags: torch.Tensor | None = None,
            key_stats: torch.Tensor | None = None) -> UrgencyOut:
    """Step 2 over the whole fleet: one fused kernel (kr_urgency)."""
    d = dev.device()
    n = fleet.n
    out = UrgencyOut(keys=keys if keys is not None else new_keys(n, d))
    if need_time:
        out.need_time = torch.empty(n, dtype=torch.int64, device=d)
    if intermediates:
        out.total_wait = torch.empty(n, dtype=torch.int64, device=d)
        out.wr = torch.empty(n, dtype=torch.float64, device=d)
        out.bucket = torch.empty(n, dtype=torch.int32, device=d)
        out.est = torch.empty(n, dtype=torch.int64, device=d)
    if slot_waits:
        out.slot_wait = torch.full((fleet.t["slots"].shape[0],), -1, dtype=torch.int64, device=d)
    fs = fleet.c_struct()
    _lib.check(_lib.load().kr_urgency(
        ctypes.byref(fs), ctypes.byref(sched), out.keys.data_ptr(), _lib.ptr(out.need_time),
        _lib.ptr(out.total_wait), _lib.ptr(out.wr), _lib.ptr(out.bucket), _lib.ptr(out.est),
        _lib.ptr(out.slot_wait), _lib.ptr(key_stats), _lib.ptr(flags), dev.stream()),
        "kr_urgency")
    return out


class Workspace:
    """Caller-owned scratch for select / sort (kr_workspace_bytes)."""

    def __init__(self, n: int):
        self.n = n
        self.nbytes = int(_lib.load().kr_workspace_bytes(max(n, 1)))
        self.buf = torch.empty(self.nbytes, dtype=torch.uint8, device=dev.device())

    def ptr(self) -> int:
        return self.buf.data_ptr()


def sort_keys(keys: torch.Tensor, ws: Workspace, order: torch.Tensor | None = None,
              sorted_keys: torch.Tensor | None = None) -> tuple[torch.Tensor, torch.Tensor]:
    """Full ascending argsort of unique keys (kr_sort_keys)."""
    n = keys.shape[0]
    d = keys.device
    order = order if order is not None else torch.empty(n, dtype=torch.int32, device=d)
    sorted_keys = sorted_keys if sorted_keys is not None else new_keys(n, d)
    _lib.check(_lib.load().kr_sort_keys(keys.data_ptr(), n, order.data_ptr(),
                                        sorted_keys.data_ptr(), ws.ptr(), ws.nbytes,
                                        dev.stream()), "kr_sort_keys")
    return order, sorted_keys


def topk_select(keys: torch.Tensor, k: int, ws: Workspace,
                kth: torch.Tensor | None = None) -> torch.Tensor:
    """Device-side k-th smallest key (kr_topk_select); returns int64 [1, 2]."""
    kth = kth if kth is not None else new_keys(1, keys.device)
    _lib.check(_lib.load().kr_topk_select(keys.data_ptr(), keys.shape[0], k, kth.data_ptr(), None,
                                          ws.ptr(), ws.nbytes, dev.stream()), "kr_topk_select")
    return kth


def admit(keys: torch.Tensor, k: int, kth_ptr: int | None, fleet: DeviceFleet | None,
          sched: _lib.KrSched | None, ws: Workspace | None, *, admitted=None, refetch=None,
          edge_idx=None, edge_keys=None) -> None:
    """Admission pass (kr_admit): masks, skip counters, ordered S_e."""
    fs = fleet.c_struct() if fleet is not None else None
    _lib.check(_lib.load().kr_admit(
        keys.data_ptr(), keys.shape[0], k, kth_ptr,
        ctypes.byref(fs) if fs is not None else None,
        ctypes.byref(sched) if sched is not None else None,
        _lib.ptr(admitted), _lib.ptr(refetch), _lib.ptr(edge_idx), _lib.ptr(edge_keys),
        ws.ptr() if ws is not None else None, ws.nbytes if ws is not None else 0,
        dev.stream()), "kr_admit")


def new_key_stats(device=None) -> torch.Tensor:
    """Device buffer for the fused key statistics (4 x u64, see kr_key_stats_init)."""
    return torch.empty(4, dtype=torch.int64, device=device or dev.device())


def key_stats_init(stats: torch.Tensor) -> None:
    _lib.check(_lib.load().kr_key_stats_init(stats.data_ptr(), dev.stream()), "kr_key_stats_init")


def select_admit(keys: torch.Tensor, k: int, ws: Workspace, *, key_stats=None, fleet=None,
                 sched=None, admitted=None, refetch=None, edge_idx=None, edge_keys=None,
                 kth=None) -> None:
    """Fused select + admission + ordered S_e (kr_select_admit)."""
    fs = fleet.c_struct() if fleet is not None else None
    _lib.check(_lib.load().kr_select_admit(
        keys.data_ptr(), keys.shape[0], k, _lib.ptr(key_stats),
        ctypes.byref(fs) if fs is not None else None,
        ctypes.byref(sched) if sched is not None else None,
        _lib.ptr(admitted), _lib.ptr(refetch), _lib.ptr(edge_idx), _lib.ptr(edge_keys),
        _lib.ptr(kth), ws.ptr(), ws.nbytes, dev.stream()), "kr_select_admit")
