"""Step 2 (part): dominant-phase wait accounting and the wait-ratio signal.

Drop-in for `roboserve.waiting` (reference waiting.py:1-100).  Interval
validation stays on the host with the reference's messages; the ledger, the
ratio and the per-round waits are computed by the `kr_urgency` /
`kr_wait_ratio` CUDA kernels over the CSR history layout of fleet.py.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from types import SimpleNamespace
from typing import Sequence

import numpy as np
import torch

from . import _lib
from . import device as dev
from . import fleet as fl
from .core import Duration, Interval, TaskState, TimePoint


@dataclass(frozen=True)
class WaitLedger:
    """Per-round waits of one task and their exact sum (waiting.py:23-35)."""

    waits: tuple
    total_wait: Duration

    @classmethod
    def from_waits(cls, waits: Sequence[Duration]) -> "WaitLedger":
        ws = tuple(int(w) for w in waits)
        if any(w < 0 for w in ws):
            raise ValueError("per-round waits must be >= 0")
        return cls(waits=ws, total_wait=sum(ws))


def _check_round_pair(gen: Interval, exc: Interval, label: str) -> None:
    if exc.start < gen.end:
        raise ValueError(f"{label}: execution [{exc.start}, {exc.end}) begins before "
                         f"generation [{gen.start}, {gen.end}) ends")


def _state_fleet(state: TaskState, now_rank_task: str | None = None) -> fl.DeviceFleet:
    """A one-request fleet view of a TaskState (only its history matters)."""
    req = SimpleNamespace(task_id=state.task_id, issued_at=0, obs_captured_at=0, skipped=0,
                          last_exec_info=SimpleNamespace(remaining_actions=0))
    return fl.DeviceFleet.from_host(fl.host_soa([req], {state.task_id: state}, {state.task_id: 0}))


def _sched(now: int) -> _lib.KrSched:
    return fl.sched_struct("fifo", 1, 1, 0, 0, now, 1, 0)


_NO_REQ = SimpleNamespace(task_id=None, issued_at=0, obs_captured_at=0, skipped=0,
                          last_exec_info=SimpleNamespace(remaining_actions=0))


def _state_urgency(state: TaskState, now: int, slot_waits: bool):
    """kr_urgency over a one-request view of `state`, columns and results in the
    mapped arena (one launch + one synchronisation).  Returns (wr, slot waits
    or None, flags)."""
    req = SimpleNamespace(**{**vars(_NO_REQ), "task_id": state.task_id})
    nsl = max(len(state.gen_starts), len(state.exec_intervals), 1)
    out_bytes = 32 + (8 * nsl if slot_waits else 0)
    fs, out, d = fl.pack_mapped([req], {state.task_id: state}, {state.task_id: 0}, out_bytes)
    out[24:28].view(np.uint32)[0] = 0
    sched = _sched(now)
    st = dev.raw_stream()
    _lib.check(_lib.load().kr_urgency(
        ctypes.byref(fs), ctypes.byref(sched), d, None, None, d + 16, None, None,
        d + 32 if slot_waits else None, None, d + 24, st), "kr_urgency")
    dev.sync(st)
    sw = out[32:32 + 8 * nsl].view(np.int64).copy() if slot_waits else None
    return float(out[16:24].view(np.float64)[0]), sw, int(out[24:28].view(np.uint32)[0])


def round_wait(gen_j: Interval, exec_j: Interval, gen_next: Interval,
               exec_next: Interval) -> Duration:
    """Wait between round j and j+1 on round j's dominant side (waiting.py:46-59)."""
    _check_round_pair(gen_j, exec_j, "round j")
    _check_round_pair(gen_next, exec_next, "round j+1")
    if gen_next.start < gen_j.start or exec_next.start < exec_j.start:
        raise ValueError("round j+1 intervals precede round j: rounds out of order")
    soa = {k: np.zeros(1, np.int64) for k in fl.INT_FIELDS64}
    soa.update({k: np.zeros(1, np.int32) for k in fl.INT_FIELDS32})
    soa["n_exec"][0] = 2
    soa["n_gen"][0] = 2
    soa["slots"] = np.array([[gen_j.start, gen_j.end, exec_j.start, exec_j.end],
                             [gen_next.start, gen_next.end, exec_next.start, exec_next.end]],
                            np.int64)
    soa["n"] = 1
    out = fl.urgency(fl.DeviceFleet.from_host(soa), _sched(0), need_time=False,
                     intermediates=True)
    return int(out.total_wait.item())


def wait_ratio(ledger: WaitLedger, t_start: TimePoint, t_now: TimePoint) -> float:
    """Accumulated wait over lifetime, clamped to [0, 1] (waiting.py:62-66)."""
    if t_now <= t_start:
        raise ValueError(f"t_now {t_now} must be after t_start {t_start}")
    a = dev.arena(64)
    v = a.host[:24].view(np.int64)  # total, t_start, ratio (fp64 bits)
    f = a.host[24:28].view(np.uint32)
    v[0], v[1], f[0] = int(ledger.total_wait), int(t_start), 0
    st = dev.raw_stream()
    _lib.check(_lib.load().kr_wait_ratio(a.dbase, a.dbase + 8, 1, int(t_now), a.dbase + 16,
                                         a.dbase + 24, st), "kr_wait_ratio")
    dev.sync(st)
    if int(f[0]) & _lib.FLAG_RATIO:
        raise ValueError("wait-ratio operands beyond 2^53 are not exactly representable")
    return float(v[2:3].view(np.float64)[0])


def ledger_from_history(state: TaskState) -> WaitLedger:
    """Wait ledger from the task's recorded history (waiting.py:69-93)."""
    n_exec = len(state.exec_intervals)
    if n_exec == 0:
        return WaitLedger.from_waits([])
    _, sw, _ = _state_urgency(state, 0, True)
    return WaitLedger.from_waits([int(w) for w in sw[:n_exec] if w >= 0])


def current_wait_ratio(state: TaskState, now: TimePoint) -> float:
    """Wait ratio of a live task; 0.0 before it has any lifetime (waiting.py:96-100)."""
    return _state_urgency(state, int(now), False)[0]
