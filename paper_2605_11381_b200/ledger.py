"""Device-resident incremental task ledger for the simulator's planning loop.

SURVEY.md §8(f) row 2: `sim._on_plan` (reference sim.py:285-311) calls
`plan()` on every planning event with the full `states` mapping, and the
reference re-derives every pending task's wait ledger from its whole history
(`ledger_from_history`, waiting.py:69-93) each time.  Here the history lives on
the GPU across planning rounds:

* `DeviceLedger` holds per-task `t_start`, round counts, the append-only
  history slots [task][cap][4] (gen_start, gen_end, exec_start, exec_end) and a
  running wait total with a cursor; TaskState mutations (core.py:200-229) are
  buffered on the host and applied in one `kr_ledger_apply` launch per planning
  round (one thread per touched task, events in call order).  A round's wait
  is final the moment it is first computable and the computable rounds form a
  prefix, so the total advances instead of being recomputed.
* `LedgerStates` is the task-state mapping the simulator keeps
  (`self.states`, sim.py:226-227): inserting a TaskState registers the task and
  hooks its mutators, so every `begin_generation` / `finish_generation` /
  `record_execution` the simulator makes (sim.py:363, 376, 429) is mirrored to
  the device.  `scheduler.plan(pending, LedgerStates, ...)` then sends only the
  pending requests' scalars and runs `kr_urgency_ledger` (O(1) per request)
  followed by the usual sort / admission / cloud placement kernels.

Decisions are bit-identical to the reference `plan()` (tests replay the
reference simulator's recorded planning loop, tests/golden/sim_replay.json).
"""

from __future__ import annotations

import ctypes
from typing import Mapping, Sequence

import numpy as np
import torch

from . import _lib
from . import device as dev
from . import fleet as fl

EV_NEW, EV_BEGIN_GEN, EV_FINISH_GEN, EV_EXEC = 0, 1, 2, 3
KrLedger, KrEvents, KrRequests = _lib.KrLedger, _lib.KrEvents, _lib.KrRequests


class _AdmitView:
    """The request fields admission / placement read (kr_fleet subset)."""

    def __init__(self, n: int, obs: torch.Tensor, skipped: torch.Tensor):
        self.n = n
        self.t = {"obs_captured_at": obs, "skipped": skipped}

    def c_struct(self) -> _lib.KrFleet:
        f = _lib.KrFleet()
        f.n = self.n
        f.obs_captured_at = self.t["obs_captured_at"].data_ptr()
        f.skipped = self.t["skipped"].data_ptr()
        return f


class DeviceLedger:
    """Per-task state and history resident on one GPU, updated incrementally."""

    def __init__(self, tasks: int = 1024, rounds: int = 8):
        self.d = dev.device()
        self.slot_of: dict[str, int] = {}
        self.n_tasks = 0                      # slots in use
        self._alloc(max(tasks, 1), max(rounds, 1))
        self._n_exec = np.zeros(self.cap_tasks, np.int64)   # host mirror for capacity checks
        self._n_gen = np.zeros(self.cap_tasks, np.int64)
        self._ev: list[tuple] = []            # (slot, kind, round, a, b)
        self.flags = dev.flags()

    # -- storage -----------------------------------------------------------
    def _alloc(self, tasks: int, rounds: int) -> None:
        d = self.d
        self.cap_tasks, self.cap = tasks, rounds
        self.t_start = torch.zeros(tasks, dtype=torch.int64, device=d)
        self.n_exec = torch.zeros(tasks, dtype=torch.int32, device=d)
        self.n_gen = torch.zeros(tasks, dtype=torch.int32, device=d)
        self.wait_next = torch.zeros(tasks, dtype=torch.int32, device=d)
        self.wait_total = torch.zeros(tasks, dtype=torch.int64, device=d)
        self.slots = torch.zeros((tasks, rounds, 4), dtype=torch.int64, device=d)

    def _grow(self, tasks: int, rounds: int) -> None:
        old = (self.t_start, self.n_exec, self.n_gen, self.wait_next, self.wait_total, self.slots)
        n, r = self.cap_tasks, self.cap
        self._alloc(tasks, rounds)
        for dst, src in zip((self.t_start, self.n_exec, self.n_gen, self.wait_next,
                             self.wait_total), old[:5]):
            dst[:n].copy_(src)
        self.slots[:n, :r].copy_(old[5])
        for name in ("_n_exec", "_n_gen"):
            a = getattr(self, name)
            b = np.zeros(tasks, np.int64)
            b[:a.size] = a
            setattr(self, name, b)

    def c_struct(self) -> KrLedger:
        return KrLedger(self.cap_tasks, self.cap, 0, self.t_start.data_ptr(),
                        self.n_exec.data_ptr(), self.n_gen.data_ptr(),
                        self.wait_next.data_ptr(), self.wait_total.data_ptr(),
                        self.slots.data_ptr())

    # -- TaskState mutations (core.py:169-229) -------------------------------
    def add_task(self, task_id: str, t_start: int) -> int:
        if task_id in self.slot_of:
            raise ValueError(f"task {task_id!r} already in the ledger")
        s = self.n_tasks
        if s >= self.cap_tasks:
            self._flush_then_grow(tasks=2 * self.cap_tasks)
        self.slot_of[task_id] = s
        self.n_tasks += 1
        self._ev.append((s, EV_NEW, 0, int(t_start), 0))
        return s

    def begin_generation(self, task_id: str, round_id: int, at: int) -> None:
        s = self.slot_of[task_id]
        self._need_rounds(round_id + 1)
        self._n_gen[s] = round_id + 1
        self._ev.append((s, EV_BEGIN_GEN, round_id, int(at), 0))

    def finish_generation(self, task_id: str, round_id: int, at: int) -> None:
        self._ev.append((self.slot_of[task_id], EV_FINISH_GEN, round_id, int(at), 0))

    def record_execution(self, task_id: str, round_id: int, start: int, end: int) -> None:
        s = self.slot_of[task_id]
        self._need_rounds(round_id + 1)
        self._n_exec[s] = round_id + 1
        self._ev.append((s, EV_EXEC, round_id, int(start), int(end)))

    def _need_rounds(self, r: int) -> None:
        if r > self.cap:
            cap = self.cap
            while cap < r:
                cap *= 2
            self._flush_then_grow(rounds=cap)

    def _flush_then_grow(self, tasks: int | None = None, rounds: int | None = None) -> None:
        self.flush()
        self._grow(tasks or self.cap_tasks, rounds or self.cap)

    def flush(self) -> None:
        """Apply the buffered mutations (one kr_ledger_apply launch)."""
        if not self._ev:
            return
        ev = np.array(self._ev, dtype=np.int64)
        self._ev.clear()
        order = np.argsort(ev[:, 0], kind="stable")
        ev = ev[order]
        tasks, start = np.unique(ev[:, 0], return_index=True)
        off = np.append(start, len(ev)).astype(np.int32)
        i32 = lambda a: dev.tensor(np.ascontiguousarray(a, np.int32), torch.int32)
        i64 = lambda a: dev.tensor(np.ascontiguousarray(a, np.int64), torch.int64)
        t_task, t_off, t_kind, t_round = i32(tasks), i32(off), i32(ev[:, 1]), i32(ev[:, 2])
        t_a, t_b = i64(ev[:, 3]), i64(ev[:, 4])
        e = KrEvents(len(tasks), t_task.data_ptr(), t_off.data_ptr(), t_kind.data_ptr(),
                     t_round.data_ptr(), t_a.data_ptr(), t_b.data_ptr())
        L = self.c_struct()
        _lib.check(_lib.load().kr_ledger_apply(ctypes.byref(L), ctypes.byref(e),
                                               self.flags.data_ptr(), dev.stream()),
                   "kr_ledger_apply")
        if dev.read_flags(self.flags) & _lib.FLAG_LEDGER:
            raise ValueError("ledger event out of order or beyond the history capacity")

    # -- one planning round ---------------------------------------------------
    def urgency(self, reqs: Sequence, states: Mapping, rank: Mapping[str, int],
                sched: _lib.KrSched, flags: torch.Tensor):
        """Packed keys of the pending requests from the device ledger."""
        self.flush()
        n = len(reqs)
        i64 = np.empty((4, n), np.int64)
        i32 = np.empty((4, n), np.int32)
        for i, r in enumerate(reqs):
            i64[0, i] = r.issued_at
            i64[1, i] = r.obs_captured_at
            i64[2, i] = states[r.task_id].accumulated_generation
            i32[0, i] = self.slot_of[r.task_id]
            i32[1, i] = r.last_exec_info.remaining_actions
            i32[2, i] = rank[r.task_id]
            i32[3, i] = r.skipped
        t64 = dev.tensor(i64[:3], torch.int64)
        t32 = dev.tensor(i32, torch.int32)
        q = KrRequests(n, t32[0].data_ptr(), t64[0].data_ptr(), t64[1].data_ptr(),
                       t64[2].data_ptr(), t32[1].data_ptr(), t32[2].data_ptr(),
                       t32[3].data_ptr())
        keys = fl.new_keys(n)
        L = self.c_struct()
        _lib.check(_lib.load().kr_urgency_ledger(
            ctypes.byref(L), ctypes.byref(q), ctypes.byref(sched), keys.data_ptr(), None, None,
            None, None, None, None, flags.data_ptr(), dev.stream()), "kr_urgency_ledger")
        self._keep = (t64, t32)  # alive until the round's kernels have consumed them
        return keys, _AdmitView(n, t64[1], t32[3])

    def total_wait(self, task_id: str) -> int:
        """ledger_from_history(state).total_wait of one task (waiting.py:69-93)."""
        self.flush()
        return int(self.wait_total[self.slot_of[task_id]].item())


class LedgerStates(dict):
    """task_id -> TaskState mapping whose tasks are mirrored in a DeviceLedger.

    Drop-in for the simulator's `self.states` dict: inserting a state
    registers it (with any history it already has) and wraps its mutators so
    the device ledger sees every change; `scheduler.plan` recognises the
    mapping and plans from the device-resident history."""

    def __init__(self, ledger: DeviceLedger | None = None, tasks: int = 1024, rounds: int = 8):
        super().__init__()
        self.ledger = ledger if ledger is not None else DeviceLedger(tasks, rounds)

    def __setitem__(self, task_id, state) -> None:
        if task_id in self:
            raise ValueError(f"task {task_id!r} already tracked")
        L = self.ledger
        L.add_task(task_id, state.t_start)
        for j, gs in enumerate(state.gen_starts):
            L.begin_generation(task_id, j, gs)
            if state.gen_ends[j] is not None:
                L.finish_generation(task_id, j, state.gen_ends[j])
        for j, iv in enumerate(state.exec_intervals):
            L.record_execution(task_id, j, iv.start, iv.end)
        self._hook(task_id, state)
        super().__setitem__(task_id, state)

    def _hook(self, task_id, state) -> None:
        L = self.ledger
        bg, fg, rx = state.begin_generation, state.finish_generation, state.record_execution

        def begin_generation(round_id, at):
            bg(round_id, at)  # the reference's own validation first
            L.begin_generation(task_id, round_id, at)

        def finish_generation(round_id, at):
            fg(round_id, at)
            L.finish_generation(task_id, round_id, at)

        def record_execution(round_id, start, end, horizon):
            rx(round_id, start, end, horizon)
            L.record_execution(task_id, round_id, start, end)

        state.begin_generation = begin_generation
        state.finish_generation = finish_generation
        state.record_execution = record_execution

    def __delitem__(self, task_id) -> None:
        raise TypeError("tasks are never removed from a LedgerStates mapping")
