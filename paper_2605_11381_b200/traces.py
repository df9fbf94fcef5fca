"""Trace ingest: JSON Lines task traces -> columnar (device) tensors, and the
horizon-policy Pareto sweep over them.

Drop-in for the trace I/O of `roboserve.workload` (reference
workload.py:29-262: TraceFormatError, RoundRecord, TaskTrace, trace_to_dict,
trace_from_dict, store_traces, load_traces, load_trace_dir) and for
`cmd_pareto` (cli.py:109-140).  Parsing and validation run in the native
reader `kr_trace_parse` (csrc/kr_ingest.cpp, in libkairos_b200.so), which
keeps the reference's validation order and TraceFormatError fields; the
result is a `TraceColumns` table whose update magnitudes go to the GPU as one
[R, K, N] tensor per shape, where `kr_horizon_sweep` decides every policy
cell of a sweep in one pass.

Documented deltas: JSON syntax errors carry the same line number and a
close-but-not-identical message ("invalid JSON: Expecting ',' delimiter");
non-integer round fields / payloads, ragged magnitude arrays and integers
beyond int64 are rejected with a TraceFormatError instead of surfacing a later
TypeError / numpy error.
"""

from __future__ import annotations

import ctypes
import json
from dataclasses import dataclass
from pathlib import Path
from typing import Iterable, Optional, Sequence

import numpy as np
import torch

from . import _lib
from . import device as dev
from .horizon import HorizonPolicyConfig, UpdateMagnitudes, sweep_horizon_sums


class TraceFormatError(ValueError):
    """Malformed or invariant-violating trace data (workload.py:29-54)."""

    def __init__(self, message: str, *, line: Optional[int] = None,
                 task_id: Optional[str] = None, round_id: Optional[int] = None) -> None:
        prefix = []
        if line is not None:
            prefix.append(f"line {line}")
        if task_id is not None:
            prefix.append(f"task {task_id!r}")
        if round_id is not None:
            prefix.append(f"round {round_id}")
        full = (": ".join([", ".join(prefix), message]) if prefix else message)
        super().__init__(full)
        self.raw_message = message
        self.line = line
        self.task_id = task_id
        self.round_id = round_id


@dataclass(frozen=True)
class RoundRecord:
    """One recorded generate-execute round (workload.py:57-86)."""

    round_id: int
    trigger_action_index: int
    horizon: int
    chunk_size: int
    update_magnitudes: Optional[UpdateMagnitudes] = None
    action_trajectory: Optional[tuple] = None

    def __post_init__(self) -> None:
        if self.round_id < 0:
            raise TraceFormatError("round_id must be >= 0", round_id=self.round_id)
        if self.trigger_action_index < 0:
            raise TraceFormatError("trigger_action_index must be >= 0", round_id=self.round_id)
        if not 1 <= self.horizon <= self.chunk_size:
            raise TraceFormatError(
                f"horizon {self.horizon} outside [1, chunk_size={self.chunk_size}]",
                round_id=self.round_id)


@dataclass(frozen=True)
class TaskTrace:
    """A task's full observation-inference-execution history (workload.py:89-131)."""

    task_id: str
    control_hz: float
    obs_payload_bytes: int
    action_payload_bytes: int
    success: bool
    rounds: tuple

    def __post_init__(self) -> None:
        if not self.task_id:
            raise TraceFormatError("task_id must be non-empty")
        if self.control_hz <= 0:
            raise TraceFormatError("control_hz must be > 0", task_id=self.task_id)
        if self.obs_payload_bytes < 0 or self.action_payload_bytes < 0:
            raise TraceFormatError("payload sizes must be >= 0", task_id=self.task_id)
        if not self.rounds:
            raise TraceFormatError("trace has no rounds", task_id=self.task_id)
        for idx, rnd in enumerate(self.rounds):
            if rnd.round_id != idx:
                raise TraceFormatError(
                    f"round ids must be contiguous from 0, found {rnd.round_id} at position {idx}",
                    task_id=self.task_id, round_id=rnd.round_id)
            if idx >= 1:
                prev_h = self.rounds[idx - 1].horizon
                if rnd.trigger_action_index >= prev_h:
                    raise TraceFormatError(
                        f"trigger_action_index {rnd.trigger_action_index} must be "
                        f"< previous horizon {prev_h}",
                        task_id=self.task_id, round_id=rnd.round_id)

    @property
    def total_actions(self) -> int:
        return sum(r.horizon for r in self.rounds)


# --- JSONL serialization (workload.py:136-262) ---------------------------------

def _round_to_dict(rnd: RoundRecord) -> dict:
    out = {"round_id": rnd.round_id, "trigger_action_index": rnd.trigger_action_index,
           "horizon": rnd.horizon, "chunk_size": rnd.chunk_size, "update_magnitudes": None,
           "action_trajectory": None}
    if rnd.update_magnitudes is not None:
        out["update_magnitudes"] = rnd.update_magnitudes.u.tolist()
    if rnd.action_trajectory is not None:
        out["action_trajectory"] = [list(row) for row in rnd.action_trajectory]
    return out


def trace_to_dict(trace: TaskTrace) -> dict:
    return {"task_id": trace.task_id, "control_hz": trace.control_hz,
            "obs_payload_bytes": trace.obs_payload_bytes,
            "action_payload_bytes": trace.action_payload_bytes, "success": trace.success,
            "rounds": [_round_to_dict(r) for r in trace.rounds]}


def _jsonable(x):
    if isinstance(x, np.ndarray):
        return x.tolist()
    if isinstance(x, np.generic):
        return x.item()
    if isinstance(x, UpdateMagnitudes):
        return x.u.tolist()
    if isinstance(x, tuple):
        return list(x)
    raise TypeError(f"cannot serialise {type(x).__name__} in a trace")


def trace_from_dict(data: dict, line: int = 0) -> TaskTrace:
    """One decoded trace object -> TaskTrace, through the native validator
    (numpy arrays are accepted where the reference's np.asarray would be)."""
    return _objects(parse_jsonl(json.dumps(data, allow_nan=True, default=_jsonable),
                                first_line=line, line_override=line))[0]


def store_traces(traces: Iterable[TaskTrace], path: str | Path) -> None:
    with Path(path).open("w", encoding="utf-8") as fh:
        for trace in traces:
            fh.write(json.dumps(trace_to_dict(trace), separators=(",", ":")))
            fh.write("\n")


# --- native columnar reader ------------------------------------------------------

_Cols = _lib.KrTraceColumns


def _arr(ptr, n, dtype) -> np.ndarray:
    if n == 0 or not ptr:
        return np.zeros(0, dtype)
    ct = np.ctypeslib.as_ctypes_type(np.dtype(dtype))
    return np.ctypeslib.as_array(ctypes.cast(ptr, ctypes.POINTER(ct)), shape=(n,)).copy()


@dataclass
class TraceColumns:
    """Columnar trace table (host numpy arrays, owned)."""

    task_ids: list
    round_off: np.ndarray          # [T+1]
    control_hz: np.ndarray         # [T] float64
    control_hz_is_int: np.ndarray  # [T] bool
    obs_payload_bytes: np.ndarray  # [T] int64
    action_payload_bytes: np.ndarray
    success: np.ndarray            # [T] bool
    round_id: np.ndarray           # [R] int32
    trigger_action_index: np.ndarray
    horizon: np.ndarray
    chunk_size: np.ndarray
    mag_k: np.ndarray              # [R] int32 (0: no magnitudes)
    mag_n: np.ndarray
    mag_off: np.ndarray            # [R+1] int64
    mags: np.ndarray               # float64, K x N per round concatenated
    traj_rows: np.ndarray          # [R] int32 (-1: none)
    traj_row0: np.ndarray          # [R+1]
    traj_off: np.ndarray           # [rows+1]
    traj: np.ndarray

    @property
    def n_traces(self) -> int:
        return len(self.task_ids)

    @property
    def n_rounds(self) -> int:
        return int(self.round_id.size)

    def magnitude_groups(self) -> dict:
        """{(K, N): (round indices, U[R_g, K, N] float64)} over rounds with magnitudes."""
        out = {}
        has = self.mag_k > 0
        shapes = np.stack([self.mag_k, self.mag_n], axis=1)
        for K, N in sorted(set(map(tuple, shapes[has].tolist()))):
            idx = np.nonzero(has & (self.mag_k == K) & (self.mag_n == N))[0]
            gather = self.mag_off[idx][:, None] + np.arange(K * N)[None, :]
            out[(K, N)] = (idx, self.mags[gather].reshape(len(idx), K, N))
        return out

    def to_device(self, dtype: torch.dtype = torch.float64) -> dict:
        """{(K, N): (round indices, CUDA tensor U[R_g, K, N])}."""
        return {s: (idx, dev.tensor(U, dtype)) for s, (idx, U) in self.magnitude_groups().items()}


def _columns(c: _Cols) -> TraceColumns:
    T, R = c.n_traces, c.n_rounds
    id_off = _arr(c.id_off, T + 1, np.int64)
    raw = ctypes.string_at(c.ids, int(id_off[-1])) if T else b""
    ids = [raw[id_off[i]:id_off[i + 1]].decode("utf-8", "surrogatepass") for i in range(T)]
    return TraceColumns(
        task_ids=ids, round_off=_arr(c.round_off, T + 1, np.int64),
        control_hz=_arr(c.control_hz, T, np.float64),
        control_hz_is_int=_arr(c.control_hz_is_int, T, np.uint8).astype(bool),
        obs_payload_bytes=_arr(c.obs_payload_bytes, T, np.int64),
        action_payload_bytes=_arr(c.action_payload_bytes, T, np.int64),
        success=_arr(c.success, T, np.uint8).astype(bool),
        round_id=_arr(c.round_id, R, np.int32),
        trigger_action_index=_arr(c.trigger_action_index, R, np.int32),
        horizon=_arr(c.horizon, R, np.int32), chunk_size=_arr(c.chunk_size, R, np.int32),
        mag_k=_arr(c.mag_k, R, np.int32), mag_n=_arr(c.mag_n, R, np.int32),
        mag_off=_arr(c.mag_off, R + 1, np.int64), mags=_arr(c.mags, c.n_mag_values, np.float64),
        traj_rows=_arr(c.traj_rows, R, np.int32), traj_row0=_arr(c.traj_row0, R + 1, np.int64),
        traj_off=_arr(c.traj_off, c.n_traj_rows + 1, np.int64),
        traj=_arr(c.traj, c.n_traj_values, np.float64))


def _finish(status: int, handle: ctypes.c_void_p, line_override=None) -> TraceColumns:
    lib = _lib.load()
    try:
        c = lib.kr_trace_columns_of(handle).contents
        if status == _lib.KR_EFORMAT:
            line = line_override if line_override is not None else int(c.err_line)
            raise TraceFormatError(
                c.err_message.decode("utf-8", "replace"), line=line,
                task_id=c.err_task.decode("utf-8", "surrogatepass") if c.err_has_task else None,
                round_id=int(c.err_round) if c.err_has_round else None)
        _lib.check(status, "kr_trace_parse")
        return _columns(c)
    finally:
        lib.kr_trace_free(handle)


def parse_jsonl(text: str | bytes, first_line: int = 1, line_override=None) -> TraceColumns:
    """JSON Lines text -> TraceColumns (load_traces semantics)."""
    data = text.encode("utf-8", "surrogatepass") if isinstance(text, str) else bytes(text)
    h = ctypes.c_void_p()
    st = _lib.load().kr_trace_parse(data, len(data), first_line, ctypes.byref(h))
    return _finish(st, h, line_override)


def load_trace_columns(path: str | Path) -> TraceColumns:
    """One .jsonl file, or every *.jsonl under a directory in sorted order."""
    p = Path(path)
    files = sorted(p.glob("*.jsonl")) if p.is_dir() else [p]
    parts = []
    for f in files:
        h = ctypes.c_void_p()
        st = _lib.load().kr_trace_load(str(f).encode(), ctypes.byref(h))
        if st == _lib.KR_EINVAL and not h.value:
            raise FileNotFoundError(str(f))
        parts.append(_finish(st, h))
    return _concat(parts)


def _concat(parts: Sequence[TraceColumns]) -> TraceColumns:
    if len(parts) == 1:
        return parts[0]
    if not parts:
        return parse_jsonl("")
    kw = {"task_ids": [t for p in parts for t in p.task_ids]}
    for name in ("control_hz", "control_hz_is_int", "obs_payload_bytes", "action_payload_bytes",
                 "success", "round_id", "trigger_action_index", "horizon", "chunk_size", "mag_k",
                 "mag_n", "traj_rows", "mags", "traj"):
        kw[name] = np.concatenate([getattr(p, name) for p in parts])
    # offset arrays and the size of what they index
    for name, size in (("round_off", lambda p: p.n_rounds), ("mag_off", lambda p: p.mags.size),
                       ("traj_row0", lambda p: p.traj_off.size - 1),
                       ("traj_off", lambda p: p.traj.size)):
        out, shift = [np.zeros(1, np.int64)], 0
        for p in parts:
            out.append(getattr(p, name)[1:] + shift)
            shift += int(size(p))
        kw[name] = np.concatenate(out)
    return TraceColumns(**kw)


def _objects(cols: TraceColumns) -> list[TaskTrace]:
    traces = []
    for t in range(cols.n_traces):
        rounds = []
        for r in range(int(cols.round_off[t]), int(cols.round_off[t + 1])):
            mags = None
            if cols.mag_k[r] > 0:
                K, N = int(cols.mag_k[r]), int(cols.mag_n[r])
                mags = UpdateMagnitudes(cols.mags[cols.mag_off[r]:cols.mag_off[r + 1]].reshape(K, N))
            traj = None
            if cols.traj_rows[r] >= 0:
                rows = range(int(cols.traj_row0[r]), int(cols.traj_row0[r]) + int(cols.traj_rows[r]))
                traj = tuple(tuple(float(v) for v in cols.traj[cols.traj_off[i]:cols.traj_off[i + 1]])
                             for i in rows)
            rounds.append(RoundRecord(int(cols.round_id[r]), int(cols.trigger_action_index[r]),
                                      int(cols.horizon[r]), int(cols.chunk_size[r]), mags, traj))
        hz = cols.control_hz[t]
        traces.append(TaskTrace(task_id=cols.task_ids[t],
                                control_hz=int(hz) if cols.control_hz_is_int[t] else float(hz),
                                obs_payload_bytes=int(cols.obs_payload_bytes[t]),
                                action_payload_bytes=int(cols.action_payload_bytes[t]),
                                success=bool(cols.success[t]), rounds=tuple(rounds)))
    return traces


def load_traces(path: str | Path) -> list[TaskTrace]:
    """workload.py:229-250, parsed natively."""
    return _objects(load_trace_columns(Path(path)))


def load_trace_dir(path: str | Path) -> list[TaskTrace]:
    """All traces under a directory, files in sorted order (workload.py:253-262)."""
    return _objects(load_trace_columns(Path(path)))


# --- horizon-policy Pareto sweep (cli.py:104-140) -----------------------------------

def _parse_grid(text: str, cast):
    return [cast(tok) for tok in text.split(",") if tok.strip()]


def pareto_rows(traces: str | Path | TraceColumns, static_grid: str = "10,20,30,40,50",
                threshold_grid: str = "0.1,0.2,0.4,0.6,0.8", h_min: int = 5) -> list[str]:
    """The CSV lines `roboserve pareto` writes: mean decided horizon of every
    static / confidence cell over every recorded round, all cells of a shape
    decided in one pass over the device-resident magnitudes."""
    cols = traces if isinstance(traces, TraceColumns) else load_trace_columns(traces)
    if cols.n_traces == 0:
        raise ValueError(f"no traces found under {traces}")
    missing = np.nonzero(cols.mag_k == 0)[0]
    if missing.size:
        r = int(missing[0])
        t = int(np.searchsorted(cols.round_off, r, side="right") - 1)
        raise ValueError(f"trace {cols.task_ids[t]!r} round {int(cols.round_id[r])} has no "
                         "update magnitudes; pareto sweeps need them")
    success_fraction = sum(1 for s in cols.success if s) / cols.n_traces
    cells = []
    for h in _parse_grid(static_grid, int):
        cells.append(("static", float(h), HorizonPolicyConfig.static(h)))
    for t in _parse_grid(threshold_grid, float):
        cells.append(("confidence", t, HorizonPolicyConfig.confidence(t, min_horizon=h_min)))
    totals = [0] * len(cells)
    if cells:
        for _, (_, U) in cols.to_device().items():
            sums = sweep_horizon_sums([c for _, _, c in cells], U, validate=False).cpu().tolist()
            totals = [a + b for a, b in zip(totals, sums)]
    lines = ["policy,parameter,mean_horizon,success_fraction"]
    for (name, param, _), tot in zip(cells, totals):
        lines.append(f"{name},{param},{tot / cols.n_rounds},{success_fraction}")
    return lines


def cmd_pareto(traces: str | Path, out: str | Path, static_grid: str = "10,20,30,40,50",
               threshold_grid: str = "0.1,0.2,0.4,0.6,0.8", h_min: int = 5) -> int:
    lines = pareto_rows(traces, static_grid, threshold_grid, h_min)
    Path(out).write_text("\n".join(lines) + "\n", encoding="utf-8")
    print(f"wrote {len(lines) - 1} sweep rows to {out}")
    return 0
