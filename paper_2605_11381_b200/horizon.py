"""Step 1a: execution-horizon policies over refinement-update magnitudes.

Drop-in for `roboserve.horizon` (reference horizon.py:1-151).  The policy
objects keep the reference's fields, defaults and validation; every decision
runs in the `kr_horizon_confidence` / `kr_horizon_static` / `kr_horizon_sweep`
CUDA kernels, in fp64 with the reference's numpy evaluation order, so results
are bit-exact.
`decide_horizon_batch` is the fleet-scale entry point over a device tensor
U[R, K, N] (fp32 or fp64 storage).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Iterable, Sequence

import numpy as np
import torch

from . import _lib
from . import device as dev

DEFAULT_THRESHOLD = 0.4
DEFAULT_MIN_HORIZON = 5

STATIC = "static"
CONFIDENCE_THRESHOLD = "confidence_threshold"


@dataclass(frozen=True, eq=False)
class UpdateMagnitudes:
    """K x N per-step, per-action update norms of one round (horizon.py:26-61)."""

    u: np.ndarray

    def __post_init__(self) -> None:
        arr = np.asarray(self.u, dtype=np.float64)
        if arr.ndim != 2:
            raise ValueError(f"update magnitudes must be 2-D (K x N), got shape {arr.shape}")
        k, n = arr.shape
        if k < 2:
            raise ValueError(f"need at least 2 refinement steps, got {k}")
        if n < 1:
            raise ValueError("chunk size must be >= 1")
        if not np.isfinite(arr).all():
            raise ValueError("update magnitudes must be finite")
        if (arr < 0).any():
            raise ValueError("update magnitudes must be >= 0")
        frozen = arr.copy()
        frozen.setflags(write=False)
        object.__setattr__(self, "u", frozen)

    @property
    def steps(self) -> int:
        return self.u.shape[0]

    @property
    def chunk_size(self) -> int:
        return self.u.shape[1]


@dataclass(frozen=True)
class HorizonPolicyConfig:
    """Static horizon or confidence threshold with a floor (horizon.py:64-105)."""

    kind: str
    static_h: int = 0
    threshold: float = DEFAULT_THRESHOLD
    min_horizon: int = DEFAULT_MIN_HORIZON

    def __post_init__(self) -> None:
        if self.kind not in (STATIC, CONFIDENCE_THRESHOLD):
            raise ValueError(f"unknown horizon policy kind {self.kind!r}")
        if self.kind == STATIC and self.static_h < 1:
            raise ValueError(f"static horizon must be >= 1, got {self.static_h}")
        if self.kind == CONFIDENCE_THRESHOLD:
            if self.threshold < 0:
                raise ValueError(f"threshold must be >= 0, got {self.threshold}")
            if self.min_horizon < 1:
                raise ValueError(f"min_horizon must be >= 1, got {self.min_horizon}")

    @classmethod
    def static(cls, horizon: int) -> "HorizonPolicyConfig":
        return cls(kind=STATIC, static_h=horizon)

    @classmethod
    def confidence(cls, threshold: float = DEFAULT_THRESHOLD,
                   min_horizon: int = DEFAULT_MIN_HORIZON) -> "HorizonPolicyConfig":
        return cls(kind=CONFIDENCE_THRESHOLD, threshold=threshold, min_horizon=min_horizon)

    @property
    def floor(self) -> int:
        return self.static_h if self.kind == STATIC else self.min_horizon


def decide_horizon_batch(cfg: HorizonPolicyConfig, U: torch.Tensor,
                         out: torch.Tensor | None = None, validate: bool = True,
                         max_sms: int = 0) -> torch.Tensor:
    """H[r] = decide_horizon(cfg, U[r]) for a device tensor U[R, K, N].

    fp32 storage is upcast exactly; all arithmetic is fp64.  With
    `validate`, non-finite or negative magnitudes raise the reference's
    ValueError (one device->host read of the flag word); without it the call
    is fully asynchronous on the current stream.
    """
    if U.dim() != 3:
        raise ValueError(f"update magnitudes must be R x K x N, got shape {tuple(U.shape)}")
    if U.dtype not in (torch.float32, torch.float64):
        raise ValueError(f"U must be float32 or float64, got {U.dtype}")
    R, K, N = U.shape
    if K < 2:
        raise ValueError(f"need at least 2 refinement steps, got {K}")
    if N < 1:
        raise ValueError("chunk size must be >= 1")
    dev.device()
    if not U.is_cuda:
        U = U.to(dev.device())
    U = U.contiguous()
    if out is None:
        out = torch.empty(R, dtype=torch.int32, device=U.device)
    lib = _lib.load()
    if cfg.kind == STATIC:
        _lib.check(lib.kr_horizon_static(R, N, cfg.static_h, out.data_ptr(), dev.stream()),
                   "kr_horizon_static")
        return out
    fl = dev.flags() if validate else None
    dtype = _lib.KR_F64 if U.dtype == torch.float64 else _lib.KR_F32
    _lib.check(lib.kr_horizon_confidence(U.data_ptr(), dtype, R, K, N, 1.0 + cfg.threshold,
                                         cfg.min_horizon, out.data_ptr(), _lib.ptr(fl), max_sms,
                                         dev.stream()), "kr_horizon_confidence")
    if validate:
        f = dev.read_flags(fl)
        if f & _lib.FLAG_NONFINITE:
            raise ValueError("update magnitudes must be finite")
        if f & _lib.FLAG_NEGATIVE:
            raise ValueError("update magnitudes must be >= 0")
    return out


def decide_horizon(cfg: HorizonPolicyConfig, magnitudes: UpdateMagnitudes) -> int:
    """One round's execution horizon (horizon.py:108-132), on the device."""
    u = magnitudes.u
    K, N = u.shape
    a = dev.arena(8 * u.size + 64)
    a.host[64:64 + 8 * u.size].view(np.float64)[:] = u.reshape(-1)
    H = a.host[:4].view(np.int32)
    st = dev.raw_stream()
    lib = _lib.load()
    if cfg.kind == STATIC:
        _lib.check(lib.kr_horizon_static(1, N, cfg.static_h, a.dbase, st),
                   "kr_horizon_static")
    else:
        # the magnitudes (validated by UpdateMagnitudes) staged into device
        # scratch: the streaming kernel's TMA reads HBM; the horizon comes
        # back through the mapped arena -- one copy, one launch, one sync
        dU = a.device_scratch(8 * u.size)
        _lib.check(lib.kr_memcpy_async(dU, a.dbase + 64, 8 * u.size, st),
                   "kr_memcpy_async")
        _lib.check(lib.kr_horizon_confidence(dU, _lib.KR_F64, 1, K, N, 1.0 + cfg.threshold,
                                             cfg.min_horizon, a.dbase, None, 0, st),
                   "kr_horizon_confidence")
    dev.sync(st)
    return int(H[0])


SWEEP_MAX_CONFIGS = 64  # per kernel launch (kr_horizon_sweep); more are split


def _addr(arr) -> int:
    return ctypes.addressof(arr)


def sweep_horizon_sums(cfgs: Sequence[HorizonPolicyConfig], U: torch.Tensor,
                       H: torch.Tensor | None = None, validate: bool = True) -> torch.Tensor:
    """Device sums[c] = sum_r decide_horizon(cfgs[c], U[r]) (int64 [C]) in one
    pass over U[R, K, N] per 64 configurations (kr_horizon_sweep).  With `H`
    (int32 [C, R]) every decision is written too.  Asynchronous unless
    `validate` (one flag-word read)."""
    if not cfgs:
        raise ValueError("no policy configurations given")
    if U.dim() != 3:
        raise ValueError(f"update magnitudes must be R x K x N, got shape {tuple(U.shape)}")
    if U.dtype not in (torch.float32, torch.float64):
        raise ValueError(f"U must be float32 or float64, got {U.dtype}")
    R, K, N = U.shape
    if K < 2:
        raise ValueError(f"need at least 2 refinement steps, got {K}")
    if N < 1:
        raise ValueError("chunk size must be >= 1")
    dev.device()
    if not U.is_cuda:
        U = U.to(dev.device())
    U = U.contiguous()
    C = len(cfgs)
    if H is not None and (tuple(H.shape) != (C, R) or H.dtype != torch.int32 or not H.is_cuda):
        raise ValueError(f"H must be a CUDA int32 tensor of shape {(C, R)}")
    sums = torch.zeros(C, dtype=torch.int64, device=U.device)
    lib = _lib.load()
    fl = dev.flags() if validate else None
    dtype = _lib.KR_F64 if U.dtype == torch.float64 else _lib.KR_F32
    for c0 in range(0, C, SWEEP_MAX_CONFIGS):
        part = cfgs[c0:c0 + SWEEP_MAX_CONFIGS]
        n = len(part)
        # a NaN / +inf threshold never trips (f > NaN and f > inf are false), so
        # the reference decides N for every round: a static cell of N
        never = [c.kind != STATIC and not np.isfinite(1.0 + c.threshold) for c in part]
        kind = (ctypes.c_int32 * n)(*[0 if c.kind == STATIC or nv else 1
                                      for c, nv in zip(part, never)])
        opt = (ctypes.c_double * n)(*[1.0 if nv else 1.0 + c.threshold
                                      for c, nv in zip(part, never)])
        prm = (ctypes.c_int32 * n)(*[N if nv else (c.static_h if c.kind == STATIC else c.min_horizon)
                                     for c, nv in zip(part, never)])
        _lib.check(lib.kr_horizon_sweep(U.data_ptr(), dtype, R, K, N, n, _addr(kind), _addr(opt), _addr(prm),
                                        sums[c0:].data_ptr(),
                                        None if H is None else H[c0].data_ptr(),
                                        _lib.ptr(fl), dev.stream()), "kr_horizon_sweep")
    if validate:
        f = dev.read_flags(fl)
        if f & _lib.FLAG_NONFINITE:
            raise ValueError("update magnitudes must be finite")
        if f & _lib.FLAG_NEGATIVE:
            raise ValueError("update magnitudes must be >= 0")
    return sums


def sweep_thresholds(cfgs: Sequence[HorizonPolicyConfig],
                     magnitude_sequence: Iterable[UpdateMagnitudes]) -> list[float]:
    """Mean decided horizon of each config over the rounds (horizon.py:135-151).

    Rounds of equal shape are stacked into one device tensor and every config
    is decided in a single pass over it (kr_horizon_sweep); the mean is the
    reference's int sum / len(seq)."""
    seq = list(magnitude_sequence)
    if not cfgs:
        raise ValueError("no policy configurations given")
    if not seq:
        raise ValueError("no update-magnitude rounds given")
    groups: dict[tuple, list[np.ndarray]] = {}
    for m in seq:
        groups.setdefault(m.u.shape, []).append(m.u)
    totals = [0] * len(cfgs)
    for g in groups.values():
        sums = sweep_horizon_sums(list(cfgs), dev.tensor(np.stack(g), torch.float64),
                                  validate=False).cpu().tolist()
        totals = [a + b for a, b in zip(totals, sums)]
    return [t / len(seq) for t in totals]
