"""Device plumbing shared by the drop-in modules: host->device staging of small
inputs, the validation-flag word, and raising the reference's ValueErrors
from flags the kernels set."""

from __future__ import annotations

import ctypes
import functools
import threading
from fractions import Fraction

import numpy as np
import torch

from . import _lib

INT64_MAX = (1 << 63) - 1


def device() -> torch.device:
    _lib.load()
    return _lib.require_cuda()


def tensor(data, dtype: torch.dtype) -> torch.Tensor:
    """Host data -> contiguous CUDA tensor (pinned staging for arrays)."""
    dev = device()
    if isinstance(data, torch.Tensor):
        return data.to(device=dev, dtype=dtype).contiguous()
    arr = np.ascontiguousarray(data)
    if not arr.flags.writeable:
        arr = arr.copy()
    t = torch.from_numpy(arr) if arr.dtype != object else torch.tensor(data)
    return t.to(dtype=dtype).to(dev, non_blocking=False).contiguous()


def empty(shape, dtype: torch.dtype) -> torch.Tensor:
    return torch.empty(shape, dtype=dtype, device=device())


def flags() -> torch.Tensor:
    """A zeroed device word the kernels atomically OR their validation bits into."""
    return torch.zeros(1, dtype=torch.int32, device=device())


def read_flags(flag_t: torch.Tensor) -> int:
    return int(flag_t.item()) & 0xFFFFFFFF


def _hz_ratio(control_hz) -> tuple[int, int]:
    fr = Fraction(control_hz)
    if fr.numerator > INT64_MAX or fr.denominator > INT64_MAX:
        raise ValueError(f"control_hz {control_hz!r} has no int64 rational form")
    return fr.numerator, fr.denominator


_hz_cached = functools.lru_cache(maxsize=64)(_hz_ratio)


def hz_ratio(control_hz) -> tuple[int, int]:
    """Exact integer ratio of control_hz (core.py:42 takes floats at their exact
    binary value); both parts must fit the C ABI's int64."""
    try:
        return _hz_cached(control_hz)
    except TypeError:  # unhashable numeric types
        return _hz_ratio(control_hz)


def stream() -> int:
    return _lib.stream_handle()


class MappedArena(threading.local):
    """Per-thread mapped pinned host buffer for small calls (plan() at the
    simulator's sizes, the scalar drop-ins): the host writes a call's inputs
    into it, the kernel reads them over PCIe (zero-copy) and writes its
    results back into it, and one stream synchronisation returns them -- one
    launch per call, no device allocation, no copy calls.  Grows by doubling;
    every call waits for its kernel before the buffer is reused."""

    def __init__(self):
        self.nbytes = 0
        self.blob = None
        self.host = None
        self.dbase = 0
        self.scratch = None  # device buffer for kernels that stream from HBM (TMA)

    def device_scratch(self, nbytes: int) -> int:
        """Address of a per-thread device buffer of >= nbytes (grows by doubling)."""
        if self.scratch is None or self.scratch.numel() < nbytes:
            size = max(1 << 16, 1 << (max(nbytes, 1) - 1).bit_length())
            self.scratch = torch.empty(size, dtype=torch.uint8, device=device())
        return self.scratch.data_ptr()

    def ensure(self, nbytes: int) -> "MappedArena":
        if nbytes > self.nbytes or self.blob is None:
            size = max(1 << 16, 1 << (max(nbytes, 1) - 1).bit_length())
            blob = torch.empty(size, dtype=torch.uint8, pin_memory=True)
            dptr = ctypes.c_void_p()
            _lib.check(_lib.load().kr_mapped_ptr(blob.data_ptr(), ctypes.byref(dptr)),
                       "kr_mapped_ptr")
            self.blob, self.host, self.dbase, self.nbytes = blob, blob.numpy(), int(dptr.value), size
        return self


_ARENA = MappedArena()


def arena(nbytes: int = 0) -> MappedArena:
    if nbytes > _ARENA.nbytes or _ARENA.blob is None:
        device()
        _ARENA.ensure(nbytes)
    return _ARENA


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def raw_stream() -> int:
    """cudaStream_t of the current stream (cheap path for per-call launches)."""
    if _raw_stream is not None:
        return _raw_stream(torch._C._cuda_getDevice())
    return torch.cuda.current_stream().cuda_stream


def sync(stream_handle: int) -> None:
    """cudaStreamSynchronize through the C ABI (raises on a CUDA error)."""
    _lib.check(_lib.load().kr_stream_synchronize(stream_handle), "kr_stream_synchronize")
