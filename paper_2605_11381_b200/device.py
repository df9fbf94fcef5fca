"""Device plumbing shared by the drop-in modules: host->device staging of small
inputs, the validation-flag word, and raising the reference's ValueErrors
from flags the kernels set."""

from __future__ import annotations

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


def hz_ratio(control_hz) -> tuple[int, int]:
    """Exact integer ratio of control_hz (core.py:42 takes floats at their exact
    binary value); both parts must fit the C ABI's int64."""
    fr = Fraction(control_hz)
    if fr.numerator > INT64_MAX or fr.denominator > INT64_MAX:
        raise ValueError(f"control_hz {control_hz!r} has no int64 rational form")
    return fr.numerator, fr.denominator


def stream() -> int:
    return _lib.stream_handle()
