"""Step 1b: divergence-based execution horizon.

Drop-in for `roboserve.workload.round_optimal_horizon` / `_cosine`
(reference workload.py:461-496): the longest prefix of a candidate chunk whose
per-action cosine similarity to the reference trajectory stays at or above the
threshold.  At fleet scale the reference trajectory of robot r is the
unexecuted overlap of its previous chunk, prev[r, offset_r:], and a round may
carry S candidate samples; `round_optimal_horizon_batch` returns
H[r] = min_s round_optimal_horizon(prev[r, offset_r:len_prev_r],
cand[r, s, :len_cand_r], thr) from the `kr_horizon_divergence` CUDA kernel
(fp64 cosines in OpenBLAS' SkylakeX ddot order: bit-exact with numpy).
"""

from __future__ import annotations

from typing import Sequence

import numpy as np
import torch

from . import _lib
from . import device as dev


def set_dot_order(order: str) -> None:
    """Choose the OpenBLAS core whose ddot order the exact fp64 cosines follow:
    "skylakex" (SkylakeX / Cooperlake / SapphireRapids hosts) or "haswell"
    (Haswell / Zen hosts).  The default is the core numpy's own OpenBLAS runs
    in this process (threadpoolctl), so results match `numpy.dot` on this
    host; KR_DOT_ORDER overrides it at load.  Process-wide, like OpenBLAS'."""
    if order not in _lib.DOT_ORDERS:
        raise ValueError(f"dot order must be one of {sorted(_lib.DOT_ORDERS)}, got {order!r}")
    _lib.check(_lib.load().kr_set_dot_order(_lib.DOT_ORDERS[order]), "kr_set_dot_order")


def dot_order() -> str:
    code = _lib.load().kr_get_dot_order()
    return next(k for k, v in _lib.DOT_ORDERS.items() if v == code)


def _check_thr(sim_threshold: float) -> None:
    if not 0.0 < sim_threshold <= 1.0:
        raise ValueError(f"sim_threshold must be in (0, 1], got {sim_threshold}")


def round_optimal_horizon_batch(prev: torch.Tensor, cand: torch.Tensor, sim_threshold: float,
                                offset: torch.Tensor | None = None,
                                len_prev: torch.Tensor | None = None,
                                len_cand: torch.Tensor | None = None,
                                return_cos: bool = False, out: torch.Tensor | None = None):
    """Per-robot divergence horizons for device tensors.

    prev: [R, Lp, D]; cand: [R, Lc, D] or [R, S, Lc, D] (same float dtype).
    offset / len_prev / len_cand: optional int32 [R] (defaults 0 / Lp / Lc).
    Returns int32 H[R] (and fp64 cos[R, S, Lc], NaN past each limit).
    Fully asynchronous on the current stream.
    """
    _check_thr(sim_threshold)
    if cand.dim() == 3:
        cand = cand.unsqueeze(1)
    if prev.dim() != 3 or cand.dim() != 4:
        raise ValueError(f"trajectories must be [R,L,D] / [R,S,L,D], got shapes "
                         f"{tuple(prev.shape)} and {tuple(cand.shape)}")
    if prev.shape[0] != cand.shape[0] or prev.shape[2] != cand.shape[3]:
        raise ValueError(f"trajectories must share action dimensionality, got shapes "
                         f"{tuple(prev.shape)} and {tuple(cand.shape)}")
    if prev.dtype != cand.dtype or prev.dtype not in (torch.float32, torch.float64):
        raise ValueError("prev and cand must share a float32 / float64 dtype")
    d = dev.device()
    prev = prev.to(d).contiguous()
    cand = cand.to(d).contiguous()
    R, Lp, D = prev.shape
    S, Lc = cand.shape[1], cand.shape[2]

    def opt(t):
        return None if t is None else t.to(device=d, dtype=torch.int32).contiguous()

    offset, len_prev, len_cand = opt(offset), opt(len_prev), opt(len_cand)
    if out is None:
        out = torch.empty(R, dtype=torch.int32, device=d)
    cos = torch.empty((R, S, Lc), dtype=torch.float64, device=d) if return_cos else None
    dtype = _lib.KR_F64 if prev.dtype == torch.float64 else _lib.KR_F32
    _lib.check(_lib.load().kr_horizon_divergence(
        prev.data_ptr(), cand.data_ptr(), dtype, R, S, Lp, Lc, D, _lib.ptr(offset),
        _lib.ptr(len_prev), _lib.ptr(len_cand), float(sim_threshold), out.data_ptr(),
        _lib.ptr(cos), 0, dev.stream()), "kr_horizon_divergence")
    return (out, cos) if return_cos else out


def _cosine(a, b) -> float:
    """workload.py:461-468 on one pair of action vectors (device kernel)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    prev = dev.tensor(b[None, None, :], torch.float64)
    cand = dev.tensor(a[None, None, :], torch.float64)
    _, cos = round_optimal_horizon_batch(prev, cand, 1.0, return_cos=True)
    return float(cos[0, 0, 0].item())


def round_optimal_horizon(reference: Sequence[Sequence[float]],
                          candidate: Sequence[Sequence[float]], sim_threshold: float) -> int:
    """Longest candidate prefix tracking the reference (workload.py:471-496)."""
    _check_thr(sim_threshold)
    ref = np.asarray(reference, dtype=np.float64)
    cand = np.asarray(candidate, dtype=np.float64)
    if ref.ndim != 2 or cand.ndim != 2 or ref.shape[1] != cand.shape[1]:
        raise ValueError(f"trajectories must share action dimensionality, got shapes "
                         f"{ref.shape} and {cand.shape}")
    (Lp, D), Lc = ref.shape, cand.shape[0]
    if Lp == 0 or Lc == 0 or D == 0:
        H = round_optimal_horizon_batch(dev.tensor(ref[None], torch.float64),
                                        dev.tensor(cand[None], torch.float64), sim_threshold)
        return int(H.item())
    # both trajectories staged through the mapped arena into device scratch
    # (the kernel's TMA reads HBM), the horizon returned through the arena:
    # one copy, one launch, one synchronisation
    nb = 8 * (ref.size + cand.size)
    a = dev.arena(nb + 64)
    f = a.host[64:64 + nb].view(np.float64)
    f[:ref.size] = ref.reshape(-1)
    f[ref.size:] = cand.reshape(-1)
    scr = a.device_scratch(nb)
    st = dev.raw_stream()
    lib = _lib.load()
    _lib.check(lib.kr_memcpy_async(scr, a.dbase + 64, nb, st), "kr_memcpy_async")
    _lib.check(lib.kr_horizon_divergence(scr, scr + 8 * ref.size, _lib.KR_F64, 1, 1, Lp, Lc, D,
                                         None, None, None, float(sim_threshold), a.dbase, None, 0,
                                         st), "kr_horizon_divergence")
    dev.sync(st)
    return int(a.host[:4].view(np.int32)[0])
