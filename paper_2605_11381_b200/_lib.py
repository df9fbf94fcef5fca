"""ctypes binding of libkairos_b200.so (include/kairos_b200.h).

The decision core has no CPU fallback: if the library is missing, or no CUDA
device is visible, every compute entry point raises instead of silently
computing on the host.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import torch

_PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ["KR_LIB_PATH"]) if os.environ.get("KR_LIB_PATH") else _PKG / "libkairos_b200.so"  # KR_LIB_PATH: A/B builds (tools/)

KR_OK, KR_EINVAL, KR_ECUDA, KR_ENOSPACE, KR_EFORMAT = 0, 1, 2, 3, 4
KR_F32, KR_F64 = 0, 1
KR_KAIROS, KR_FIFO, KR_LAS = 0, 1, 2

FLAG_NONFINITE = 0x1
FLAG_NEGATIVE = 0x2
FLAG_KEY_RANGE = 0x4
FLAG_TIME_RANGE = 0x8
FLAG_RATIO = 0x10
FLAG_LEDGER = 0x20
FLAG_DUP_KEY = 0x40

_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32
_f64 = ctypes.c_double


class KrFleet(ctypes.Structure):
    """kr_fleet: device pointers of the fleet structure-of-arrays."""

    _fields_ = [("n", _i64)] + [(name, _vp) for name in (
        "t_start", "issued_at", "obs_captured_at", "accum_gen", "remaining", "lexrank",
        "skipped", "hist_off", "n_exec", "n_gen", "slots")]


class KrSched(ctypes.Structure):
    """kr_sched: SchedulerConfig plus the round's scalars."""

    _fields_ = [("policy", _i32), ("buckets", _i32), ("aging_interval", _i32), ("pad_", _i32),
                ("stale_threshold", _i64), ("default_exec_estimate", _i64), ("now", _i64),
                ("hz_num", _i64), ("hz_den", _i64), ("issued_base", _i64)]


class KrLedger(ctypes.Structure):
    """kr_ledger: device-resident per-task state and history."""

    _fields_ = [("n_tasks", _i64), ("cap", _i32), ("pad_", _i32)] + [(k, _vp) for k in (
        "t_start", "n_exec", "n_gen", "wait_next", "wait_total", "slots")]


class KrEvents(ctypes.Structure):
    """kr_events: TaskState mutations grouped by task."""

    _fields_ = [("n_groups", _i64)] + [(k, _vp) for k in ("task", "off", "kind", "round", "a", "b")]


class KrRequests(ctypes.Structure):
    """kr_requests: one planning round's pending requests against a kr_ledger."""

    _fields_ = [("n", _i64)] + [(k, _vp) for k in (
        "task", "issued_at", "obs_captured_at", "accum_gen", "remaining", "lexrank", "skipped")]


class KrTraceColumns(ctypes.Structure):
    """kr_trace_columns: columnar view of a parsed trace file (host memory)."""

    _fields_ = ([(k, _i64) for k in ("n_traces", "n_rounds", "n_mag_values", "n_traj_rows",
                                      "n_traj_values")] +
                [(k, _vp) for k in (
                    "round_off", "ids", "id_off", "control_hz", "control_hz_is_int",
                    "obs_payload_bytes", "action_payload_bytes", "success", "round_id",
                    "trigger_action_index", "horizon", "chunk_size", "mag_k", "mag_n", "mag_off",
                    "mags", "traj_rows", "traj_row0", "traj_off", "traj")] +
                [("err_line", _i64), ("err_has_task", _i32), ("err_has_round", _i32),
                 ("err_task", ctypes.c_char_p), ("err_round", _i64),
                 ("err_message", ctypes.c_char_p)])


class KrSynthSpec(ctypes.Structure):
    """kr_synth_spec: the SyntheticSpec fields the synthesis kernels read."""

    _fields_ = [("chunk_size", _i32), ("diffusion_steps", _i32), ("decay", ctypes.c_double),
                ("noise_scale", ctypes.c_double), ("bump_factor", ctypes.c_double),
                ("uncertain_fraction", ctypes.c_double)]


_SIGNATURES = {
    "kr_version": (ctypes.c_char_p, []),
    "kr_status_string": (ctypes.c_char_p, [ctypes.c_int]),
    "kr_last_error": (ctypes.c_char_p, []),
    "kr_launch_count": (ctypes.c_ulonglong, []),
    "kr_horizon_confidence": (ctypes.c_int, [_vp, ctypes.c_int, _i64, _i32, _i32, _f64, _i32,
                                             _vp, _vp, _i32, _vp]),
    "kr_horizon_static": (ctypes.c_int, [_i64, _i32, _i32, _vp, _vp]),
    "kr_horizon_sweep": (ctypes.c_int, [_vp, ctypes.c_int, _i64, _i32, _i32, _i32, _vp, _vp, _vp,
                                        _vp, _vp, _vp, _vp]),
    "kr_horizon_divergence": (ctypes.c_int, [_vp, _vp, ctypes.c_int, _i64, _i32, _i32, _i32,
                                             _i32, _vp, _vp, _vp, _f64, _vp, _vp, _i32, _vp]),
    "kr_us_from_actions": (ctypes.c_int, [_vp, _vp, _i64, _i64, _i64, _vp, _vp, _vp]),
    "kr_wait_ratio": (ctypes.c_int, [_vp, _vp, _i64, _i64, _vp, _vp, _vp]),
    "kr_assign_bucket": (ctypes.c_int, [_vp, _vp, _i64, _i32, _i32, _vp, _vp]),
    "kr_urgency": (ctypes.c_int, [ctypes.POINTER(KrFleet), ctypes.POINTER(KrSched), _vp, _vp,
                                  _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "kr_key_stats_init": (ctypes.c_int, [_vp, _vp]),
    "kr_urgency_prep": (ctypes.c_int, [ctypes.POINTER(KrFleet), ctypes.POINTER(KrSched), _vp, _vp,
                                       _vp, _i64, _vp, ctypes.c_size_t, _vp]),
    "kr_plan_small": (ctypes.c_int, [ctypes.POINTER(KrFleet), ctypes.POINTER(KrSched), _i64, _vp,
                                     _vp]),
    "kr_mapped_ptr": (ctypes.c_int, [_vp, ctypes.POINTER(ctypes.c_void_p)]),
    "kr_memcpy_async": (ctypes.c_int, [_vp, _vp, ctypes.c_size_t, _vp]),
    "kr_stream_synchronize": (ctypes.c_int, [_vp]),
    "kr_ledger_apply": (ctypes.c_int, [ctypes.POINTER(KrLedger), ctypes.POINTER(KrEvents), _vp,
                                       _vp]),
    "kr_urgency_ledger": (ctypes.c_int, [ctypes.POINTER(KrLedger), ctypes.POINTER(KrRequests),
                                         ctypes.POINTER(KrSched), _vp, _vp, _vp, _vp, _vp, _vp,
                                         _vp, _vp, _vp]),
    "kr_workspace_bytes": (ctypes.c_size_t, [_i64]),
    "kr_topk_select": (ctypes.c_int, [_vp, _i64, _i64, _vp, _vp, _vp, ctypes.c_size_t, _vp]),
    "kr_select_admit": (ctypes.c_int, [_vp, _i64, _i64, _vp, ctypes.POINTER(KrFleet),
                                       ctypes.POINTER(KrSched), _vp, _vp, _vp, _vp, _vp, _vp,
                                       ctypes.c_size_t, _vp]),
    "kr_select_admit_prepared": (ctypes.c_int, [_vp, _i64, _i64, ctypes.POINTER(KrFleet),
                                                ctypes.POINTER(KrSched), _vp, _vp, _vp, _vp, _vp,
                                                _vp, ctypes.c_size_t, _vp]),
    "kr_admit": (ctypes.c_int, [_vp, _i64, _i64, _vp, ctypes.POINTER(KrFleet),
                                ctypes.POINTER(KrSched), _vp, _vp, _vp, _vp, _vp,
                                ctypes.c_size_t, _vp]),
    "kr_sort_keys": (ctypes.c_int, [_vp, _i64, _vp, _vp, _vp, ctypes.c_size_t, _vp]),
    "kr_merge_runs": (ctypes.c_int, [_vp, _i32, _i64, _i64, _vp, _vp, _vp, _vp]),
    "kr_merge_runs_pos": (ctypes.c_int, [_vp, _i32, _i64, _i64, _vp, _vp, _vp, _vp, _vp]),
    "kr_transfer_time": (ctypes.c_int, [_vp, _i64, _i64, _i64, _vp, _vp]),
    "kr_trace_parse": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_size_t, _i64,
                                      ctypes.POINTER(_vp)]),
    "kr_trace_load": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(_vp)]),
    "kr_trace_columns_of": (ctypes.POINTER(KrTraceColumns), [_vp]),
    "kr_trace_free": (None, [_vp]),
    "kr_synth_magnitudes": (ctypes.c_int, [ctypes.POINTER(KrSynthSpec), ctypes.c_uint64, _vp, _i64,
                                            _i32, _i32, _vp, _vp]),
    "kr_synth_close": (ctypes.c_int, [_vp, _i64, _i32, _i32, _i32, _vp, _vp, _vp, _vp]),
    "kr_synth_success": (ctypes.c_int, [ctypes.c_uint64, _vp, _i64, ctypes.c_double, _vp, _vp]),
    "kr_synth_trajectories": (ctypes.c_int, [ctypes.c_uint64, _vp, _vp, _vp, _vp, _i64, _i32, _vp,
                                              _vp]),
    "kr_set_dot_order": (ctypes.c_int, [_i32]),
    "kr_get_dot_order": (_i32, []),
    "kr_place_cloud": (ctypes.c_int, [_vp, _i64, _i64, _vp, _vp, _i64, ctypes.POINTER(KrFleet),
                                      ctypes.POINTER(KrSched), _vp, _vp, _vp, _vp]),
    "kr_apply_placements": (ctypes.c_int, [_vp, _vp, _i64, _i64, _i32, _vp,
                                           ctypes.POINTER(KrFleet), ctypes.POINTER(KrSched), _vp,
                                           _vp]),
}

EXPORTED = tuple(_SIGNATURES)

_LIB = None


class KairosError(RuntimeError):
    """A C-ABI call failed (bad argument or CUDA error)."""


def load(path: os.PathLike | None = None) -> ctypes.CDLL:
    """Load the in-tree library; raise loudly if it has not been built."""
    global _LIB
    if _LIB is not None and path is None:
        return _LIB
    p = Path(path) if path is not None else LIB_PATH
    if not p.exists():
        raise ImportError(
            f"{p} is missing: the B200 decision core has no CPU fallback. Build it with "
            "`python -m paper_2605_11381_b200.build_lib` (nvcc, sm_100a).")
    lib = ctypes.CDLL(str(p))
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    lib.kr_set_dot_order(DOT_ORDERS[_dot_order_choice()[0]])
    if path is None:
        _LIB = lib
    return lib


# --- exact-cosine ddot order (workload.py:461-468 through numpy's OpenBLAS) ----
DOT_ORDERS = {"skylakex": 0, "haswell": 1}
# OpenBLAS 0.3.30 runtime cores -> the ddot kernel they run (kernel/x86_64/ddot.c
# with the skylakex / haswell micro-kernels; Zen shares Haswell's kernels)
_CORE_ORDER = {"skylakex": "skylakex", "cooperlake": "skylakex", "sapphirerapids": "skylakex",
               "haswell": "haswell", "zen": "haswell"}
_DOT_CHOICE = None


def numpy_blas_core() -> str | None:
    """The OpenBLAS core numpy's own BLAS runs in this process (threadpoolctl),
    or None when numpy is not on OpenBLAS / threadpoolctl is unavailable."""
    try:
        import numpy  # noqa: F401  (its BLAS must be loaded to be reported)
        import threadpoolctl
    except ImportError:
        return None
    infos = [i for i in threadpoolctl.threadpool_info() if i.get("internal_api") == "openblas"]
    infos.sort(key=lambda i: "numpy" not in i.get("filepath", ""))
    return infos[0].get("architecture") if infos else None


def _dot_order_choice() -> tuple[str, str]:
    """(order, why): KR_DOT_ORDER=skylakex|haswell overrides; otherwise the
    order of numpy's OpenBLAS core; SkylakeX (with a warning) when that core's
    order is not one this library reproduces."""
    global _DOT_CHOICE
    if _DOT_CHOICE is None:
        env = os.environ.get("KR_DOT_ORDER", "auto").lower()
        if env in DOT_ORDERS:
            _DOT_CHOICE = (env, "KR_DOT_ORDER")
        else:
            core = numpy_blas_core()
            order = _CORE_ORDER.get((core or "").lower())
            if order is None:
                import warnings
                warnings.warn(f"numpy's BLAS core {core!r} has no reproduced ddot order; exact "
                              "cosines follow OpenBLAS SkylakeX (set KR_DOT_ORDER to choose)",
                              RuntimeWarning, stacklevel=3)
                order = "skylakex"
            _DOT_CHOICE = (order, f"numpy OpenBLAS core {core}")
    return _DOT_CHOICE


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("a CUDA device (B200, sm_100a) is required: the Kairos decision core "
                           "runs only as CUDA kernels and has no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def stream_handle(stream: torch.cuda.Stream | None = None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def check(status: int, what: str) -> None:
    if status != KR_OK:
        lib = load()
        msg = lib.kr_status_string(status).decode()
        detail = lib.kr_last_error().decode() if status == KR_ECUDA else ""
        raise KairosError(f"{what}: {msg}" + (f" ({detail})" if detail else ""))


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()
