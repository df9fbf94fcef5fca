"""`roboserve.workload` hot-path names (reference workload.py:461-496):
the divergence horizon lives in divergence.py; trace I/O and synthesis are
outside the decision core."""

from .divergence import _cosine, round_optimal_horizon, round_optimal_horizon_batch  # noqa: F401
