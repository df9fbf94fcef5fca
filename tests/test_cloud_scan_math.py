"""The phase-3 offload scan as the device computes it (kr_select.cu
k_place_cloud), checked on CPU against the reference's greedy walk
(scheduler.py:210-221): with m_r = #{c < cap : T(c) > up_r} (T non-increasing)
the walk is fire_r = [c_r < m_r]; the kernel resolves it 32 requests at a time
by a ballot fixed point.  Host-only (numpy restatement of the kernel's steps)."""
from __future__ import annotations

import numpy as np
import pytest


def greedy(up, T, cap):
    c, fired = 0, []
    for r, u in enumerate(up):
        if c < cap and u < T[c]:
            fired.append(r)
            c += 1
    return fired


def ballot_fixed_point(up, T, cap):
    m = np.searchsorted(-np.asarray(T[:cap]), -np.asarray(up), side="left")  # #{c: T(c) > u}
    c, fired = 0, []
    for base in range(0, len(up), 32):
        mm = m[base:base + 32]
        f = (c < mm)                       # "no earlier fires in the chunk"
        for _ in range(33):
            g = (c + np.concatenate([[0], np.cumsum(f)[:-1]]) < mm)
            if np.array_equal(g, f):
                break
            f = g
        else:
            raise AssertionError("no fixed point")
        fired += [base + i for i in np.nonzero(f)[0]]
        c += int(f.sum())
    return fired


@pytest.mark.parametrize("seed", range(40))
def test_ballot_fixed_point_equals_greedy(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 3000))
    cap = int(rng.integers(1, 400))
    T = np.sort(rng.integers(0, 1000, cap))[::-1].astype(np.int64)  # non-increasing
    if seed % 3 == 0:
        T = np.repeat(T[:1], cap)  # flat thresholds: a prefix of every qualifier fires
    up = rng.choice(rng.integers(0, 1100, 5), n).astype(np.int64)  # few distinct payloads
    if seed % 4 == 1:
        up = rng.choice(T, n).astype(np.int64)  # uplinks equal to thresholds: T(c) > up is strict
    assert ballot_fixed_point(up, T, cap) == greedy(up, T, cap)
