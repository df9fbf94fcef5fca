"""Step 2 (kr_urgency) on fleets whose CSR history layout exercises both paths
of the warp-segmented pass (kr_urgency.cu k_urgency_warp): compact robot-order
histories (slot-parallel segmented walk), scrambled / gapped / overlapping
layouts and histories longer than the per-warp span (per-lane walk), mixed
inside one warp -- every intermediate (total wait, wait ratio, bucket,
estimate, need time) and the resulting order vs the oracle
(waiting.py:69-100, scheduler.py:79-140), bit-exact."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import oracle as orc

pytestmark = pytest.mark.gpu

SCHED = ("kairos", 10, 5, 150_000, 166_667)


def _check(soa, k=None):
    from paper_2605_11381_b200 import fleet as fl, synthetic
    n = soa["n"]
    k = n // 3 if k is None else k
    fleet = fl.DeviceFleet.from_host(soa)
    sched = fl.sched_struct(*SCHED, synthetic.NOW, 30, int(soa["issued_at"].min()))
    u = fl.urgency(fleet, sched, intermediates=True)
    torch.cuda.synchronize()
    res = orc.plan_soa(soa, *SCHED, synthetic.NOW, 30, k)
    assert np.array_equal(u.total_wait.cpu().numpy(), res["total_wait"])
    assert np.array_equal(u.wr.cpu().numpy().view(np.int64), res["wr"].view(np.int64))
    assert np.array_equal(u.bucket.cpu().numpy(), res["bucket"])
    assert np.array_equal(u.est.cpu().numpy(), res["est"])
    assert np.array_equal(u.need_time.cpu().numpy(), res["need_time"])
    keys = u.keys.cpu().numpy().view(np.uint64).reshape(-1, 2)
    order = np.lexsort((keys[:, 1], keys[:, 0]))
    assert np.array_equal(order, res["order"])


def _relayout(soa, rng, mode):
    """Same histories, different CSR placement of each robot's slot block."""
    n = soa["n"]
    nslots = np.maximum(soa["n_exec"], soa["n_gen"]).astype(np.int64)
    blocks = [soa["slots"][o:o + m] for o, m in zip(soa["hist_off"], nslots)]
    if mode == "reversed":            # robot order reversed in the slot array
        place = np.arange(n)[::-1]
    elif mode == "shuffled":          # random robot order
        place = rng.permutation(n)
    else:                             # robot order, random gaps between blocks
        place = np.arange(n)
    gaps = rng.integers(0, 3, n) if mode == "gapped" else np.zeros(n, np.int64)
    off = np.empty(n, np.int64)
    pos = 0
    for r in place:
        pos += gaps[r]
        off[r] = pos
        pos += nslots[r]
    slots = np.full((max(pos, 1), 4), -7, np.int64)
    for r in range(n):
        slots[off[r]:off[r] + nslots[r]] = blocks[r]
    out = dict(soa)
    out["hist_off"], out["slots"] = off, slots
    return out


@pytest.mark.parametrize("R", [1, 31, 33, 1000, 100_003, 1 << 20])
def test_urgency_compact(R):
    from paper_2605_11381_b200 import synthetic
    _check(synthetic.fleet_soa(R, seed=R))


@pytest.mark.parametrize("mode", ["reversed", "shuffled", "gapped"])
def test_urgency_relayout(mode):
    from paper_2605_11381_b200 import synthetic
    R = 20_011
    soa = synthetic.fleet_soa(R, seed=5)
    _check(_relayout(soa, np.random.default_rng(1), mode))


def test_urgency_shared_and_long_histories():
    """Robots sharing one slot block (overlapping ranges) and histories of up
    to 80 rounds (spans beyond the segmented path's cap) next to short ones."""
    from paper_2605_11381_b200 import synthetic
    R = 4096
    soa = synthetic.fleet_soa(R, seed=3, max_rounds=5)
    rng = np.random.default_rng(2)
    long_ = synthetic.fleet_soa(64, seed=4, max_rounds=80)
    # robots 0..63 of every 512 get an 80-round history appended at the end
    nsl = np.maximum(soa["n_exec"], soa["n_gen"]).astype(np.int64)
    slots = [soa["slots"]]
    pos = soa["slots"].shape[0]
    lnsl = np.maximum(long_["n_exec"], long_["n_gen"]).astype(np.int64)
    for r in range(0, R, 512):
        for j in range(64):
            L = long_["slots"][long_["hist_off"][j]:long_["hist_off"][j] + lnsl[j]]
            soa["hist_off"][r + j] = pos
            soa["n_exec"][r + j] = long_["n_exec"][j]
            soa["n_gen"][r + j] = long_["n_gen"][j]
            soa["t_start"][r + j] = long_["t_start"][j]
            slots.append(L)
            pos += L.shape[0]
    # pairs of robots sharing one history block (identical ranges)
    for r in range(1000, 1200, 2):
        for f in ("hist_off", "n_exec", "n_gen", "t_start"):
            soa[f][r + 1] = soa[f][r]
    soa["slots"] = np.concatenate(slots)
    assert nsl.sum() <= soa["slots"].shape[0]
    _check(soa, k=777)
    del rng
