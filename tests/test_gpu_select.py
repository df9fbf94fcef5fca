"""Device radix select / sort / admission vs numpy on unique 128-bit keys."""

from __future__ import annotations

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _keys(n, rng, spread):
    hi = rng.integers(0, spread, n, dtype=np.uint64) << np.uint64(40)
    hi |= rng.integers(0, 1 << 20, n, dtype=np.uint64)
    lo = (rng.integers(0, 1 << 30, n, dtype=np.uint64) << np.uint64(24)) | np.arange(n, dtype=np.uint64)
    k = np.stack([hi, lo], 1)
    return k


def _order(k):
    return np.lexsort((k[:, 1], k[:, 0]))


@pytest.mark.parametrize("n", [1, 2, 3, 100, 4097, 8192, 8193, 70000, 1 << 20])
@pytest.mark.parametrize("spread", [1, 16, 1 << 24])
def test_sort_keys(n, spread):
    from paper_2605_11381_b200 import fleet as fl
    rng = np.random.default_rng(n + spread)
    k = _keys(n, rng, spread)
    kt = torch.from_numpy(k.view(np.int64)).cuda()
    order, sk = fl.sort_keys(kt, fl.Workspace(n))
    exp = _order(k)
    assert np.array_equal(order.cpu().numpy(), exp)
    assert np.array_equal(sk.cpu().numpy().view(np.uint64), k[exp])


@pytest.mark.parametrize("n,k", [(10, 1), (10, 9), (1000, 64), (1 << 16, 1024), (1 << 20, 8192),
                                 (1 << 20, 1), (1 << 20, (1 << 20) - 1), (300000, 20000)])
@pytest.mark.parametrize("spread", [1, 10, 1 << 30])
def test_topk_select_and_admit(n, k, spread):
    from paper_2605_11381_b200 import fleet as fl
    rng = np.random.default_rng(n * 3 + k + spread)
    keys = _keys(n, rng, spread)
    kt = torch.from_numpy(keys.view(np.int64)).cuda()
    ws = fl.Workspace(n)
    kth = fl.topk_select(kt, k, ws)
    exp = _order(keys)
    assert np.array_equal(kth.cpu().numpy().view(np.uint64)[0], keys[exp[k - 1]])
    adm = torch.empty(n, dtype=torch.uint8, device="cuda")
    edge_idx = torch.empty(k, dtype=torch.int32, device="cuda")
    fl.admit(kt, k, kth.data_ptr(), None, None, ws, admitted=adm, edge_idx=edge_idx)
    mask = np.zeros(n, bool)
    mask[exp[:k]] = True
    assert np.array_equal(adm.cpu().numpy().astype(bool), mask)
    assert np.array_equal(edge_idx.cpu().numpy(), exp[:k])


def test_admit_all_and_none():
    from paper_2605_11381_b200 import fleet as fl
    rng = np.random.default_rng(1)
    keys = _keys(500, rng, 7)
    kt = torch.from_numpy(keys.view(np.int64)).cuda()
    ws = fl.Workspace(500)
    adm = torch.empty(500, dtype=torch.uint8, device="cuda")
    idx = torch.empty(500, dtype=torch.int32, device="cuda")
    fl.admit(kt, 500, None, None, None, ws, admitted=adm, edge_idx=idx)
    assert adm.all() and np.array_equal(idx.cpu().numpy(), _order(keys))
    fl.admit(kt, 0, None, None, None, ws, admitted=adm)
    assert not adm.any()


def _skewed(n, rng, mode):
    if mode == "dense_low_bin":      # > kSegMax admitted keys share the level-0 bin
        hi = np.where(rng.random(n) < 0.7, 0, rng.integers(1, 1 << 11, n)).astype(np.uint64) << np.uint64(40)
        lo = (rng.integers(0, 1 << 30, n, dtype=np.uint64) << np.uint64(24)) | np.arange(n, dtype=np.uint64)
    elif mode == "one_outlier":      # the top digit separates one key: the boundary bin
        hi = np.zeros(n, np.uint64)  # holds all others (the single-CTA finish does the rest)
        hi[n // 2] = np.uint64(1) << np.uint64(63)
        lo = (rng.integers(0, 1 << 30, n, dtype=np.uint64) << np.uint64(24)) | np.arange(n, dtype=np.uint64)
    elif mode == "few_bits":         # only rank bits differ
        hi = np.zeros(n, np.uint64)
        lo = rng.permutation(n).astype(np.uint64)
    else:                            # bucket field + wide gap + low aged bits (kairos-like)
        hi = (rng.integers(0, 10, n, dtype=np.uint64) << np.uint64(56)) | \
             ((np.uint64((1 << 56) - 1)) - rng.integers(1 << 18, 1 << 25, n, dtype=np.uint64))
        lo = (rng.integers(0, 1 << 20, n, dtype=np.uint64) << np.uint64(24)) | np.arange(n, dtype=np.uint64)
    return np.stack([hi, lo], 1)


@pytest.mark.parametrize("n,k,mode", [(1 << 20, 8192, "kairos"), (300000, 1024, "kairos"),
                                      (20000, 6000, "dense_low_bin"), (4096, 100, "few_bits"),
                                      (70000, 69999, "kairos"), (50, 49, "few_bits"),
                                      (1 << 16, 1 << 15, "kairos"), (2, 1, "kairos"),
                                      (1024, 64, "kairos"), (4096, 4095, "few_bits"),
                                      (4097, 4000, "kairos"), (12000, 1024, "kairos"),
                                      (16384, 16383, "few_bits"), (16384, 1, "kairos"),
                                      (16385, 1024, "kairos"), (9000, 4500, "dense_low_bin"),
                                      (300000, 1000, "one_outlier"), (1 << 18, (1 << 18) - 1,
                                                                       "one_outlier")])
def test_select_admit_fused(n, k, mode):
    from paper_2605_11381_b200 import fleet as fl
    rng = np.random.default_rng(n + k)
    keys = _skewed(n, rng, mode)
    kt = torch.from_numpy(keys.view(np.int64)).cuda()
    ws = fl.Workspace(n)
    exp = _order(keys)
    for use_stats in (False, True):
        stats = None
        if use_stats:
            stats = fl.new_key_stats()
            stats[0] = int(np.bitwise_or.reduce(keys[:, 0]).view(np.int64))
            stats[1] = int(np.bitwise_or.reduce(keys[:, 1]).view(np.int64))
            stats[2] = int(np.bitwise_and.reduce(keys[:, 0]).view(np.int64))
            stats[3] = int(np.bitwise_and.reduce(keys[:, 1]).view(np.int64))
        adm = torch.empty(n, dtype=torch.uint8, device="cuda")
        edge_idx = torch.empty(k, dtype=torch.int32, device="cuda")
        edge_keys = fl.new_keys(k)
        kth = fl.new_keys(1)
        fl.select_admit(kt, k, ws, key_stats=stats, admitted=adm, edge_idx=edge_idx,
                        edge_keys=edge_keys, kth=kth)
        mask = np.zeros(n, bool)
        mask[exp[:k]] = True
        assert np.array_equal(adm.cpu().numpy().astype(bool), mask)
        assert np.array_equal(edge_idx.cpu().numpy(), exp[:k])
        assert np.array_equal(edge_keys.cpu().numpy().view(np.uint64), keys[exp[:k]])
        assert np.array_equal(kth.cpu().numpy().view(np.uint64)[0], keys[exp[k - 1]])


@pytest.mark.parametrize("W,len_,fill", [(1, 50, 50), (8, 1024, 700), (3, 257, 0), (32, 64, 64),
                                         (40, 16, 9)])
def test_merge_runs(W, len_, fill):
    """kr_merge_runs over W ascending runs, each with `fill` real keys then the
    all-ones sentinel padding (a sharded round's all-gathered candidates)."""
    from paper_2605_11381_b200 import _lib, device as dev, fleet as fl
    rng = np.random.default_rng(W * 1000 + len_)
    runs = np.full((W, len_, 2), np.iinfo(np.uint64).max, np.uint64)
    real = []
    for w in range(W):
        f = int(rng.integers(0, fill + 1)) if fill else 0
        hi = rng.integers(0, 4, f, dtype=np.uint64) << np.uint64(60)
        lo = (rng.integers(0, 1 << 30, f, dtype=np.uint64) << np.uint64(24)) | \
            np.uint64(w * len_) + np.arange(f, dtype=np.uint64)  # unique keys
        k = np.stack([hi, lo], 1)
        k = k[_order(k)]
        runs[w, :f] = k
        real.append(k)
    allreal = np.concatenate(real) if real else np.zeros((0, 2), np.uint64)
    exp = allreal[_order(allreal)]
    t = torch.from_numpy(runs.reshape(-1, 2).view(np.int64)).cuda()
    for kk in sorted({1, max(1, len(exp) // 2), max(1, len(exp)), min(W * len_, len(exp) + 3)}):
        out = fl.new_keys(kk)
        kth = fl.new_keys(1)
        _lib.check(_lib.load().kr_merge_runs(t.data_ptr(), W, len_, kk, out.data_ptr(),
                                             kth.data_ptr(), None, dev.stream()), "kr_merge_runs")
        got = out.cpu().numpy().view(np.uint64)
        n_real = min(kk, len(exp))
        assert np.array_equal(got[:n_real], exp[:n_real])
        assert (got[n_real:] == np.iinfo(np.uint64).max).all()
        assert np.array_equal(kth.cpu().numpy().view(np.uint64)[0],
                              exp[kk - 1] if kk <= len(exp) else np.array([np.iinfo(np.uint64).max] * 2, np.uint64))
