"""Step 1 on the GPU vs the reference's golden vectors and the CPU oracle:
bit-exact horizons (and bit-exact fp64 cosine scores)."""

from __future__ import annotations

from collections import defaultdict

import numpy as np
import pytest
import torch

import golden_io
from oracle import oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def kb():
    import paper_2605_11381_b200 as kb
    return kb


def test_confidence_golden_scalar(kb):
    cases = golden_io.confidence_cases()
    bad = []
    for i, (u, t, hmin, exp) in enumerate(cases[::7]):
        cfg = kb.HorizonPolicyConfig.confidence(threshold=t, min_horizon=hmin)
        if kb.decide_horizon(cfg, kb.UpdateMagnitudes(u)) != exp:
            bad.append(i)
    assert not bad


@pytest.mark.parametrize("storage", [torch.float64, torch.float32])
def test_confidence_golden_batched(kb, storage):
    groups = defaultdict(list)
    for u, t, hmin, exp in golden_io.confidence_cases():
        if storage == torch.float32 and not np.array_equal(u.astype(np.float32).astype(np.float64), u):
            continue
        groups[(u.shape, t, hmin)].append((u, exp))
    checked = 0
    for (shape, t, hmin), items in groups.items():
        U = torch.tensor(np.stack([u for u, _ in items]), dtype=storage, device="cuda")
        H = kb.decide_horizon_batch(kb.HorizonPolicyConfig.confidence(t, hmin), U)
        assert H.cpu().tolist() == [e for _, e in items], (shape, t, hmin)
        checked += len(items)
    assert checked > 300


@pytest.mark.parametrize("R,K,N", [(1, 2, 1), (37, 6, 50), (4099, 6, 64), (1000, 10, 50),
                                   (513, 3, 1), (64, 130, 1), (257, 4, 300)])
@pytest.mark.parametrize("storage", [np.float32, np.float64])
def test_confidence_random_vs_oracle(kb, R, K, N, storage):
    rng = np.random.default_rng(R * 31 + K * 7 + N)
    U = (rng.uniform(0.5, 2.0, (R, 1, N)) * rng.uniform(0.3, 0.8, (R, 1, N)) **
         np.arange(K)[None, :, None] * rng.uniform(0.95, 1.05, (R, K, N)))
    tail = rng.integers(0, N + 1, R)
    for r in range(R):
        if tail[r] < N:
            U[r, -1, tail[r]:] = 1.8 * U[r, :-1, tail[r]:].mean(axis=0)
    U = U.astype(storage)
    for t, hmin in [(0.4, 5), (0.8, 1), (0.0, 1)]:
        exp = orc.horizon_conf_batch(U, t, hmin)
        H = kb.decide_horizon_batch(kb.HorizonPolicyConfig.confidence(t, hmin),
                                    torch.from_numpy(U).cuda())
        assert np.array_equal(H.cpu().numpy(), exp)


def test_confidence_unaligned_and_static(kb):
    rng = np.random.default_rng(3)
    base = torch.tensor(rng.uniform(0, 1, 1 + 33 * 6 * 7), dtype=torch.float32, device="cuda")
    U = base[1:].view(33, 6, 7)          # 4-byte aligned only: plain-staging path
    exp = orc.horizon_conf_batch(U.cpu().numpy(), 0.4, 2)
    H = kb.decide_horizon_batch(kb.HorizonPolicyConfig.confidence(0.4, 2), U)
    assert np.array_equal(H.cpu().numpy(), exp)
    Hs = kb.decide_horizon_batch(kb.HorizonPolicyConfig.static(5), U)
    assert (Hs == 5).all()


def test_confidence_validation_flags(kb):
    U = torch.ones(8, 3, 4, dtype=torch.float32, device="cuda")
    U[5, 1, 2] = float("nan")
    with pytest.raises(ValueError, match="finite"):
        kb.decide_horizon_batch(kb.HorizonPolicyConfig.confidence(), U)
    U[5, 1, 2] = -1.0
    with pytest.raises(ValueError, match=">= 0"):
        kb.decide_horizon_batch(kb.HorizonPolicyConfig.confidence(), U)


def test_divergence_golden(kb):
    from paper_2605_11381_b200.divergence import round_optimal_horizon_batch
    bad_h, bad_c = [], []
    for i, (ref, cand, thr, exp, cos) in enumerate(golden_io.divergence_cases()):
        H, c = round_optimal_horizon_batch(torch.tensor(ref[None], device="cuda"),
                                           torch.tensor(cand[None], device="cuda"), thr,
                                           return_cos=True)
        if int(H.item()) != exp:
            bad_h.append(i)
        got = c[0, 0, :len(cos)].cpu().numpy()
        if not np.array_equal(got, cos):
            bad_c.append(i)
        if i % 9 == 0:
            assert kb.round_optimal_horizon(ref, cand, thr) == exp
    assert not bad_h and not bad_c, (bad_h[:5], bad_c[:5])


@pytest.fixture
def haswell(kb):
    """Run a test with the exact cosines in OpenBLAS' Haswell ddot order (the
    device library and the oracle), restoring both afterwards."""
    prev_dev, prev_orc = kb.dot_order(), orc.set_dot_order("haswell")
    kb.set_dot_order("haswell")
    try:
        yield
    finally:
        kb.set_dot_order(prev_dev)
        orc.set_dot_order(prev_orc)


def test_divergence_golden_haswell_order(kb, haswell):
    """The reference run under numpy's OpenBLAS Haswell core (also Zen's):
    horizons and every cosine bit-exact with the device's Haswell order."""
    from paper_2605_11381_b200.divergence import round_optimal_horizon_batch
    bad_h, bad_c = [], []
    for i, (ref, cand, thr, exp, cos) in enumerate(
            golden_io.divergence_cases("divergence_haswell.npz")):
        r = torch.tensor(ref[None], device="cuda")
        c_ = torch.tensor(cand[None], device="cuda")
        H, c = round_optimal_horizon_batch(r, c_, thr, return_cos=True)
        H2 = round_optimal_horizon_batch(r, c_, thr)  # fp32 filter + exact fallback
        if int(H.item()) != exp or int(H2.item()) != exp:
            bad_h.append(i)
        if not np.array_equal(c[0, 0, :len(cos)].cpu().numpy(), cos):
            bad_c.append(i)
    assert not bad_h and not bad_c, (bad_h[:5], bad_c[:5])


@pytest.mark.parametrize("R,S,Lp,Lc,D", [(1024, 1, 50, 50, 7), (300, 1, 64, 64, 32),
                                         (130, 8, 50, 50, 7), (65, 2, 40, 40, 48),
                                         (33, 1, 10, 10, 16)])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_divergence_haswell_order_vs_oracle(kb, haswell, R, S, Lp, Lc, D, dtype):
    """Every kernel variant (D = 7 / 32 specialisations, generic D, ensembles,
    fp64 storage) in the Haswell order against the oracle in that order, with
    thresholds placed exactly on computed cosines so the exact path decides."""
    from paper_2605_11381_b200.divergence import round_optimal_horizon_batch
    rng = np.random.default_rng(R * 7 + D)
    prev = rng.normal(size=(R, Lp, D)).astype(dtype)
    noise = rng.normal(size=(R, S, Lc, D)) * (0.35 * np.arange(1, Lc + 1) / Lc)[None, None, :, None]
    cand = (prev[:, None, :Lc] + noise).astype(dtype)
    _, cos0 = orc.divergence_batch(prev, cand, 0.9, want_cos=True)
    for thr in (0.9, float(np.clip(np.nanmedian(cos0[:, :, Lc // 3]), 1e-3, 1.0))):
        exp, exp_cos = orc.divergence_batch(prev, cand, thr, want_cos=True)
        t = lambda a: torch.from_numpy(a).cuda()
        H, cos = round_optimal_horizon_batch(t(prev), t(cand), thr, return_cos=True)
        assert np.array_equal(H.cpu().numpy(), exp)
        assert np.array_equal(cos.cpu().numpy(), exp_cos, equal_nan=True)
        assert np.array_equal(round_optimal_horizon_batch(t(prev), t(cand), thr).cpu().numpy(), exp)


@pytest.mark.parametrize("R,S,Lp,Lc,D", [(1024, 1, 50, 50, 7), (300, 1, 64, 64, 32),
                                         (130, 8, 50, 50, 7), (77, 3, 20, 16, 5),
                                         (65, 2, 40, 40, 48), (33, 1, 10, 10, 16),
                                         (700, 4, 64, 64, 32), (5000, 8, 50, 50, 7)])
def test_divergence_random_vs_oracle(kb, R, S, Lp, Lc, D):
    from paper_2605_11381_b200.divergence import round_optimal_horizon_batch
    rng = np.random.default_rng(R + S + D)
    prev = rng.normal(size=(R, Lp, D)).astype(np.float32)
    noise = rng.normal(size=(R, S, Lc, D)) * (0.35 * np.arange(1, Lc + 1) / Lc)[None, None, :, None]
    cand = (prev[:, None, :Lc] if Lp >= Lc else np.pad(prev, ((0, 0), (0, Lc - Lp), (0, 0)))[:, None])
    cand = (cand + noise).astype(np.float32)
    ragged = S > 1 or Lp != Lc
    off = rng.integers(0, 4, R).astype(np.int32) if ragged else None
    lp = rng.integers(0, Lp + 1, R).astype(np.int32) if ragged else None
    lc = rng.integers(0, Lc + 1, R).astype(np.int32) if ragged else None
    exp, exp_cos = orc.divergence_batch(prev, cand, 0.9, off, lp, lc, want_cos=True)
    t = lambda a: None if a is None else torch.from_numpy(a).cuda()
    H, cos = round_optimal_horizon_batch(t(prev), t(cand), 0.9, t(off), t(lp), t(lc),
                                         return_cos=True)
    assert np.array_equal(H.cpu().numpy(), exp)
    assert np.array_equal(cos.cpu().numpy(), exp_cos, equal_nan=True)


@pytest.mark.parametrize("N", [1, 7, 50, 64])
@pytest.mark.parametrize("storage", [np.float32, np.float64])
def test_confidence_threshold_boundary(kb, N, storage):
    """f placed at, one ulp above and one ulp below opt * mean (the reference's
    own fp64 evaluation), plus zero / subnormal / huge columns: every fp32 and
    fp64 filter decision next to its margin is exercised against the oracle."""
    rng = np.random.default_rng(N * 13 + (storage == np.float32))
    R, K, t = 600, 6, 0.4
    extremes = [1e-300, 1e300] if storage == np.float64 else [1e-44, 1e36]
    scale = np.array([1.0, 1e-3, 1e3, 1e-38, *extremes, 3.0, 1e-30])[rng.integers(0, 8, R)]
    U = (rng.uniform(0.1, 1.0, (R, K, N)) * scale[:, None, None]).astype(storage)
    opt = 1.0 + t
    mean = U[:, :-1].astype(np.float64).sum(axis=1) / (K - 1)  # sequential for N >= 2
    target = (opt * mean).astype(storage)
    pick = rng.integers(0, 6, (R, N))
    up = np.nextafter(target, np.array(np.inf, storage))
    dn = np.nextafter(target, np.array(0, storage))
    last = np.select([pick == 0, pick == 1, pick == 2, pick == 3, pick == 4],
                     [target, up, dn, np.zeros_like(target), U[:, -1]], default=target * 2)
    U[:, -1] = last.astype(storage)
    U[rng.integers(0, R, 20), :-1] = 0  # zero means
    U = np.ascontiguousarray(U)
    for hmin in (1, 3):
        exp = orc.horizon_conf_batch(U, t, hmin)
        H = kb.decide_horizon_batch(kb.HorizonPolicyConfig.confidence(t, hmin),
                                    torch.from_numpy(U).cuda())
        got = H.cpu().numpy()
        bad = np.nonzero(got != exp)[0]
        assert bad.size == 0, (bad[:5], got[bad[:5]], exp[bad[:5]], scale[bad[:5]])


# --- threshold sweep (horizon.py:135-151, cli.py:109-140) -------------------

def _cfg(kb, c):
    kind, static_h, t, hmin = c
    return (kb.HorizonPolicyConfig.confidence(t, hmin) if kind
            else kb.HorizonPolicyConfig.static(static_h))


def test_sweep_golden(kb):
    """The reference's own sweep_thresholds means (48 sequences, mixed shapes,
    up to 70 configurations -> two kernel launches)."""
    for rounds, cfgs, exp in golden_io.sweep_cases():
        got = kb.sweep_thresholds([_cfg(kb, c) for c in cfgs],
                                  [kb.UpdateMagnitudes(u) for u in rounds])
        assert got == exp


@pytest.mark.parametrize("R,K,N", [(1, 2, 1), (999, 6, 50), (4099, 6, 64), (513, 3, 1),
                                   (300, 10, 7), (257, 4, 300), (700, 10, 64), (333, 3, 2),
                                   (65, 7, 66), (500, 6, 49), (90, 5, 63), (41, 6, 33),
                                   (301, 6, 128), (203, 6, 256), (150, 6, 96), (100, 6, 16),
                                   (120, 6, 32), (77, 6, 512)])
@pytest.mark.parametrize("storage", [np.float32, np.float64])
def test_sweep_vs_oracle_every_decision(kb, R, K, N, storage):
    rng = np.random.default_rng(R + K + N)
    U = (rng.uniform(0.5, 2.0, (R, 1, N)) * rng.uniform(0.3, 0.8, (R, 1, N)) **
         np.arange(K)[None, :, None] * rng.uniform(0.95, 1.05, (R, K, N)))
    tail = rng.integers(0, N + 1, R)
    for r in range(R):
        if tail[r] < N:
            U[r, -1, tail[r]:] = rng.choice([1.2, 1.8, 3.0]) * U[r, :-1, tail[r]:].mean(axis=0)
    U[rng.integers(0, R, max(1, R // 50)), :-1] = 0  # zero means
    U = np.ascontiguousarray(U.astype(storage))
    cfgs = [(1, 0, t, h) for t in (0.0, 0.1, 0.2, 0.4, 0.4, 0.8, 1.0, 1.7, 2.5) for h in (1, 5)]
    cfgs += [(0, s, 0.4, 5) for s in (1, 10, 400)]
    C = len(cfgs)
    H = torch.empty(C, R, dtype=torch.int32, device="cuda")
    sums = kb.sweep_horizon_sums([_cfg(kb, c) for c in cfgs], torch.from_numpy(U).cuda(), H=H)
    Hh = H.cpu().numpy()
    for c, (kind, s, t, h) in enumerate(cfgs):
        exp = (np.full(R, min(s, N), np.int32) if kind == 0 else orc.horizon_conf_batch(U, t, h))
        assert np.array_equal(Hh[c], exp), (c, cfgs[c])
    exp_sums = orc.sweep_sums(U, cfgs)
    assert np.array_equal(sums.cpu().numpy(), exp_sums)
    # sums-only launch (no per-decision writes) and a permuted configuration list
    perm = rng.permutation(C)
    sums2 = kb.sweep_horizon_sums([_cfg(kb, cfgs[i]) for i in perm], torch.from_numpy(U).cuda())
    assert np.array_equal(sums2.cpu().numpy(), exp_sums[perm])


@pytest.mark.parametrize("storage", [np.float32, np.float64])
def test_sweep_threshold_boundary(kb, storage):
    """Final magnitudes at / one ulp around (1 + t) * mean for several t of the
    sweep at once: the per-configuration binary search next to its margins."""
    rng = np.random.default_rng(5)
    R, K, N = 2000, 6, 50
    ts = [0.0, 0.25, 0.4, 0.5, 0.8]
    U = (rng.uniform(0.1, 1.0, (R, K, N)) *
         np.array([1.0, 1e-3, 1e3, 1e-30, 1e30])[rng.integers(0, 5, R)][:, None, None]).astype(storage)
    mean = U[:, :-1].astype(np.float64).sum(axis=1) / (K - 1)
    t_pick = np.array(ts)[rng.integers(0, len(ts), (R, N))]
    target = ((1.0 + t_pick) * mean).astype(storage)
    step = rng.integers(-1, 2, (R, N))
    last = np.where(step == 0, target, np.where(step > 0, np.nextafter(target, np.array(np.inf, storage)),
                                                np.nextafter(target, np.array(0, storage))))
    U[:, -1] = last.astype(storage)
    U = np.ascontiguousarray(U)
    cfgs = [(1, 0, t, 1) for t in ts] + [(1, 0, t, 3) for t in ts[::-1]]
    H = torch.empty(len(cfgs), R, dtype=torch.int32, device="cuda")
    kb.sweep_horizon_sums([_cfg(kb, c) for c in cfgs], torch.from_numpy(U).cuda(), H=H)
    for c, (_, _, t, h) in enumerate(cfgs):
        assert np.array_equal(H[c].cpu().numpy(), orc.horizon_conf_batch(U, t, h)), cfgs[c]


def test_sweep_validation(kb):
    U = torch.ones(4, 6, 50, dtype=torch.float64, device="cuda")
    U[2, 3, 7] = float("nan")
    with pytest.raises(ValueError, match="finite"):
        kb.sweep_horizon_sums([kb.HorizonPolicyConfig.confidence()], U)
    U[2, 3, 7] = -1.0
    with pytest.raises(ValueError, match=">= 0"):
        kb.sweep_horizon_sums([kb.HorizonPolicyConfig.static(3)], U)
    with pytest.raises(ValueError, match="no policy"):
        kb.sweep_horizon_sums([], U)


def test_nonfinite_thresholds(kb):
    """HorizonPolicyConfig accepts NaN / +inf thresholds (only t < 0 is rejected,
    horizon.py:86); f > (1 + t) * m is then never true, so every round decides N."""
    rng = np.random.default_rng(9)
    U = rng.uniform(0.0, 2.0, (300, 6, 50))
    U[:, -1, 30:] *= 5.0
    Ut = torch.from_numpy(U).cuda()
    for t in (float("nan"), float("inf")):
        cfg = kb.HorizonPolicyConfig.confidence(t, 5)
        exp = orc.horizon_conf_batch(U, t, 5)
        assert (exp == 50).all()
        assert np.array_equal(kb.decide_horizon_batch(cfg, Ut).cpu().numpy(), exp)
        cells = [cfg, kb.HorizonPolicyConfig.confidence(0.4, 5), cfg]
        sums = kb.sweep_horizon_sums(cells, Ut).cpu().numpy()
        assert sums[0] == sums[2] == 300 * 50
        assert sums[1] == orc.horizon_conf_batch(U, 0.4, 5).sum()


@pytest.mark.parametrize("storage", [torch.float32, torch.float64])
def test_zero_mean_columns_huge_thresholds(kb, storage):
    """Columns whose earlier steps are all zero: the reference's threshold is
    (1 + t) * 0.0 = 0, so any f > 0 trips for every finite t -- including
    t beyond FLT_MAX, where the fp32 filter's folded factor overflows --
    and nothing trips for t = inf / NaN ((1 + t) * 0.0 is NaN)."""
    rng = np.random.default_rng(17)
    U = rng.uniform(0.5, 2.0, (500, 6, 50))
    zc = rng.integers(0, 50, 500)
    U[np.arange(500), :-1, zc] = 0.0                       # zero mean in one column
    U[np.arange(500), -1, zc] = rng.choice([0.0, 0.25], 500)
    U = U.astype(np.float32 if storage == torch.float32 else np.float64)
    Ut = torch.from_numpy(U).cuda()
    for t in (1e39, 1e300, 3.5e38, 0.4, float("inf"), float("nan")):
        cfg = kb.HorizonPolicyConfig.confidence(t, 1)
        exp = orc.horizon_conf_batch(U.astype(np.float64), t, 1)
        assert np.array_equal(kb.decide_horizon_batch(cfg, Ut).cpu().numpy(), exp), t
        if t == 1e39:  # the zero-mean trips decide these horizons
            assert (exp < 50).sum() > 100
    cells = [kb.HorizonPolicyConfig.confidence(t, h) for t in (1e39, 0.4, float("inf"), 3.5e38)
             for h in (1, 5)]
    sums = kb.sweep_horizon_sums(cells, Ut).cpu().numpy()
    exp = orc.sweep_sums(U.astype(np.float64), [(1, 0, c.threshold, c.min_horizon) for c in cells])
    assert np.array_equal(sums, exp)


@pytest.mark.parametrize("storage", [torch.float32, torch.float64])
def test_segmented_validation_and_negative_zero(kb, storage):
    """The segmented sweep / decide kernels' validation: NaN, +inf and negative
    magnitudes in any lane's window raise the reference's ValueError; -0.0 is a
    valid magnitude (horizon.py:47-50: isfinite and not < 0) and decides like
    +0.0 through the exact path."""
    rng = np.random.default_rng(23)
    base = rng.uniform(0.2, 1.5, (257, 6, 50))
    base[:, -1, 35:] *= 2.5
    for bad, msg in ((float("nan"), "finite"), (float("inf"), "finite"), (-1e-3, ">= 0")):
        for col in (0, 13, 29, 49):  # the windows of different lanes
            U = torch.from_numpy(base.copy()).to(storage).cuda()
            U[101, 2, col] = bad
            with pytest.raises(ValueError, match=msg):
                kb.sweep_horizon_sums([kb.HorizonPolicyConfig.confidence(0.4, 5)], U)
            with pytest.raises(ValueError, match=msg):
                kb.decide_horizon_batch(kb.HorizonPolicyConfig.confidence(0.4, 5), U)
    U = base.copy()
    U[5, :, 7] = -0.0
    U[9, 1, 20] = -0.0
    Ut = torch.from_numpy(U).to(storage).cuda()
    Un = Ut.cpu().numpy()
    for t, h in ((0.4, 5), (0.0, 1), (1.3, 3)):
        cfg = kb.HorizonPolicyConfig.confidence(t, h)
        exp = orc.horizon_conf_batch(Un, t, h)
        assert np.array_equal(kb.decide_horizon_batch(cfg, Ut).cpu().numpy(), exp)
        assert int(kb.sweep_horizon_sums([cfg], Ut).cpu()[0]) == int(exp.sum())


def test_dynamic_tile_counters_across_launches(kb):
    """Launches captured into CUDA graphs claim their tail tiles from a counter
    pair of their own (kr_plan.cuh stream_counters) that each replay's last CTA
    resets; eager launches keep the static schedule.  Three graphs replayed
    interleaved, 20 times each, on two streams, and 50 eager launches must all
    decide exactly what the oracle decides (a counter left non-zero, or shared
    by two graphs, would skip tiles)."""
    from paper_2605_11381_b200 import synthetic
    from paper_2605_11381_b200.divergence import round_optimal_horizon_batch
    R = 1 << 16  # many tiles per CTA: the dynamic tail is in use
    prev, cand, off = synthetic.chunks(R, seed=5)
    exp = orc.divergence_batch(prev.cpu().numpy(), cand.cpu().numpy(), 0.9,
                               off.cpu().numpy(), None, None)
    outs = [torch.empty(R, dtype=torch.int32, device="cuda") for _ in range(4)]
    for _ in range(50):
        round_optimal_horizon_batch(prev, cand, 0.9, off, out=outs[3])
    graphs = []
    for j in range(3):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            round_optimal_horizon_batch(prev, cand, 0.9, off, out=outs[j])
        graphs.append(g)
    side = torch.cuda.Stream()
    for _ in range(20):
        for j, g in enumerate(graphs):
            outs[j].fill_(-1)
            if j == 1:  # one graph on a second stream, overlapping the others
                side.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(side):
                    g.replay()
            else:
                g.replay()
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        for o in outs:
            assert np.array_equal(o.cpu().numpy(), exp)
