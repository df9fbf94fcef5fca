"""The reference test suite's property tests and hand-computed fixtures
(pkg/tests/test_horizon.py, test_core.py, test_waiting.py), re-run against the
drop-in package on the GPU.  Hypothesis strategies mirror the reference's."""

from __future__ import annotations

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st
from hypothesis.extra import numpy as npst

pytestmark = pytest.mark.gpu

import paper_2605_11381_b200 as kb  # noqa: E402

magnitude_arrays = npst.arrays(
    dtype=np.float64,
    shape=st.tuples(st.integers(2, 6), st.integers(1, 20)),
    elements=st.floats(0.0, 1e6, allow_nan=False, allow_infinity=False, width=32),
)
FAST = settings(max_examples=60, deadline=None)


@given(u=magnitude_arrays, t1=st.floats(0, 3), t2=st.floats(0, 3), hmin=st.integers(1, 5))
@FAST
def test_monotone_in_threshold(u, t1, t2, hmin):           # test_horizon.py:126-133
    mags = kb.UpdateMagnitudes(u)
    lo, hi = sorted((t1, t2))
    assert (kb.decide_horizon(kb.HorizonPolicyConfig.confidence(lo, hmin), mags)
            <= kb.decide_horizon(kb.HorizonPolicyConfig.confidence(hi, hmin), mags))


@given(u=magnitude_arrays, t=st.floats(0, 3), hmin=st.integers(1, 5))
@FAST
def test_bounds(u, t, hmin):                                 # test_horizon.py:136-141
    mags = kb.UpdateMagnitudes(u)
    h = kb.decide_horizon(kb.HorizonPolicyConfig.confidence(t, hmin), mags)
    assert min(hmin, mags.chunk_size) <= h <= mags.chunk_size


@given(u=magnitude_arrays, t=st.floats(0, 3), scale_exp=st.integers(-20, 20))
@FAST
def test_scale_invariance(u, t, scale_exp):                  # test_horizon.py:144-156
    cfg = kb.HorizonPolicyConfig.confidence(t, 1)
    assert (kb.decide_horizon(cfg, kb.UpdateMagnitudes(u))
            == kb.decide_horizon(cfg, kb.UpdateMagnitudes(u * (2.0 ** scale_exp))))


@given(u=magnitude_arrays, t=st.floats(0, 3), seed=st.integers(0, 2**31))
@FAST
def test_prefix_rule(u, t, seed):                            # test_horizon.py:159-174
    mags = kb.UpdateMagnitudes(u)
    cfg = kb.HorizonPolicyConfig.confidence(t, 1)
    h = kb.decide_horizon(cfg, mags)
    if h >= mags.chunk_size - 1:
        return
    perm = np.random.default_rng(seed).permutation(np.arange(h + 1, mags.chunk_size))
    shuffled = u.copy()
    shuffled[:, h + 1:] = u[:, perm]
    assert kb.decide_horizon(cfg, kb.UpdateMagnitudes(shuffled)) == h


@given(count=st.integers(0, 10_000), hz=st.sampled_from([1, 3, 7.5, 10, 30, 50, 100]))
@FAST
def test_time_closed_over_integers(count, hz):               # test_core.py:70-74
    out = kb.us_from_actions(count, hz)
    assert isinstance(out, int) and out >= 0


@given(a=st.integers(0, 500), b=st.integers(0, 500), hz=st.sampled_from([3, 30, 50]))
@FAST
def test_us_from_actions_monotone(a, b, hz):                 # test_core.py:77-80
    lo, hi = sorted((a, b))
    assert kb.us_from_actions(lo, hz) <= kb.us_from_actions(hi, hz)


def test_horizon_reference_goldens():                        # test_horizon.py:17-114
    u = np.ones((4, 6)); u[-1, 4] = 1.5
    fig = kb.UpdateMagnitudes(u)
    conf = kb.HorizonPolicyConfig.confidence
    assert kb.decide_horizon(conf(threshold=0.4, min_horizon=1), fig) == 4
    u = np.ones((3, 8)); u[-1, :] = 0.0
    assert kb.decide_horizon(conf(threshold=0.0, min_horizon=1), kb.UpdateMagnitudes(u)) == 8
    u = np.array([[1, 1, 1], [1, 1, 1], [1.3, 1.5, 1.1]], dtype=float)
    assert kb.decide_horizon(conf(threshold=0.4, min_horizon=1), kb.UpdateMagnitudes(u)) == 1
    assert kb.decide_horizon(conf(threshold=0.6, min_horizon=1), kb.UpdateMagnitudes(u)) == 3
    u = np.ones((3, 10)); u[-1, 0] = 10.0
    assert kb.decide_horizon(conf(threshold=0.4, min_horizon=4), kb.UpdateMagnitudes(u)) == 4
    assert kb.decide_horizon(conf(threshold=0.0, min_horizon=1), kb.UpdateMagnitudes(np.zeros((3, 4)))) == 4
    u = np.zeros((3, 4)); u[-1, 1] = 0.5
    assert kb.decide_horizon(conf(threshold=10.0, min_horizon=1), kb.UpdateMagnitudes(u)) == 1
    with pytest.raises(ValueError):
        kb.UpdateMagnitudes(np.ones((1, 4)))
    with pytest.raises(ValueError):
        conf(threshold=-0.1)
    assert kb.decide_horizon(kb.HorizonPolicyConfig.static(80), kb.UpdateMagnitudes(np.ones((2, 50)))) == 50
    assert kb.decide_horizon(kb.HorizonPolicyConfig.static(7), fig) == 6
    assert kb.sweep_thresholds([kb.HorizonPolicyConfig.static(20)], [kb.UpdateMagnitudes(np.ones((2, 30)))]) == [20.0]
    u4 = np.ones((3, 10)); u4[-1, 4] = 5.0
    u6 = np.ones((3, 10)); u6[-1, 6] = 5.0
    assert kb.sweep_thresholds([conf(threshold=0.4, min_horizon=1)],
                               [kb.UpdateMagnitudes(u4), kb.UpdateMagnitudes(u6)]) == [5.0]
    assert kb.sweep_thresholds([conf(threshold=0.4, min_horizon=1)], [fig] * 10) == [4.0]
    with pytest.raises(ValueError):
        kb.sweep_thresholds([], [fig])
    with pytest.raises(ValueError):
        kb.sweep_thresholds([kb.HorizonPolicyConfig.static(1)], [])


def test_divergence_reference_goldens():                     # test_workload.py:211-239
    ref = [[1.0, 0.0], [0.0, 1.0], [1.0, 1.0]]
    assert kb.round_optimal_horizon(ref, ref, 0.9) == 3
    rng = np.random.default_rng(0)
    r = rng.normal(size=(20, 3))
    c = r.copy()
    for i in range(12, 20):
        v = r[i]
        c[i] = np.array([-v[1], v[0], 0.0])
    assert kb.round_optimal_horizon(r, c, 0.9) == 12
    z = [[0.0, 0.0]]
    assert kb.round_optimal_horizon(z, z, 0.9) == 1
    assert kb.round_optimal_horizon([[1.0, 0.0]], z, 0.9) == 0
    for bad in (0.0, 1.5):
        with pytest.raises(ValueError):
            kb.round_optimal_horizon([[1.0]], [[1.0]], bad)
    with pytest.raises(ValueError):
        kb.round_optimal_horizon([[1.0, 2.0]], [[1.0]], 0.9)


MS = 1000
I = kb.Interval
# test_waiting.py:20-73, all 22 hand-computed (G_j, E_j, G_next, E_next, wait) rows
WAIT_FIXTURES = [
    (I(1_600_000, 2_000_000), I(2_000_000, 2_300_000), I(2_500_000, 2_900_000), I(2_900_000, 3_200_000), 500 * MS),
    (I(0, 400_000), I(400_000, 500_000), I(400_000, 800_000), I(800_000, 900_000), 0),
    (I(0, 300_000), I(300_000, 500_000), I(310_000, 610_000), I(700_000, 900_000), 10 * MS),
    (I(0, 500_000), I(500_000, 600_000), I(1_500_000, 2_000_000), I(2_000_000, 2_100_000), 1_000 * MS),
    (I(100_000, 200_000), I(200_000, 250_000), I(200_000, 300_000), I(300_000, 350_000), 0),
    (I(0, 600_000), I(600_000, 700_000), I(550_000, 1_150_000), I(1_150_000, 1_250_000), 0),
    (I(0, 1_000_000), I(1_000_000, 1_000_000), I(1_250_000, 2_250_000), I(2_250_000, 2_250_000), 250 * MS),
    (I(0, 300_000), I(300_000, 600_000), I(450_000, 750_000), I(750_000, 1_050_000), 150 * MS),
    (I(0, 300_000), I(300_000, 600_000), I(300_000, 600_000), I(600_000, 900_000), 0),
    (I(0, 200_000), I(200_000, 400_000), I(200_000, 400_000), I(999_000, 1_199_000), 0),
    (I(4_000_000, 4_200_000), I(4_200_000, 5_000_000), I(4_500_000, 4_700_000), I(5_000_000, 5_800_000), 0),
    (I(0, 200_000), I(200_000, 1_100_000), I(500_000, 700_000), I(1_100_000, 2_000_000), 0),
    (I(0, 200_000), I(200_000, 1_100_000), I(1_100_000, 1_300_000), I(1_300_000, 2_200_000), 200 * MS),
    (I(0, 100_000), I(100_000, 800_000), I(900_000, 1_000_000), I(1_000_000, 1_700_000), 200 * MS),
    (I(0, 300_000), I(300_000, 1_000_000), I(600_000, 900_000), I(1_033_333, 1_733_333), 33_333),
    (I(0, 300_000), I(300_000, 1_200_000), I(600_000, 900_000), I(1_200_000, 2_100_000), 0),
    (I(0, 100_000), I(100_000, 700_000), I(200_000, 300_000), I(650_000, 1_250_000), 0),
    (I(0, 50_000), I(50_000, 60_000), I(75_000, 125_000), I(125_000, 135_000), 25 * MS),
    (I(0, 10_000), I(10_000, 500_000), I(505_000, 515_000), I(515_000, 1_005_000), 15 * MS),
    (I(0, 1), I(1, 2), I(1, 2), I(2, 3), 0),
    (I(0, 2), I(2, 3), I(5, 7), I(7, 8), 3),
    (I(0, 1), I(1, 4), I(2, 3), I(9, 12), 5),
]


@pytest.mark.parametrize("g1, e1, g2, e2, expected", WAIT_FIXTURES)
def test_round_wait_fixture(g1, e1, g2, e2, expected):
    assert kb.round_wait(g1, e1, g2, e2) == expected


def test_round_wait_rejects():                                # test_waiting.py:81-94
    with pytest.raises(ValueError):
        kb.round_wait(I(1_000, 2_000), I(2_000, 3_000), I(0, 500), I(500, 600))
    with pytest.raises(ValueError):
        kb.round_wait(I(1_000, 2_000), I(1_500, 3_000), I(3_000, 4_000), I(4_000, 5_000))


def test_core_reference_goldens():                            # test_core.py:31-67
    req = lambda at, rem: kb.PendingRequest("t", 1, at, at, kb.LastExecInfo(0, rem), 0)
    assert kb.exec_end_from_piggyback(req(1_000_000, 10), 30) == 1_333_333
    assert kb.exec_end_from_piggyback(req(5_000_000, 0), 30) == 5_000_000
    assert kb.exec_end_from_piggyback(req(0, 30), 30) == 1_000_000
    assert kb.exec_duration(10, 30) == 333_333
    assert kb.exec_duration(50, 30) == 1_666_667
    assert kb.exec_duration(0, 30) == 0 and kb.exec_duration(0, 7.5) == 0
    for bad in ((-1, 30), (1, 0)):
        with pytest.raises(ValueError):
            kb.exec_duration(*bad)
    assert [kb.us_from_actions(1, 2), kb.us_from_actions(1, 3), kb.us_from_actions(2, 3)] == \
        [500_000, 333_333, 666_667]
