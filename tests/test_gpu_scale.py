"""Parity at the BASELINE sizes: the exact benchmarked rounds vs the CPU oracle.

The other GPU tests pin every function on small and medium inputs; these run
the configurations bench.py measures, at their full sizes and through the same
code path (captured CUDA graphs, concurrent split layout, the same reserved-SM
counts), and compare every output with the oracle (oracle/kairos_oracle.c,
which is itself pinned to the unmodified reference by tests/golden):

  (i)   configs[4] per-GPU share: 2^20 robots, 50x7 fp32, offsets U[0,10],
        thr 0.9, k = 8192, split layout / 10 reserved SMs, several evolving
        rounds (new chunks every round, skip counters carried over);
  (ii)  configs[2]: 16,384 robots, 8k arms 64x7 + 8k humanoids 64x32, k = 1024;
  (iii) configs[3]: 65,536 robots x 8-sample ensembles, k = 8192;
  (iv)  the 2^20 confidence round, fp32 and fp64 storage;
  (v)   a 2^20 divergence pass whose cosines sit within the fp32 filter's
        margin of the threshold, so millions of decisions take the exact fp64
        fallback (fp32 and fp64 storage).

Reference functions: workload.py:471-496 (round_optimal_horizon),
horizon.py:108-132 (decide_horizon), scheduler.py:254-276 (plan)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import oracle as orc

pytestmark = pytest.mark.gpu

NOW = 100_000_000


def _sched(base):
    from paper_2605_11381_b200 import fleet as fl
    return fl.sched_struct("kairos", 10, 5, 150_000, 166_667, NOW, 30, base)


def _plan(soa, k):
    return orc.plan_soa(soa, "kairos", 10, 5, 150_000, 166_667, NOW, 30, k)


def _check_plan(out, fleet, res, k, tag):
    assert np.array_equal(out.need_time.cpu().numpy(), res["need_time"]), tag
    assert np.array_equal(out.admitted.cpu().numpy(), res["admitted"]), tag
    assert np.array_equal(out.refetch.cpu().numpy(), res["refetch"]), tag
    assert np.array_equal(fleet.t["skipped"].cpu().numpy(), res["skipped_out"]), tag
    assert np.array_equal(out.edge_idx[:k].cpu().numpy(), res["order"][:k]), tag


def test_bench_round_2p20_evolving():
    """(i) bench.py's exact round: same seeds, issued base, budget, layout and
    reserved SMs; three rounds with fresh chunks copied into the captured
    buffers and the skip counters evolving as in a trace replay."""
    from paper_2605_11381_b200 import fleet as fl, rounds, synthetic
    R, k = 1 << 20, 8192
    soa = synthetic.fleet_soa(R, seed=1000, rank_offset=0)
    fleet = fl.DeviceFleet.from_host(soa)
    prev, cand, off = synthetic.chunks(R, seed=2000)
    rnd = rounds.DecisionRound(R, k, _sched(NOW - (1 << 39)))
    inputs = rounds.DivergenceInputs(prev, cand, 0.9, offset=off)
    rnd.capture(fleet, inputs, reserve_sms=2, layout="split")
    torch.cuda.synchronize()
    fleet.t["skipped"].copy_(torch.from_numpy(soa["skipped"]).cuda())  # undo the warm-up round
    for r in range(3):
        p2, c2, o2 = synthetic.chunks(R, seed=2001 + r)
        prev.copy_(p2), cand.copy_(c2), off.copy_(o2)
        out = rnd.replay()
        torch.cuda.synchronize()
        H = orc.divergence_batch(p2.cpu().numpy(), c2.cpu().numpy(), 0.9, o2.cpu().numpy())
        assert np.array_equal(out.horizon.cpu().numpy(), H), r
        res = _plan(soa, k)
        _check_plan(out, fleet, res, k, r)
        soa["skipped"] = res["skipped_out"]
    # the skip counters did evolve: aged robots reached the admission set
    assert int(res["skipped_out"].max()) >= 14


def test_config2_mixed_16k():
    """(ii) configs[2]: two homogeneous chunk tensors, captured split/8."""
    from paper_2605_11381_b200 import fleet as fl, rounds, synthetic
    R, k = 16384, 1024
    soa = synthetic.fleet_soa(R, seed=13)
    pa, ca, oa = synthetic.chunks(R // 2, seed=14, Lp=64, Lc=64, D=7)
    ph, ch, oh = synthetic.chunks(R // 2, seed=15, Lp=64, Lc=64, D=32)
    inp = rounds.MixedInputs([(0, rounds.DivergenceInputs(pa, ca, 0.9, offset=oa)),
                              (R // 2, rounds.DivergenceInputs(ph, ch, 0.9, offset=oh))])
    fleet = fl.DeviceFleet.from_host(soa)
    rnd = rounds.DecisionRound(R, k, _sched(int(soa["issued_at"].min())))
    rnd.capture(fleet, inp, reserve_sms=8, layout="split")
    fleet.t["skipped"].copy_(torch.from_numpy(soa["skipped"]).cuda())
    out = rnd.replay()
    torch.cuda.synchronize()
    H = np.concatenate([
        orc.divergence_batch(pa.cpu().numpy(), ca.cpu().numpy(), 0.9, oa.cpu().numpy()),
        orc.divergence_batch(ph.cpu().numpy(), ch.cpu().numpy(), 0.9, oh.cpu().numpy())])
    assert np.array_equal(out.horizon.cpu().numpy(), H)
    _check_plan(out, fleet, _plan(soa, k), k, "configs[2]")


def test_config3_ensembles_64k():
    """(iii) configs[3]: 65,536 robots x S=8 samples, captured split/1 (bench.py)."""
    from paper_2605_11381_b200 import fleet as fl, rounds, synthetic
    R, k = 65536, 8192
    soa = synthetic.fleet_soa(R, seed=16)
    prev, cand, off = synthetic.chunks(R, seed=17, S=8)
    fleet = fl.DeviceFleet.from_host(soa)
    rnd = rounds.DecisionRound(R, k, _sched(int(soa["issued_at"].min())))
    rnd.capture(fleet, rounds.DivergenceInputs(prev, cand, 0.9, offset=off), reserve_sms=1,
                layout="split")
    fleet.t["skipped"].copy_(torch.from_numpy(soa["skipped"]).cuda())
    out = rnd.replay()
    torch.cuda.synchronize()
    H = orc.divergence_batch(prev.cpu().numpy(), cand.cpu().numpy(), 0.9, off.cpu().numpy())
    assert np.array_equal(out.horizon.cpu().numpy(), H)
    _check_plan(out, fleet, _plan(soa, k), k, "configs[3]")


@pytest.mark.parametrize("storage", [torch.float32, torch.float64])
def test_confidence_round_2p20(storage):
    """(iv) the headline fleet under the confidence policy, as bench.py's
    other_configs runs it (split; 8 reserved SMs for fp32, 16 for fp64)."""
    from paper_2605_11381_b200 import HorizonPolicyConfig, fleet as fl, rounds, synthetic
    R, k = 1 << 20, 8192
    soa = synthetic.fleet_soa(R, seed=18)
    U = synthetic.magnitudes(R, seed=19, dtype=storage)
    fleet = fl.DeviceFleet.from_host(soa)
    rnd = rounds.DecisionRound(R, k, _sched(int(soa["issued_at"].min())))
    rnd.capture(fleet, rounds.ConfidenceInputs(U, HorizonPolicyConfig.confidence(0.4, 5)),
                reserve_sms=8 if storage == torch.float32 else 16, layout="split")
    fleet.t["skipped"].copy_(torch.from_numpy(soa["skipped"]).cuda())
    out = rnd.replay()
    torch.cuda.synchronize()
    H = orc.horizon_conf_batch(U.cpu().numpy(), 0.4, 5)
    assert np.array_equal(out.horizon.cpu().numpy(), H)
    _check_plan(out, fleet, _plan(soa, k), k, "confidence")


def _near_threshold_chunks(R, thr, frac, seed, dtype):
    """prev ~ N(0,1) [R,50,7]; cand tracks prev[off:] with noise, except that a
    fraction `frac` of the actions is rebuilt as thr * u + sqrt(1-thr^2) * v
    (u = the reference row's direction, v a unit vector orthogonal to it), so
    its cosine equals thr up to storage rounding: far inside the fp32
    filter's margin, i.e. decided by the exact fp64 path, on both sides of
    the threshold."""
    from paper_2605_11381_b200 import synthetic
    prev, cand, off = synthetic.chunks(R, seed=seed, device="cuda")
    g = torch.Generator(device="cuda")
    g.manual_seed(seed + 1)
    Lc = cand.shape[2]
    idx = (off[:, None].long() + torch.arange(Lc, device="cuda")[None, :]).clamp_(max=49)
    ref = torch.gather(prev.double(), 1, idx[:, :, None].expand(R, Lc, 7))
    u = ref / ref.norm(dim=-1, keepdim=True)
    w = torch.randn(ref.shape, generator=g, device="cuda", dtype=torch.float64)
    v = w - (w * u).sum(-1, keepdim=True) * u
    v = v / v.norm(dim=-1, keepdim=True)
    scale = torch.rand((R, Lc, 1), generator=g, device="cuda", dtype=torch.float64) * 2 + 0.1
    near = (thr * u + (1 - thr * thr) ** 0.5 * v) * scale
    pick = torch.rand((R, Lc, 1), generator=g, device="cuda") < frac
    c = torch.where(pick, near, cand[:, 0].double())
    return prev.to(dtype), c.to(dtype).unsqueeze(1).contiguous(), off


@pytest.mark.parametrize("storage", [torch.float32, torch.float64])
def test_divergence_fp64_fallback_at_scale(storage):
    """(v) 2^20 robots with ~8% of the actions' cosines at the threshold up to
    rounding: the fp32 pre-decision must hand every one of them to the exact
    fp64 OpenBLAS-order cosine, and the horizons stay bit-exact."""
    from paper_2605_11381_b200 import fleet as fl, rounds, synthetic
    R, thr = 1 << 20, 0.9
    prev, cand, off = _near_threshold_chunks(R, thr, 0.08, seed=51, dtype=storage)
    H = orc.divergence_batch(prev.cpu().numpy(), cand.cpu().numpy(), thr, off.cpu().numpy())
    soa = synthetic.fleet_soa(R, seed=52)
    fleet = fl.DeviceFleet.from_host(soa)
    rnd = rounds.DecisionRound(R, 8192, _sched(int(soa["issued_at"].min())))
    inputs = rounds.DivergenceInputs(prev, cand, thr, offset=off)
    rnd.capture(fleet, inputs, reserve_sms=10, layout="split")
    out = rnd.replay()
    torch.cuda.synchronize()
    got = out.horizon.cpu().numpy()
    assert np.array_equal(got, H), int((got != H).sum())
    # the construction does cut prefixes at the near-threshold actions: a large
    # share of the horizons differ from the plain noisy chunk's
    base = orc.divergence_batch(prev.cpu().numpy(), synthetic.chunks(R, seed=51)[1].to(storage)
                                .cpu().numpy(), thr, off.cpu().numpy())
    assert (H != base).mean() > 0.3
