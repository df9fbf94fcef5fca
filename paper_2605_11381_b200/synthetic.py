"""Seeded synthetic decision-round inputs (SURVEY.md §8(d) recipes).

Used by bench.py, __graft_entry__.smoke() and the tests; not part of the
decision path itself.  Fleet histories follow the survey's pending-state
generator (1-5 recorded rounds, generation 100-400 ms, execution
exec_duration(U[10,50], 30 Hz), optional in-flight successor generation);
action chunks follow config 2/5: prev ~ N(0, 1) [R, Lp, D], the new chunk
tracks the unexecuted overlap prev[r, off_r:] with noise growing along the
chunk, so the cosine prefix cut lands mid-chunk.
"""

from __future__ import annotations

import numpy as np
import torch

NOW = 100_000_000
HZ = 30


def exec_us(h: np.ndarray, hz: int = HZ) -> np.ndarray:
    """us_from_actions for integer hz, vectorised (core.py:31-42)."""
    return (2 * h.astype(np.int64) * 1_000_000 + hz) // (2 * hz)


def fleet_soa(R: int, seed: int, now: int = NOW, max_rounds: int = 5, p_inflight: float = 0.4,
              rank_offset: int = 0) -> dict:
    """Host structure-of-arrays of R pending robots (fleet.py layout)."""
    rng = np.random.default_rng(seed)
    n_exec = rng.integers(0, max_rounds + 1, R).astype(np.int32)
    inflight = (rng.random(R) < p_inflight).astype(np.int32)
    n_gen = n_exec + inflight
    t_start = now - rng.integers(5_000_000, 20_000_000, R)
    M = max_rounds + 1
    gs = np.zeros((R, M), np.int64)
    ge = np.zeros((R, M), np.int64)
    es = np.zeros((R, M), np.int64)
    ee = np.zeros((R, M), np.int64)
    cur = t_start.copy()
    for j in range(M):
        gs[:, j] = cur + rng.integers(0, 200_000, R)
        ge[:, j] = gs[:, j] + rng.integers(100_000, 400_000, R)
        es[:, j] = ge[:, j] + rng.integers(0, 50_000, R)
        ee[:, j] = es[:, j] + exec_us(rng.integers(10, 51, R))
        cur = ee[:, j] - rng.integers(0, 300_000, R)
    nslots = np.maximum(n_exec, n_gen)
    j = np.arange(M)[None, :]
    mask = j < nslots[:, None]
    ge = np.where(j < n_exec[:, None], ge, 0)   # in-flight successor: start only
    es = np.where(j < n_exec[:, None], es, 0)
    ee = np.where(j < n_exec[:, None], ee, 0)
    slots = np.stack([gs[mask], ge[mask], es[mask], ee[mask]], axis=1).astype(np.int64)
    if slots.shape[0] == 0:
        slots = np.zeros((1, 4), np.int64)
    hist_off = np.concatenate([[0], np.cumsum(nslots)[:-1]]).astype(np.int64)
    issued = now - rng.integers(0, 1_000_000, R)
    return {
        "n": R,
        "t_start": t_start.astype(np.int64),
        "issued_at": issued.astype(np.int64),
        "obs_captured_at": (issued - rng.integers(0, 300_000, R)).astype(np.int64),
        "accum_gen": rng.integers(0, 5_000_000, R).astype(np.int64),
        "remaining": rng.integers(0, 40, R).astype(np.int32),
        "lexrank": (rank_offset + np.arange(R)).astype(np.int32),
        "skipped": rng.integers(0, 13, R).astype(np.int32),
        "hist_off": hist_off,
        "n_exec": n_exec,
        "n_gen": n_gen.astype(np.int32),
        "slots": slots,
    }


def chunks(R: int, seed: int, Lp: int = 50, Lc: int = 50, D: int = 7, S: int = 1,
           max_offset: int = 10, device="cuda", dtype=torch.float32):
    """(prev [R,Lp,D], cand [R,S,Lc,D], offset [R] int32) generated on `device`."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    prev = torch.randn((R, Lp, D), generator=g, device=device, dtype=torch.float32)
    off = torch.randint(0, max_offset + 1, (R,), generator=g, device=device, dtype=torch.int32)
    idx = (off[:, None].long() + torch.arange(Lc, device=device)[None, :]).clamp_(max=Lp - 1)
    base = torch.gather(prev, 1, idx[:, :, None].expand(R, Lc, D))
    sigma = 0.35 * torch.arange(1, Lc + 1, device=device, dtype=torch.float32) / Lc
    cand = base[:, None] + torch.randn((R, S, Lc, D), generator=g, device=device,
                                       dtype=torch.float32) * sigma[None, None, :, None]
    return prev.to(dtype), cand.to(dtype), off


def magnitudes(R: int, seed: int, K: int = 6, N: int = 50, device="cuda",
               dtype=torch.float32) -> torch.Tensor:
    """U[R, K, N]: the reference's geometric-decay magnitude model with an
    uncertain tail bumped to 1.8x its earlier mean (workload.py:341-359)."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    rho = torch.rand((R, 1, N), generator=g, device=device, dtype=torch.float64) * 0.3 + 0.4
    u0 = torch.rand((R, 1, N), generator=g, device=device, dtype=torch.float64) * 1.5 + 0.5
    k = torch.arange(K, device=device, dtype=torch.float64)[None, :, None]
    noise = 1.0 + (torch.rand((R, K, N), generator=g, device=device, dtype=torch.float64) - 0.5) * 0.1
    U = u0 * rho ** k * noise
    frac = torch.rand((R,), generator=g, device=device, dtype=torch.float64) * 0.4
    n_unc = torch.round(frac * N).long()
    col = torch.arange(N, device=device)[None, :]
    tail = col >= (N - n_unc)[:, None]
    U[:, -1, :] = torch.where(tail, 1.8 * U[:, :-1, :].mean(dim=1), U[:, -1, :])
    return U.to(dtype)
