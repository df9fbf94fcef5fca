"""Synthetic traces generated on the device (reference workload.py:296-456:
`SyntheticSpec`, `_synth_round_magnitudes`, `generation_slack_actions`,
`synthesize_trace`, `synthesize_family`).

Same names, arguments, validation and construction as the reference; the
randomness is the device's counter-based Philox stream keyed by (seed, task
index) instead of numpy's Generator (bit parity with numpy's RNG is not a
goal), so the traces follow the reference's distributions, not its draws.
Per round: K x N magnitudes u0 * rho^k * noise with the uncertain tail's final
row set to bump * mean(earlier rows) (kr_synth_magnitudes), the policy's
horizon decided by the horizon kernels (bit-exact `decide_horizon`), then the
trigger placement / action-budget loop (kr_synth_close).  Families are
generated a few rounds per launch for every task still below its budget;
`synthesize_family_columns` keeps everything in device columns.
"""

from __future__ import annotations

import ctypes
import json
import math
from dataclasses import dataclass
from fractions import Fraction
from pathlib import Path
from typing import Optional

import torch

from . import _lib
from . import device as dev
from .core import Duration, exec_duration
from .horizon import HorizonPolicyConfig, UpdateMagnitudes, decide_horizon_batch
from .traces import RoundRecord, TaskTrace, store_traces


@dataclass(frozen=True)
class SyntheticSpec:
    """Knobs of the synthetic workload (workload.py:296-338)."""

    chunk_size: int = 50
    diffusion_steps: int = 6
    control_hz: float = 30.0
    action_budget: int = 200
    uncertain_fraction: float = 0.2
    decay: float = 0.55
    noise_scale: float = 0.05
    bump_factor: float = 1.8
    obs_payload_bytes: int = 300_000
    action_payload_bytes: int = 4_000
    success_rate: float = 1.0

    def __post_init__(self) -> None:
        if self.chunk_size < 1:
            raise ValueError("chunk_size must be >= 1")
        if self.diffusion_steps < 2:
            raise ValueError("diffusion_steps must be >= 2")
        if self.control_hz <= 0:
            raise ValueError("control_hz must be > 0")
        if self.action_budget < 1:
            raise ValueError("action_budget must be >= 1")
        if not 0.0 <= self.uncertain_fraction <= 1.0:
            raise ValueError("uncertain_fraction must be in [0, 1]")
        if not 0.0 < self.decay < 1.0:
            raise ValueError("decay must be in (0, 1)")
        if not 0.0 <= self.noise_scale < 0.5:
            raise ValueError("noise_scale must be in [0, 0.5)")
        if self.bump_factor <= 1.0:
            raise ValueError("bump_factor must be > 1")
        if not 0.0 <= self.success_rate <= 1.0:
            raise ValueError("success_rate must be in [0, 1]")

    @classmethod
    def from_dict(cls, data: dict) -> "SyntheticSpec":
        known = set(cls.__dataclass_fields__)
        unknown = set(data) - known
        if unknown:
            raise ValueError(f"unknown synthetic-spec fields: {sorted(unknown)}")
        return cls(**data)

    def c_struct(self) -> _lib.KrSynthSpec:
        return _lib.KrSynthSpec(self.chunk_size, self.diffusion_steps, self.decay, self.noise_scale,
                                self.bump_factor, self.uncertain_fraction)


def generation_slack_actions(gen_latency: Duration, control_hz: float) -> int:
    """Actions the robot executes while one generation is in flight (ceil)
    (workload.py:366-368)."""
    return math.ceil(Fraction(gen_latency) * Fraction(control_hz) / 1_000_000)


def _check_fits(spec: SyntheticSpec, policy: HorizonPolicyConfig, gen_latency: Duration) -> None:
    floor_duration = exec_duration(min(policy.floor, spec.chunk_size), spec.control_hz)
    if gen_latency >= floor_duration:  # workload.py:386-391
        raise ValueError(
            f"gen_latency {gen_latency}us does not fit inside the smallest "
            f"retained prefix ({floor_duration}us); the task could never keep up")


@dataclass
class SynthColumns:
    """A synthetic trace family in device columns (rounds sorted by task, then
    round id)."""

    task_ids: list
    spec: SyntheticSpec
    round_off: torch.Tensor        # [T+1] int64
    round_task: torch.Tensor       # [R] int64 task index
    round_id: torch.Tensor         # [R] int32
    trigger_action_index: torch.Tensor  # [R] int32
    horizon: torch.Tensor          # [R] int32
    U: torch.Tensor                # [R, K, N] float64
    success: torch.Tensor          # [T] bool
    traj_row_off: Optional[torch.Tensor] = None  # [R+1] int64
    traj: Optional[torch.Tensor] = None          # [rows, dim] float64

    @property
    def n_traces(self) -> int:
        return len(self.task_ids)

    @property
    def n_rounds(self) -> int:
        return int(self.round_id.numel())

    def to_traces(self) -> list:
        """The family as the reference's TaskTrace objects (host)."""
        s = self.spec
        off = self.round_off.cpu().numpy()
        rid = self.round_id.cpu().numpy()
        trig = self.trigger_action_index.cpu().numpy()
        hor = self.horizon.cpu().numpy()
        U = self.U.cpu().numpy()
        succ = self.success.cpu().numpy()
        if self.traj is not None:
            toff = self.traj_row_off.cpu().numpy()
            traj = self.traj.cpu().numpy()
        out = []
        for t, tid in enumerate(self.task_ids):
            rounds = []
            for r in range(off[t], off[t + 1]):
                tr = None
                if self.traj is not None:
                    tr = tuple(tuple(float(v) for v in row) for row in traj[toff[r]:toff[r + 1]])
                rounds.append(RoundRecord(round_id=int(rid[r]), trigger_action_index=int(trig[r]),
                                          horizon=int(hor[r]), chunk_size=s.chunk_size,
                                          update_magnitudes=UpdateMagnitudes(U[r]),
                                          action_trajectory=tr))
            out.append(TaskTrace(task_id=tid, control_hz=s.control_hz,
                                 obs_payload_bytes=s.obs_payload_bytes,
                                 action_payload_bytes=s.action_payload_bytes,
                                 success=bool(succ[t]), rounds=tuple(rounds)))
        return out


def synthesize_family_columns(spec: SyntheticSpec, policy: HorizonPolicyConfig,
                              gen_latency: Duration, count: int, seed: int,
                              id_prefix: str = "task", with_trajectories: bool = False,
                              trajectory_dim: int = 3, task_ids: Optional[list] = None,
                              rounds_per_launch: int = 8) -> SynthColumns:
    """`count` synthetic traces on the device.  Task i draws from the Philox
    stream (seed, i); ids are f"{id_prefix}-{i:04d}" (workload.py:453) unless
    `task_ids` is given."""
    _check_fits(spec, policy, gen_latency)
    if count < 0:
        raise ValueError("count must be >= 0")
    lib = _lib.load()
    d = dev.device()
    st = dev.stream()
    seed64 = int(seed) & ((1 << 64) - 1)
    K, N, G = spec.diffusion_steps, spec.chunk_size, max(1, int(rounds_per_launch))
    slack = generation_slack_actions(gen_latency, spec.control_hz)
    ids = list(task_ids) if task_ids is not None else [f"{id_prefix}-{i:04d}" for i in range(count)]
    if len(ids) != count:
        raise ValueError("task_ids must have `count` entries")
    c_spec = spec.c_struct()
    keys = torch.arange(count, dtype=torch.int64, device=d)
    state = torch.zeros((count, 4), dtype=torch.int32, device=d)
    state[:, 1] = -1
    active = keys
    parts = []
    round0 = 0
    while active.numel():
        A = active.numel()
        U = torch.empty((A, G, K, N), dtype=torch.float64, device=d)
        _lib.check(lib.kr_synth_magnitudes(ctypes.byref(c_spec), seed64, active.data_ptr(), A,
                                           round0, G, U.data_ptr(), st), "kr_synth_magnitudes")
        H = decide_horizon_batch(policy, U.view(A * G, K, N), validate=False).view(A, G)
        s_act = state[active].contiguous()
        trig = torch.empty((A, G), dtype=torch.int32, device=d)
        used = torch.empty((A, G), dtype=torch.uint8, device=d)
        _lib.check(lib.kr_synth_close(H.data_ptr(), A, G, spec.action_budget, slack,
                                      s_act.data_ptr(), trig.data_ptr(), used.data_ptr(), st),
                   "kr_synth_close")
        state[active] = s_act
        m = used.bool()
        g_idx = torch.arange(G, dtype=torch.int32, device=d).expand(A, G)
        parts.append((active.view(A, 1).expand(A, G)[m], (g_idx + round0)[m], trig[m], H[m], U[m]))
        active = active[s_act[:, 3] == 0]
        round0 += G
    if parts:
        task = torch.cat([p[0] for p in parts])
        rid = torch.cat([p[1] for p in parts])
        order = torch.argsort(task * (round0 + 1) + rid.to(torch.int64))
        task, rid = task[order], rid[order]
        trig = torch.cat([p[2] for p in parts])[order]
        hor = torch.cat([p[3] for p in parts])[order]
        U = torch.cat([p[4] for p in parts])[order]
    else:
        task = torch.zeros(0, dtype=torch.int64, device=d)
        rid = trig = hor = torch.zeros(0, dtype=torch.int32, device=d)
        U = torch.zeros((0, K, N), dtype=torch.float64, device=d)
    counts = torch.bincount(task, minlength=count)
    round_off = torch.zeros(count + 1, dtype=torch.int64, device=d)
    round_off[1:] = torch.cumsum(counts, 0)
    success = torch.empty(count, dtype=torch.uint8, device=d)
    _lib.check(lib.kr_synth_success(seed64, keys.data_ptr(), count, float(spec.success_rate),
                                    success.data_ptr(), st), "kr_synth_success")
    cols = SynthColumns(task_ids=ids, spec=spec, round_off=round_off, round_task=task,
                        round_id=rid.to(torch.int32), trigger_action_index=trig, horizon=hor,
                        U=U, success=success.bool())
    if with_trajectories:
        nr = cols.n_rounds
        toff = torch.zeros(nr + 1, dtype=torch.int64, device=d)
        toff[1:] = torch.cumsum(hor.to(torch.int64), 0)
        rows = int(toff[-1].item()) if nr else 0
        traj = torch.empty((rows, trajectory_dim), dtype=torch.float64, device=d)
        rid32 = cols.round_id.contiguous()
        hor32 = hor.contiguous()
        _lib.check(lib.kr_synth_trajectories(seed64, task.data_ptr(), rid32.data_ptr(),
                                             hor32.data_ptr(), toff.data_ptr(), nr, trajectory_dim,
                                             traj.data_ptr(), st), "kr_synth_trajectories")
        cols.traj_row_off, cols.traj = toff, traj
    return cols


def synthesize_trace(spec: SyntheticSpec, policy: HorizonPolicyConfig, gen_latency: Duration,
                     seed: int, task_id: str = "task-0", with_trajectories: bool = False,
                     trajectory_dim: int = 3) -> TaskTrace:
    """One task trace whose request timing assumes zero contention
    (workload.py:371-442): the Philox stream (seed, 0)."""
    return synthesize_family_columns(spec, policy, gen_latency, 1, seed, task_ids=[task_id],
                                     with_trajectories=with_trajectories,
                                     trajectory_dim=trajectory_dim).to_traces()[0]


def synthesize_family(spec: SyntheticSpec, policy: HorizonPolicyConfig, gen_latency: Duration,
                      count: int, seed: int, id_prefix: str = "task", **kwargs) -> list:
    """A family of traces, task i on the Philox stream (seed, i)
    (workload.py:445-456)."""
    return synthesize_family_columns(spec, policy, gen_latency, count, seed, id_prefix=id_prefix,
                                     **kwargs).to_traces()


def cmd_gen_traces(spec: str | Path, out_dir: str | Path, policy: str = "confidence",
                   static_h: Optional[int] = None, threshold: float = 0.4, h_min: int = 5) -> int:
    """`roboserve gen-traces` (cli.py:32-53): a spec file (SyntheticSpec fields
    plus `count`, `seed`, `gen_latency_us`) -> out_dir/traces.jsonl, the family
    synthesised on the device."""
    if policy == "static":
        if static_h is None:
            raise ValueError("--static-h is required with --policy static")
        pol = HorizonPolicyConfig.static(static_h)
    else:
        pol = HorizonPolicyConfig.confidence(threshold=threshold, min_horizon=h_min)
    spec_data = json.loads(Path(spec).read_text(encoding="utf-8"))
    count = spec_data.pop("count", 1)
    seed = spec_data.pop("seed", 0)
    gen_latency = spec_data.pop("gen_latency_us", 300_000)
    traces = synthesize_family(SyntheticSpec.from_dict(spec_data), pol, gen_latency, count, seed)
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    out_path = out / "traces.jsonl"
    store_traces(traces, out_path)
    print(f"wrote {len(traces)} traces to {out_path}")
    return 0
