"""B200-native Kairos decision core (arXiv 2605.11381), drop-in for the hot path
of the reference package `roboserve`:

* step 1, execution-horizon selection: `decide_horizon` (confidence threshold
  over refinement-update magnitudes) and `round_optimal_horizon` (per-action
  cosine divergence against the unexecuted overlap of the previous chunk);
* step 2, execution-aware urgency: wait ledger, wait ratio, bucket with aging,
  projected execution duration and next-need time;
* step 3, priority ordering and top-k edge admission: `plan` (with
  `LedgerStates`, the simulator's planning loop runs against a
  device-resident incremental task ledger).

Every decision runs in hand-written sm_100a CUDA kernels behind the C ABI in
include/kairos_b200.h (libkairos_b200.so); there is no CPU fallback.  The
reference's names and signatures are kept; `*_batch` variants and
`DecisionRound` (fleet-scale, device-resident) are the production entry points.
"""

from .core import (ActionChunk, Duration, Interval, LastExecInfo, PendingRequest,  # noqa: F401
                   RoundTimeline, TaskState, TimePoint, exec_duration, exec_end_from_piggyback,
                   us_from_actions, us_from_actions_batch)
from .divergence import (dot_order, round_optimal_horizon, round_optimal_horizon_batch,  # noqa: F401
                         set_dot_order)
from .engines import (EngineProfile, NetworkModel, ProfileError, batch_latency,  # noqa: F401
                      cloud_round_trip, transfer_time)
from .ledger import DeviceLedger, LedgerStates  # noqa: F401
from .horizon import (HorizonPolicyConfig, UpdateMagnitudes, decide_horizon,  # noqa: F401
                      decide_horizon_batch, sweep_horizon_sums, sweep_thresholds)
from .scheduler import (DispatchPlan, SchedulerConfig, assign_bucket,  # noqa: F401
                        estimate_exec_latency, order_within_bucket, plan, plan_fifo, plan_las)
from .synth import (SynthColumns, SyntheticSpec, generation_slack_actions,  # noqa: F401
                    synthesize_family, synthesize_family_columns, synthesize_trace)
from .traces import (RoundRecord, TaskTrace, TraceColumns, TraceFormatError,  # noqa: F401
                     load_trace_columns, load_trace_dir, load_traces, pareto_rows, store_traces,
                     trace_from_dict, trace_to_dict)
from .waiting import (WaitLedger, current_wait_ratio, ledger_from_history,  # noqa: F401
                      round_wait, wait_ratio)

__version__ = "0.1.0"
