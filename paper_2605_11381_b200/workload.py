"""`roboserve.workload` names: the divergence horizon (workload.py:461-496,
divergence.py), trace I/O (workload.py:29-262, traces.py) and synthesis on
the device (workload.py:296-456, synth.py)."""

from .divergence import _cosine, round_optimal_horizon, round_optimal_horizon_batch  # noqa: F401
from .synth import (SyntheticSpec, SynthColumns, generation_slack_actions,  # noqa: F401
                    synthesize_family, synthesize_family_columns, synthesize_trace)
from .traces import (RoundRecord, TaskTrace, TraceFormatError, load_trace_dir,  # noqa: F401
                     load_traces, store_traces, trace_from_dict, trace_to_dict)
