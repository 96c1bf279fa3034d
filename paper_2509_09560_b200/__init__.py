"""B200-native Auras hot path: perception -> public-context ring in HBM ->
batched staggered-timestep denoise chain, run as a frame-clocked pipeline on
two CUDA streams.

Drop-in names of the reference package (fp/__init__.py:5-37) for the hot path:
`ContextKind`, `ContextStore`, `PublicContext`, `PipelineConfig`, `RunResult`,
`RequestRecord`, `run_pipelined`, `run_sequential`, `Policy`,
`make_conditioning_policy`, `StagePlan`, `plan_stages`, `split_generation`,
`split_perception`, `RolloutMetrics`, `summarize`; plus the Diffusion Policy
CNN plugin `make_diffusion_policy`.
"""

__version__ = "0.1.0"

from .context import ContextKind, ContextStore, PublicContext
from .errors import (LengthExceeded, SequenceComplete, BaselineMissing, ConfigInvalid, NoFeasibleConfig, DeadlockDetected, DeviceError, FramepipeError,
                     IncompleteGeneration, InvalidStageCount, KindMismatch, NotYetPublished,
                     OffsetOutOfRange, ShapeMismatch, StaleWrite, TooManyStages)
from .executor import (PipelineConfig, RequestRecord, RunResult, run_decoupled, run_parallel, run_pipelined,
                       run_sequential)
from .metrics import ComparisonTable, RolloutMetrics, compare, read_metrics, summarize, write_trace_jsonl
from .partition import StagePlan, plan_stages, split_generation, split_perception
from .tuner import GridPoint, TuneRequest, TuneResult, finetune_alpha, grid_search
from .policy import make_autoregressive_policy, ActionOutput, Observation, Policy, make_conditioning_policy


def make_diffusion_policy(*args, **kwargs):
    from .diffusion import make_diffusion_policy as _make
    return _make(*args, **kwargs)


from .transformer import CausalTransformer, KvCache, TransformerConfig

__all__ = [
    "CausalTransformer", "KvCache", "TransformerConfig", "LengthExceeded", "SequenceComplete",
    "ActionOutput", "ConfigInvalid", "ContextKind", "ContextStore", "DeadlockDetected",
    "BaselineMissing", "NoFeasibleConfig", "DeviceError", "FramepipeError", "IncompleteGeneration", "InvalidStageCount", "KindMismatch",
    "NotYetPublished", "Observation", "OffsetOutOfRange", "PipelineConfig", "Policy",
    "PublicContext", "RequestRecord", "RolloutMetrics", "RunResult", "ShapeMismatch",
    "StagePlan", "StaleWrite", "TooManyStages", "make_conditioning_policy", "make_autoregressive_policy",
    "make_diffusion_policy", "plan_stages", "run_decoupled", "run_parallel", "run_pipelined", "run_sequential",
    "split_generation", "split_perception", "summarize", "compare", "ComparisonTable", "read_metrics",
    "write_trace_jsonl", "TuneRequest", "TuneResult", "GridPoint", "grid_search", "finetune_alpha",
]
