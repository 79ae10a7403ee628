"""B200-native search engine for the model-checking auto-tuner of arXiv:2305.09130.

Drop-in for the reference's tuning path (mctune: model / explore / search):
the configuration-space evaluation, the schedule trajectories, the
interleaving exploration and the bound-lowering driver run as sm_100a CUDA
kernels behind the C ABI in include/mctune_b200.h.
"""
from ._lib import (ConfigError, CorruptTrace, CudaError, LimitError, MctuneError, ModelBug,
                   NoDeviceError, device_count)
from .model import (ABSTRACT, MINIMUM, LaunchPlan, PlatformConfig, ProblemSpec, TuningParams,
                    config_feasible, derive_launch, enumerate_configs, kernel_kind_from_string,
                    log2_exact, validate_params)
from .machine import (FIRST, MT19937, PHILOX, ROUND_ROBIN, SEEDED_RANDOM, Machine, RunOutcome,
                      Trace, TrajectoryBatch, replay, trace_to_text, trajectories)
from .explore import ExploreStats, SweepInfo, check_nontermination, explore_configs, explore_machine
from .search import (RankedTrail, SweepRow, TuneProbe, TuneResult, Verdict, bisect_min_time, check_overtime,
                     exhaustive_sweep, extract_params, rank_trails, swarm_min_time, tune)
from .space import KEY_INDEX_BITS, KEY_SAT, KEY_TIME_BITS, Space, SpaceResult, space_argmin

__all__ = [
    "ABSTRACT", "MINIMUM", "ConfigError", "CorruptTrace", "CudaError", "LimitError",
    "MctuneError", "ModelBug", "NoDeviceError", "LaunchPlan", "PlatformConfig", "ProblemSpec",
    "TuningParams", "SweepRow", "Space", "SpaceResult", "KEY_INDEX_BITS", "KEY_SAT",
    "KEY_TIME_BITS", "config_feasible", "derive_launch", "device_count", "enumerate_configs",
    "exhaustive_sweep", "kernel_kind_from_string", "log2_exact", "space_argmin",
    "validate_params", "FIRST", "MT19937", "PHILOX", "ROUND_ROBIN", "SEEDED_RANDOM", "Machine",
    "RunOutcome", "RankedTrail", "TuneProbe", "TuneResult", "Verdict", "bisect_min_time", "check_overtime",
    "extract_params", "rank_trails", "swarm_min_time", "tune", "ExploreStats", "SweepInfo", "explore_configs", "explore_machine", "check_nontermination", "Trace", "TrajectoryBatch", "replay", "trace_to_text", "trajectories",
]
