"""B200-native deterministic elastic data-parallel step (EasyScale, arxiv 2208.14228).

Drop-in for the reference `bittrain` trainer / virtual-worker / elastic-rescale
path: same public names, argument meaning and exceptions, with every
computation in hand-written sm_100a CUDA behind the C-ABI of
include/bittrain_b200.h.  Out of scope (not re-exported): the planner,
scheduler, simulator and CLI of the reference.
"""

from .buckets import BucketMap, allreduce, build_buckets_initial, layout_arrival_perm, rebuild_buckets_first_minibatch
from .checkpoint import checkpoint_restore, checkpoint_save
from .engine import (DeterminismMode, ExecutorSpec, TrainingState, TrainRunConfig, apply_layout, assign_ranks,
                     check_replica_agreement, init_training, reconfigure, run_minibatch, run_steps, split_by_rank)
from .errors import (BittrainError, ConfigError, CorruptionError, FormatError, InputError, NumericError,
                     ProgressError, StateError, VersionError)
from . import placement
from .model import OptState, ToyModel, TrackedStat, forward_backward, sgd_step
from .placement import set_devices
from .prng import derive_stream, fnv1a64, rng_uniform01, shuffled_range, splitmix64_next
from .reduction import KernelProfile, Sequential, Tree, reduce_sum
from .runlog import RunLog, bitdiff, param_fingerprint
from .sampling import DataPipeline, SamplePlan, epoch_indices, make_dataset
from .scenarios import RestartEvent, RunSpec, run_matrix, run_scenario, run_training

__version__ = "0.1.0"

__all__ = [
    "BucketMap", "allreduce", "build_buckets_initial", "layout_arrival_perm", "rebuild_buckets_first_minibatch",
    "checkpoint_restore", "checkpoint_save", "DeterminismMode", "ExecutorSpec", "TrainingState", "TrainRunConfig",
    "apply_layout", "assign_ranks", "check_replica_agreement", "init_training", "reconfigure", "run_minibatch",
    "run_steps", "split_by_rank", "BittrainError", "ConfigError", "CorruptionError", "FormatError", "InputError",
    "NumericError", "ProgressError", "StateError", "VersionError", "OptState", "ToyModel", "TrackedStat",
    "forward_backward", "sgd_step", "derive_stream", "fnv1a64", "rng_uniform01", "shuffled_range",
    "splitmix64_next", "KernelProfile", "Sequential", "Tree", "reduce_sum", "RunLog", "bitdiff",
    "param_fingerprint", "DataPipeline", "SamplePlan", "epoch_indices", "make_dataset", "RestartEvent", "RunSpec",
    "run_matrix", "run_scenario", "run_training", "placement", "set_devices",
]
