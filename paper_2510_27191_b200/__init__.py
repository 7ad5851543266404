"""B200-native PORPP planning step (arXiv 2510.27191), drop-in for ``vecpomdp.plan``.

The public names mirror the reference package (pkg/src/vecpomdp/__init__.py:
10-48): ``plan``/``search``/``backup``/``SolverConfig``/``RowRng``/... with the
tree, search and backup executed by hand-written sm_100a kernels behind the
C ABI in include/vpb200.h (libvpb200.so, loaded through ``_lib``).  There is
no CPU fallback: without the library or a CUDA device every compute entry
point raises.
"""

from . import _lib
from .backup import LevelValues, action_q_values, aggregate_leaves, backup, log_sum_exp_rows
from .belief import DeviceBelief, ParticleBelief, SirUpdate, sir_update, systematic_resample
from .core import ProblemModel, ProblemSpec, StateBatch, StepResult
from .envs import (CrowdNavModel, CrowdStates, LightDarkModel, MarsModel, NavigationModel, SyntheticModel, TabularModel, TabularPOMDP,
                   device_model, problem_from_config, tiger_model)
from .rng import BoundRng, PhiloxRowRng, RowRng
from .search import LeafResult, SearchBatch, sample_actions, search, search_recorded, softmax_rows
from .solver import Planner, PlanOutcome, RunRecord, SolverConfig, get_planner, plan, run_episode
from .shard import ShardedPlanner, shard_rows
from .plugin import CudaModel, RecordStates, compile_plugin
from .tree import DeviceTree, init_tree, match_or_append_pairs

BeliefTree = DeviceTree  # the reference's tree type (tree.py:100-132): here the device arena

__version__ = "0.1.0"

__all__ = [
    "BoundRng", "CrowdNavModel", "CrowdStates", "DeviceBelief", "DeviceTree", "LeafResult", "LightDarkModel", "MarsModel", "NavigationModel", "ParticleBelief", "PlanOutcome",
    "BeliefTree", "CudaModel", "StateBatch", "RecordStates", "compile_plugin", "Planner", "ProblemModel", "ShardedPlanner", "shard_rows", "ProblemSpec", "PhiloxRowRng", "RowRng", "RunRecord", "SearchBatch", "SirUpdate", "SolverConfig",
    "StepResult", "SyntheticModel", "TabularModel", "TabularPOMDP", "backup", "device_model", "get_planner",
    "init_tree", "log_sum_exp_rows", "plan", "problem_from_config", "run_episode", "sample_actions", "search",
    "sir_update", "search_recorded", "softmax_rows", "systematic_resample", "tiger_model", "LevelValues", "aggregate_leaves",
    "action_q_values", "match_or_append_pairs",
]
