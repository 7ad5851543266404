"""CPU oracle for the PORPP planning step -- TEST INFRASTRUCTURE ONLY.

This package is a numpy restatement of the reference solver's planning path
(``vecpomdp``: /root/reference/pkg/src/vecpomdp/{rng,core,tree,search,backup,
belief,solver}.py and envs/{mars,tabular}.py).  Every function cites the
reference file:line it follows.  It exists to *check* the B200 product, never
to run in its place:

* only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
  leg / ``--impl reference`` arm may import it;
* the product package ``paper_2510_27191_b200`` never imports it and fails
  loudly when its CUDA library is missing.

Parity pinning: ``tests/golden/make_golden.py`` imports the real reference
from /root/reference (this container only) and writes golden vectors into
``tests/golden/*.npz``; ``tests/test_oracle_golden.py`` checks this oracle
against them (RNG, formula examples, full ``plan()`` trees for MARS, Tiger and
the two new models run through the reference solver).

Two problem models here have no reference counterpart (BASELINE configs 4 and
5 name problems the reference does not ship): ``SyntheticModel`` and
``LightDarkModel``.  They are written against the reference's ProblemModel
contract (pkg/src/vecpomdp/core.py:84-142) so the *reference solver* can plan
on them when the golden vectors are generated.
"""

from .rng import RowRng, BoundRng, mix64
from .tree import ColumnarTree, match_or_append_pairs
from .search import softmax_rows, sample_actions, search, SearchBatch, LeafResult
from .backup import log_sum_exp_rows, aggregate_leaves, action_q_values, backup, LevelValues
from .belief import ParticleBelief, systematic_resample, sir_update
from .solver import SolverConfig, PlanOutcome, plan, run_episode
from .envs import (
    ProblemSpec,
    MarsModel,
    MarsStates,
    TabularPOMDP,
    TabularModel,
    TabularStates,
    tiger_model,
    SyntheticModel,
    SyntheticStates,
    LightDarkModel,
    LightDarkStates,
    NavigationModel,
    NavStates,
    CrowdNavModel,
    CrowdStates,
)

__all__ = [
    "RowRng", "BoundRng", "mix64", "ColumnarTree", "match_or_append_pairs",
    "softmax_rows", "sample_actions", "search", "SearchBatch", "LeafResult",
    "log_sum_exp_rows", "aggregate_leaves", "action_q_values", "backup", "LevelValues",
    "ParticleBelief", "systematic_resample", "sir_update",
    "SolverConfig", "PlanOutcome", "plan", "run_episode",
    "ProblemSpec", "MarsModel", "MarsStates", "TabularPOMDP", "TabularModel",
    "TabularStates", "tiger_model", "SyntheticModel", "SyntheticStates",
    "LightDarkModel", "LightDarkStates", "NavigationModel", "NavStates", "CrowdNavModel", "CrowdStates",
]
