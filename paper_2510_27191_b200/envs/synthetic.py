"""Integer-hash synthetic POMDP for the depth x width scaling sweep.

BASELINE config 5 names a "synthetic scaling sweep" the reference does not
ship.  This model (defined identically in oracle/envs.py, which the reference
solver ran to produce tests/golden/plan_synthetic.npz) has one 64-bit hidden
word per state; dynamics are SplitMix64 hashes and exactly-rounded fp64 ops,
so the device step (csrc/vp_models.cuh, SyntheticModel) is bit-identical.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from ..core import ProblemModel, ProblemSpec
from ..rng import RowRng, _mix64_np
from ._device import synthetic_descriptor


@dataclass
class SyntheticStates:
    word: np.ndarray
    terminal: np.ndarray

    def __len__(self) -> int:
        return len(self.terminal)

    def take(self, indices) -> "SyntheticStates":
        i = np.asarray(indices, dtype=np.int64)
        return SyntheticStates(self.word[i], self.terminal[i])


class SyntheticModel(ProblemModel):
    def __init__(self, n_actions: int = 16, n_obs: int = 8, branching: int = 4, obs_accuracy: float = 0.8,
                 term_per_mille: int = 10, seed: int = 0, discount: float = 0.95, max_steps: int = 100):
        if n_actions < 1 or n_obs < 1 or branching < 1:
            raise ValueError("sizes must be positive")
        if not 0 <= term_per_mille <= 1000:
            raise ValueError("term_per_mille must be in [0, 1000]")
        self.n_actions, self.n_obs, self.branching = n_actions, n_obs, branching
        self.obs_accuracy = float(obs_accuracy)
        self.term_per_mille = term_per_mille
        self.seed = seed
        self.salt = RowRng.from_seed(seed).key
        self.spec = ProblemSpec("synthetic", n_actions, n_obs, discount, max_steps)
        self._dm = None

    def device_descriptor(self):
        if self._dm is None:
            self._dm = synthetic_descriptor(
                self, lambda rec: SyntheticStates(rec["word"].astype(np.uint64), rec["term"].astype(bool)))
        return self._dm

    def sample_initial_states(self, n: int, rng) -> SyntheticStates:
        if n < 1:
            raise ValueError("n must be >= 1")
        u = rng.derive(0).uniform(np.arange(n, dtype=np.int64))
        word = _mix64_np((u * 2.0 ** 53).astype(np.uint64) ^ np.uint64(self.salt))
        return SyntheticStates(word, np.zeros(n, dtype=bool))

    def step_batch(self, states, actions, rng):
        return self.device_descriptor().step(states, actions, rng)

    def value_heuristic(self, states) -> np.ndarray:
        return self.device_descriptor().heuristic(states)

    def observation_log_likelihood(self, nxt, action: int, observation: int) -> np.ndarray:
        if not 0 <= observation <= self.spec.terminal_obs:
            raise ValueError("invalid observation code")
        out = np.full(len(nxt), -np.inf)
        if observation == self.spec.terminal_obs:
            out[nxt.terminal] = 0.0
            return out
        true_obs = ((nxt.word >> np.uint64(17)) % np.uint64(self.n_obs)).astype(np.int64)
        p = self.obs_accuracy * (true_obs == observation) + (1.0 - self.obs_accuracy) / self.n_obs
        live = ~nxt.terminal
        out[live] = np.log(p[live])
        return out
