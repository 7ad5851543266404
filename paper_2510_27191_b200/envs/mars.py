"""Two-agent rock sampling -- the reference's RockSample family.

API mirror of /root/reference/pkg/src/vecpomdp/envs/mars.py:44-257 whose
generative step and leaf heuristic run on the device (csrc/vp_models.cuh,
MarsModel).  Host code keeps what happens once per planning step: rock layout,
initial-belief sampling and the SIR likelihood.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from ..core import ProblemModel, ProblemSpec
from ..rng import RowRng
from ._device import mars_descriptor

GOOD, BAD, NULL = 0, 1, 2


@dataclass
class MarsStates:
    x: np.ndarray        # (n, 2); x == n means departed
    y: np.ndarray        # (n, 2)
    rocks: np.ndarray    # (n, m) bool
    terminal: np.ndarray

    def __len__(self) -> int:
        return len(self.terminal)

    def take(self, indices) -> "MarsStates":
        i = np.asarray(indices, dtype=np.int64)
        return MarsStates(self.x[i], self.y[i], self.rocks[i], self.terminal[i])


class MarsModel(ProblemModel):
    def __init__(self, n: int = 20, m: int = 20, layout_seed: int = 0, half_efficiency_distance: float = 20.0,
                 discount: float = 0.983, max_steps: int = 90):
        if n < 2 or m < 1:
            raise ValueError("need a grid of at least 2 and at least one rock")
        self.n, self.m = n, m
        self.half_efficiency_distance = half_efficiency_distance
        # m cells with the smallest layout-stream uniforms (mars.py:63-66)
        order = np.argsort(RowRng.from_seed(layout_seed).derive(0).uniform(np.arange(n * n, dtype=np.int64)))
        cells = order[:m]
        self.rock_x = (cells % n).astype(np.int64)
        self.rock_y = (cells // n).astype(np.int64)
        self.rock_at = np.full((n, n), -1, dtype=np.int64)
        self.rock_at[self.rock_x, self.rock_y] = np.arange(m)
        self.start_x = np.array([0, 0], dtype=np.int64)
        self.start_y = np.array([n // 3, (2 * n) // 3], dtype=np.int64)
        self.per_agent_ops = 5 + m
        self.spec = ProblemSpec("mars", self.per_agent_ops ** 2, 9, discount, max_steps)
        self._dm = None

    def device_descriptor(self):
        if self._dm is None:
            self._dm = mars_descriptor(self, self._unpack)
        return self._dm

    def _unpack(self, rec) -> MarsStates:
        x = np.stack([rec["x0"], rec["x1"]], axis=1).astype(np.int64)
        y = np.stack([rec["y0"], rec["y1"]], axis=1).astype(np.int64)
        bits = rec["rocks"].astype(np.uint64)
        rocks = ((bits[:, None] >> np.arange(self.m, dtype=np.uint64)[None, :]) & np.uint64(1)).astype(bool)
        return MarsStates(x, y, rocks, rec["term"].astype(bool))

    def check_accuracy(self, dist):
        return 0.5 * (1.0 + 2.0 ** (-dist / self.half_efficiency_distance))

    def sample_initial_states(self, n: int, rng) -> MarsStates:
        if n < 1:
            raise ValueError("n must be >= 1")
        rocks = rng.derive(0).uniform(np.arange(n, dtype=np.int64), self.m) < 0.5
        return MarsStates(np.tile(self.start_x, (n, 1)), np.tile(self.start_y, (n, 1)), rocks,
                          np.zeros(n, dtype=bool))

    def step_batch(self, states, actions, rng):
        return self.device_descriptor().step(states, actions, rng)

    def value_heuristic(self, states) -> np.ndarray:
        return self.device_descriptor().heuristic(states)

    def observation_log_likelihood(self, nxt, action: int, observation: int) -> np.ndarray:
        """Per-particle log p(o | s', a) for SIR (mars.py:182-221)."""
        if not 0 <= observation <= self.spec.terminal_obs:
            raise ValueError("invalid observation code")
        out = np.full(len(nxt), -np.inf)
        if observation == self.spec.terminal_obs:
            out[nxt.terminal] = 0.0
            return out
        logp = np.zeros(len(nxt))
        for k, (op, want) in enumerate(zip(divmod(action, self.per_agent_ops), divmod(observation, 3))):
            null_p = 1.0 if want == NULL else 0.0
            if op >= 5:
                rk = op - 5
                d = np.sqrt((nxt.x[:, k] - self.rock_x[rk]) ** 2.0 + (nxt.y[:, k] - self.rock_y[rk]) ** 2.0)
                acc = self.check_accuracy(d)
                good = nxt.rocks[:, rk]
                p = {GOOD: np.where(good, acc, 1.0 - acc), BAD: np.where(good, 1.0 - acc, acc)}.get(
                    want, np.zeros(len(nxt)))
                p = np.where(nxt.x[:, k] != self.n, p, null_p)
            else:
                p = np.full(len(nxt), null_p)
            with np.errstate(divide="ignore"):
                logp += np.log(p)
        live = ~nxt.terminal
        out[live] = logp[live]
        return out

    def step_metrics(self, states, action: int, result) -> dict:
        good = bad = 0
        rocks = states.rocks[0].copy()
        for k, op in enumerate(divmod(action, self.per_agent_ops)):
            if op == 4 and states.x[0, k] < self.n and not states.terminal[0]:
                rk = self.rock_at[states.x[0, k], states.y[0, k]]
                if rk >= 0 and rocks[rk]:
                    good += 1
                    rocks[rk] = False
                else:
                    bad += 1
        return {"rocks_good": float(good), "rocks_bad": float(bad)}
