"""2-D Light-Dark navigation with continuous, hashed observations.

BASELINE config 4 ("continuous-observation navigation (Light-Dark-style) with
per-particle observation hashing") has no reference counterpart; this model
is defined identically in oracle/envs.py (run through the reference solver
for tests/golden/plan_lightdark.npz).  Observations are the noisy next
position quantised per axis into ``bins`` cells: |O| = bins^2 codes, looked
up in the belief hash index like any other observation.  The step runs on
the device (csrc/vp_models.cuh, LightDarkModel).
"""

from __future__ import annotations

from dataclasses import dataclass
from math import erf, sqrt

import numpy as np

from ..core import ProblemModel, ProblemSpec
from ._device import lightdark_descriptor


@dataclass
class LightDarkStates:
    x: np.ndarray
    y: np.ndarray
    terminal: np.ndarray

    def __len__(self) -> int:
        return len(self.terminal)

    def take(self, indices) -> "LightDarkStates":
        i = np.asarray(indices, dtype=np.int64)
        return LightDarkStates(self.x[i], self.y[i], self.terminal[i])


class LightDarkModel(ProblemModel):
    def __init__(self, step: float = 1.0, light_x: float = 5.0, goal_radius: float = 1.0, sigma0: float = 0.05,
                 sigma_slope: float = 0.5, bin_width: float = 0.25, bins: int = 64, discount: float = 0.95,
                 max_steps: int = 60):
        if bins < 1 or bin_width <= 0:
            raise ValueError("need positive bins and bin width")
        self.step, self.light_x, self.goal_radius = float(step), float(light_x), float(goal_radius)
        self.sigma0, self.sigma_slope = float(sigma0), float(sigma_slope)
        self.bin_width, self.bins = float(bin_width), int(bins)
        self.spec = ProblemSpec("lightdark", 9, self.bins * self.bins, discount, max_steps)
        self._dm = None

    def device_descriptor(self):
        if self._dm is None:
            self._dm = lightdark_descriptor(
                self, lambda rec: LightDarkStates(rec["x"].copy(), rec["y"].copy(), rec["term"].astype(bool)))
        return self._dm

    def sample_initial_states(self, n: int, rng) -> LightDarkStates:
        if n < 1:
            raise ValueError("n must be >= 1")
        u = rng.derive(0).uniform(np.arange(n, dtype=np.int64), 2)
        return LightDarkStates(2.0 + 4.0 * u[:, 0], -2.0 + 4.0 * u[:, 1], np.zeros(n, dtype=bool))

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
        sigma = self.sigma0 + self.sigma_slope * np.abs(nxt.x - self.light_x)
        cdf = np.vectorize(lambda e, c, s: 0.5 * (1.0 + erf((e - c) / (s * sqrt(2.0)))))
        half = self.bins // 2

        def mass(center, b):
            lo = 0.0 if b == 0 else cdf((b - half) * self.bin_width, center, sigma)
            hi = 1.0 if b == self.bins - 1 else cdf((b + 1 - half) * self.bin_width, center, sigma)
            return hi - lo

        p = mass(nxt.x, observation // self.bins) * mass(nxt.y, observation % self.bins)
        live = ~nxt.terminal
        with np.errstate(divide="ignore"):
            out[live] = np.log(p[live])
        return out
