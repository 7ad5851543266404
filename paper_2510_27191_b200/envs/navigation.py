"""Grid navigation through a partially known obstacle field (device counterpart of
/root/reference/pkg/src/vecpomdp/envs/navigation.py).

A robot starts on a free top-border cell and must reach the goal at the bottom,
passing one of two gates in a wall; exactly one gate is open.  The occupancy of
the '?' cells and which gate is open are hidden; every step returns a noisy 8-bit
reading of the occupancy of the 8 neighbour cells (|A| = 9 with "stay",
|O| = 256 + terminal).  The step, the leaf heuristic and the SIR likelihood run
on the device (csrc/vp_models.cuh, NavigationModel) from per-cell tables; the
host keeps the map, the prior and the initial-state sampler.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from ..core import ProblemModel, ProblemSpec
from ._device import nav_unpacker, navigation_descriptor

DEFAULT_MAP = "\n".join([
    ".............",
    "?????????????",
    "?????????????",
    "?????????????",
    "?????????????",
    "???.?????.???",
    "###|#####|###",
    "???.?????.???",
    "?????????????",
    "?????????????",
    "??????.??????",
    "??????.??????",
    "......G......",
])
FREE, WALL, GATE, UNKNOWN = 0, 1, 2, 3
_DR = np.array([-1, -1, 0, 1, 1, 1, 0, -1], dtype=np.int64)  # N NE E SE S SW W NW
_DC = np.array([0, 1, 1, 1, 0, -1, -1, -1], dtype=np.int64)


@dataclass
class NavStates:
    pos: np.ndarray
    occ: np.ndarray
    open_gate: np.ndarray
    terminal: np.ndarray

    def __len__(self) -> int:
        return len(self.pos)

    def take(self, indices) -> "NavStates":
        i = np.asarray(indices, dtype=np.int64)
        return NavStates(self.pos[i], self.occ[i], self.open_gate[i], self.terminal[i])


class NavigationModel(ProblemModel):
    def __init__(self, map_text: str = DEFAULT_MAP, p_obstacle: float = 0.25, sensor_accuracy: float = 0.9,
                 discount: float = 0.983, max_steps: int = 60):
        lines = [ln for ln in map_text.splitlines() if ln.strip()]
        self.height, self.width = len(lines), len(lines[0])
        if any(len(ln) != self.width for ln in lines):
            raise ValueError("map rows must have equal length")
        table = {".": FREE, "G": FREE, "#": WALL, "|": GATE, "?": UNKNOWN}
        if any(ch not in table for ln in lines for ch in ln):
            raise ValueError("unknown map character")
        kind = np.array([[table[ch] for ch in ln] for ln in lines], dtype=np.int64)
        self.kind = kind.astype(np.int8)
        self.goal = np.array([[ch == "G" for ch in ln] for ln in lines])
        self.aux = np.full(kind.shape, -1, dtype=np.int64)  # index among gates / unknown cells
        for k in (GATE, UNKNOWN):
            flat = np.flatnonzero(kind.reshape(-1) == k)
            self.aux.reshape(-1)[flat] = np.arange(len(flat))
        self.n_gates, self.n_unknown = int((kind == GATE).sum()), int((kind == UNKNOWN).sum())
        if self.n_gates != 2:
            raise ValueError("map must contain exactly two gates")
        self.start_cells = np.flatnonzero((kind[0] == FREE) & ~self.goal[0]).astype(np.int64)
        if not len(self.start_cells):
            raise ValueError("top border has no free start cells")
        self.p_obstacle, self.sensor_accuracy = p_obstacle, sensor_accuracy
        self.spec = ProblemSpec("navigation", 9, 256, discount, max_steps)
        self.goal_dist = self._goal_distances()
        self._dm = None

    def _goal_distances(self) -> np.ndarray:
        """Optimistic 8-connected BFS distance to the goal (walls block; navigation.py:127-144)."""
        dist = np.full(self.kind.shape, np.inf)
        ring = [tuple(x) for x in np.argwhere(self.goal)]
        for cell in ring:
            dist[cell] = 0.0
        while ring:
            nxt = []
            for r, c in ring:
                for dr, dc in zip(_DR, _DC):
                    rr, cc = r + dr, c + dc
                    if 0 <= rr < self.height and 0 <= cc < self.width and self.kind[rr, cc] != WALL \
                            and dist[rr, cc] == np.inf:
                        dist[rr, cc] = dist[r, c] + 1
                        nxt.append((rr, cc))
            ring = nxt
        return dist

    def device_descriptor(self):
        if self._dm is None:
            self._dm = navigation_descriptor(self, nav_unpacker(self.n_unknown, NavStates))
        return self._dm

    def sample_initial_states(self, n: int, rng) -> NavStates:
        if n < 1:
            raise ValueError("n must be >= 1")
        rows = np.arange(n, dtype=np.int64)
        pos = self.start_cells[(rng.derive(0).uniform(rows) * len(self.start_cells)).astype(np.int64)]
        occ = rng.derive(1).uniform(rows, self.n_unknown) < self.p_obstacle
        gate = (rng.derive(2).uniform(rows) < 0.5).astype(np.int64)
        return NavStates(pos, occ, gate, np.zeros(n, dtype=bool))

    def step_batch(self, states, actions, rng):
        return self.device_descriptor().step(states, actions, rng)

    def value_heuristic(self, states) -> np.ndarray:
        return self.device_descriptor().heuristic(states)

    def _blocked(self, s, r, c):
        off = (r < 0) | (r >= self.height) | (c < 0) | (c >= self.width)
        rr, cc = np.clip(r, 0, self.height - 1), np.clip(c, 0, self.width - 1)
        kind, aux = self.kind[rr, cc], self.aux[rr, cc]
        out = off | (kind == WALL) | (~off & (kind == GATE) & (aux != s.open_gate))
        unk = np.flatnonzero(~off & (kind == UNKNOWN))
        out[unk] |= s.occ[unk, aux[unk]]
        return out

    def observation_log_likelihood(self, nxt, action: int, observation: int) -> np.ndarray:
        """Host likelihood for the host SIR path (the device SIR uses the kernel's)."""
        if not 0 <= observation <= self.spec.terminal_obs:
            raise ValueError("invalid observation code")
        out = np.full(len(nxt), -np.inf)
        if observation == self.spec.terminal_obs:
            out[nxt.terminal] = 0.0
            return out
        r, c = nxt.pos // self.width, nxt.pos % self.width
        bits = np.stack([self._blocked(nxt, r + _DR[i], c + _DC[i]) for i in range(8)], axis=1)
        want = ((observation >> np.arange(8)) & 1).astype(bool)
        live = ~nxt.terminal
        hits = (bits == want).sum(axis=1)[live]
        miss = 8 - hits
        with np.errstate(divide="ignore", invalid="ignore"):
            out[live] = hits * np.log(self.sensor_accuracy) + np.where(
                miss > 0, miss * np.log(1.0 - self.sensor_accuracy), 0.0)
        return out
