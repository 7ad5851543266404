"""Robot crossing a hall among a reactive crowd (device counterpart of
/root/reference/pkg/src/vecpomdp/envs/crowdnav.py).

The robot starts at the middle of the southern border of a 50 x 40 m hall and
must leave through the northern border (+1000).  300 people jitter every step;
those within r_nearby react to the robot -- curious ones approach, shy ones
back away, and everyone backs away fast when the robot yells (-25).  Bumping
into anyone costs -200.  Each person's trait is hidden; the observation is one
bit per tracked person (the 6 nearest at the last executed step) telling
whether it closed distance, |O| = 64 + terminal.

The generative step, the leaf heuristic and the likelihood run on the device
(csrc/vp_models.cuh, CrowdNavModel) on 2704-byte records: the planner steps a
row with a whole warp, the record in shared memory (``step_warp``).  The host
keeps the initial-state sampler and the tracking refresh of the one executed
state; re-anchoring every particle's observable part on it (crowdnav.py:213-224)
is a device broadcast (``reconcile_device``), so the closed loop keeps the
belief resident in HBM with the device SIR update.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from ..core import ProblemModel, ProblemSpec
from ._device import crowd_unpacker, crowdnav_descriptor

NORTH, EAST, SOUTH, WEST, YELL = range(5)


@dataclass
class CrowdStates:
    robot: np.ndarray      # (n, 2) float64
    persons: np.ndarray    # (n, people, 2) float32
    curious: np.ndarray    # (n, people) bool, hidden
    tracked: np.ndarray    # (n, k) int64 person ids the sensor watches
    prev_dist: np.ndarray  # (n, k) float64 their distances at the previous step
    last_code: np.ndarray  # (n,) int64 code emitted on entering the state
    terminal: np.ndarray   # (n,) bool

    def __len__(self) -> int:
        return len(self.robot)

    def take(self, indices) -> "CrowdStates":
        i = np.asarray(indices, dtype=np.int64)
        return CrowdStates(self.robot[i], self.persons[i], self.curious[i], self.tracked[i], self.prev_dist[i],
                           self.last_code[i], self.terminal[i])


class CrowdNavModel(ProblemModel):
    def __init__(self, p_curious: float = 0.5, n_people: int = 300, n_tracked: int = 6, hall_width: float = 50.0,
                 hall_depth: float = 40.0, motion_noise: float = 0.05, react_prob: float = 0.9,
                 r_nearby: float = 4.0, v_curious: float = 0.3, v_shy: float = 0.8, v_back: float = 2.0,
                 collision_radius: float = 0.5, discount: float = 0.97, max_steps: int = 200):
        if not 0.0 <= p_curious <= 1.0:
            raise ValueError("p_curious must be in [0, 1]")
        if n_tracked > n_people:
            raise ValueError("n_tracked must not exceed n_people")
        self.p_curious, self.n_people, self.n_tracked = p_curious, n_people, n_tracked
        self.hall = np.array([hall_width, hall_depth])
        self.motion_noise, self.react_prob, self.r_nearby = motion_noise, react_prob, r_nearby
        self.v_curious, self.v_shy, self.v_back = v_curious, v_shy, v_back
        self.collision_radius = collision_radius
        self.spec = ProblemSpec("crowdnav", 5, 2 ** n_tracked, discount, max_steps)
        self._dm = None

    def device_descriptor(self):
        if self._dm is None:
            self._dm = crowdnav_descriptor(self, crowd_unpacker(self.n_people, self.n_tracked, CrowdStates))
        return self._dm

    # -- host pieces: initial sampler and tracking (numpy; once per episode step, off the planning path)
    def _distances(self, robot, persons) -> np.ndarray:
        d = persons.astype(np.float64) - robot[:, None, :]
        return np.sqrt((d ** 2).sum(axis=2))

    def _nearest(self, robot, persons):
        """The n_tracked nearest people and their distances (crowdnav.py:93-96, 199-211)."""
        dist = self._distances(robot, persons)
        ids = np.argsort(dist, axis=1)[:, : self.n_tracked].astype(np.int64)
        return ids, np.take_along_axis(dist, ids, axis=1)

    def sample_initial_states(self, n: int, rng) -> CrowdStates:
        """crowdnav.py:98-114: people uniform over the hall, traits Bernoulli(p_curious)."""
        if n < 1:
            raise ValueError("n must be >= 1")
        rows = np.arange(n, dtype=np.int64)
        robot = np.tile(np.array([self.hall[0] / 2.0, 0.0]), (n, 1))
        uni = rng.derive(0).uniform(rows, 2 * self.n_people).reshape(n, self.n_people, 2)
        persons = (uni * self.hall).astype(np.float32)
        curious = rng.derive(1).uniform(rows, self.n_people) < self.p_curious
        tracked, prev = self._nearest(robot, persons)
        return CrowdStates(robot, persons, curious, tracked, prev, np.zeros(n, dtype=np.int64), np.zeros(n, dtype=bool))

    def refresh_executed(self, executed: CrowdStates) -> CrowdStates:
        tracked, prev = self._nearest(executed.robot, executed.persons)
        return CrowdStates(executed.robot, executed.persons, executed.curious, tracked, prev, executed.last_code,
                           executed.terminal)

    def reconcile_belief(self, particles: CrowdStates, executed: CrowdStates) -> CrowdStates:
        """Observable part from the executed state, hidden traits from each particle (crowdnav.py:213-224)."""
        n = len(particles)

        def rep(x):
            return np.repeat(np.asarray(x)[:1], n, axis=0)

        return CrowdStates(rep(executed.robot), rep(executed.persons), particles.curious, rep(executed.tracked),
                           rep(executed.prev_dist), rep(executed.last_code), rep(executed.terminal))

    def reconcile_device(self, belief, executed: CrowdStates):
        """reconcile_belief on a device-resident belief: every particle record takes the
        executed state's observable fields and keeps its own curious bits (one broadcast
        kernel, vp_broadcast_record); weights are unchanged."""
        import torch

        from .. import _lib
        from ._device import CROWD_DTYPE

        dm = self.device_descriptor()
        src = torch.from_numpy(dm.pack(executed.take([0])).view(np.uint8).reshape(-1).copy()).cuda()
        lo = CROWD_DTYPE.fields["curious"][1]
        hi = lo + CROWD_DTYPE.fields["curious"][0].itemsize
        _lib.call("vp_broadcast_record", belief.records.data_ptr(), belief.m, dm.state_bytes, src.data_ptr(), lo, hi,
                  torch.cuda.current_stream().cuda_stream)
        return belief

    # -- device pieces
    def step_batch(self, states, actions, rng):
        return self.device_descriptor().step(states, actions, rng)

    def value_heuristic(self, states) -> np.ndarray:
        return self.device_descriptor().heuristic(states)

    def observation_log_likelihood(self, nxt, action: int, observation: int) -> np.ndarray:
        """Deterministic sensor (host SIR path): 0 where the state emitted the code, else -inf."""
        if not 0 <= observation <= self.spec.terminal_obs:
            raise ValueError("invalid observation code")
        out = np.full(len(nxt), -np.inf)
        if observation == self.spec.terminal_obs:
            out[nxt.terminal] = 0.0
        else:
            out[~nxt.terminal & (nxt.last_code == observation)] = 0.0
        return out

    def step_metrics(self, states, action: int, result) -> dict:
        """crowdnav.py:226-241 on the executed row."""
        moved = float(np.linalg.norm(result.next_states.robot[0] - states.robot[0]))
        nearest = self._distances(result.next_states.robot[:1], result.next_states.persons[:1]).min()
        return {"path_length": moved, "yells": float(action == YELL), "bumps": float(nearest < self.collision_radius)}
