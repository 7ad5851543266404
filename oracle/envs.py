"""Problem models (oracle -- test infrastructure only).

* ``ProblemSpec`` / ``ProblemModel`` defaults restate
  /root/reference/pkg/src/vecpomdp/core.py:29-142.
* ``MarsModel`` restates envs/mars.py:44-257 (the reference's RockSample
  family: two agents, m rocks, |A| = (5+m)^2, 9 observation codes + TERMINAL).
* ``TabularModel`` / ``tiger_model`` restate envs/tabular.py:19-190.
* ``SyntheticModel`` and ``LightDarkModel`` are NEW (BASELINE configs 5 and 4
  name problems the reference does not ship).  They follow the ProblemModel
  contract and the absorbing-terminal convention (core.py:1-14) so the
  reference solver itself can plan on them; the device models in
  ``paper_2510_27191_b200/csrc/models.cuh`` are checked against these.
  Synthetic uses only integer hashing and exactly-rounded fp64 ops, so its
  device step is bit-identical; Light-Dark's Box-Muller noise goes through
  log/cos (1-ulp library differences can move an observation bin only when
  the noisy position lies within ~1e-16 of a bin edge).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .rng import RowRng, mix64, to_unit, U64


# --------------------------------------------------------------------------- contract


@dataclass(frozen=True)
class ProblemSpec:
    """core.py:29-52; ``terminal_obs`` is one past the regular codes."""

    name: str
    action_count: int
    observation_arity: int
    discount: float
    max_steps: int

    def __post_init__(self):
        if self.action_count < 1:
            raise ValueError("action_count must be >= 1")
        if self.observation_arity < 1:
            raise ValueError("observation_arity must be >= 1")
        if not 0.0 < self.discount < 1.0:
            raise ValueError("discount must lie in (0, 1)")
        if self.max_steps < 1:
            raise ValueError("max_steps must be >= 1")

    @property
    def terminal_obs(self) -> int:
        return self.observation_arity


@dataclass
class StepResult:
    next_states: object
    observations: np.ndarray
    rewards: np.ndarray


def check_step_inputs(spec: ProblemSpec, states, actions):
    """core.py:73-81."""
    actions = np.asarray(actions)
    if len(actions) != len(states):
        raise ValueError(f"batch-length mismatch: {len(states)} states vs {len(actions)} actions")
    if actions.size and (actions.min() < 0 or actions.max() >= spec.action_count):
        raise ValueError("invalid action id in batch")


class ProblemModel:
    """Defaults of core.py:84-142."""

    spec: ProblemSpec

    def value_heuristic(self, states) -> np.ndarray:
        return np.zeros(len(states))

    def reference_log_probs(self) -> np.ndarray:
        n = self.spec.action_count
        return np.full(n, -np.log(n))

    def refresh_executed(self, executed):
        return executed

    def reconcile_belief(self, particles, executed):
        return particles

    def step_metrics(self, states, action, result) -> dict:
        return {}


# --------------------------------------------------------------------------- MARS


@dataclass
class MarsStates:
    x: np.ndarray        # (n, 2); x == grid size means departed
    y: np.ndarray        # (n, 2)
    rocks: np.ndarray    # (n, m) bool, True while good
    terminal: np.ndarray

    def __len__(self) -> int:
        return len(self.terminal)

    def take(self, idx) -> "MarsStates":
        i = np.asarray(idx, dtype=np.int64)
        return MarsStates(self.x[i], self.y[i], self.rocks[i], self.terminal[i])


GOOD, BAD, NULL = 0, 1, 2
_STEP_X = np.array([0, 1, 0, -1], dtype=np.int64)   # N, E, S, W (mars.py:22-24)
_STEP_Y = np.array([-1, 0, 1, 0], dtype=np.int64)


class MarsModel(ProblemModel):
    """Two-agent rock sampling (mars.py:44-257)."""

    def __init__(self, n: int = 20, m: int = 20, layout_seed: int = 0,
                 half_efficiency_distance: float = 20.0, discount: float = 0.983, max_steps: int = 90):
        if n < 2 or m < 1:
            raise ValueError("need a grid of at least 2 and at least one rock")
        self.n, self.m = n, m
        self.half_efficiency_distance = half_efficiency_distance
        # rock cells: the m smallest hashed uniforms over the n*n cells (mars.py:63-66)
        u = RowRng.from_seed(layout_seed).derive(0).uniform(np.arange(n * n, dtype=np.int64))
        cells = np.argsort(u)[:m]
        self.rock_x = (cells % n).astype(np.int64)
        self.rock_y = (cells // n).astype(np.int64)
        self.rock_at = np.full((n, n), -1, dtype=np.int64)
        self.rock_at[self.rock_x, self.rock_y] = np.arange(m)
        self.start_x = np.array([0, 0], dtype=np.int64)
        self.start_y = np.array([n // 3, (2 * n) // 3], dtype=np.int64)
        self.per_agent_ops = 5 + m
        self.spec = ProblemSpec("mars", self.per_agent_ops ** 2, 9, discount, max_steps)

    def check_accuracy(self, dist):
        """0.5 (1 + 2^(-d/d0)) (mars.py:82-84)."""
        return 0.5 * (1.0 + 2.0 ** (-dist / self.half_efficiency_distance))

    def sample_initial_states(self, n: int, rng: RowRng) -> MarsStates:
        """Fair-coin rocks from derive(0).uniform(rows, m) (mars.py:86-93)."""
        if n < 1:
            raise ValueError("n must be >= 1")
        rocks = rng.derive(0).uniform(np.arange(n, dtype=np.int64), self.m) < 0.5
        return MarsStates(np.tile(self.start_x, (n, 1)), np.tile(self.start_y, (n, 1)),
                          rocks, np.zeros(n, dtype=bool))

    def step_batch(self, states: MarsStates, actions, rng) -> StepResult:
        """mars.py:146-180: moves (both agents), samples (agent 0 first),
        readings from post-sample rocks, TERMINAL when both departed,
        absorbing rows restored with reward 0."""
        check_step_inputs(self.spec, states, actions)
        act = np.asarray(actions, dtype=np.int64)
        cnt = len(states)
        ops = (act // self.per_agent_ops, act % self.per_agent_ops)
        x, y, rocks = states.x.copy(), states.y.copy(), states.rocks.copy()
        gone = states.x == self.n
        reward = np.zeros(cnt)
        for k in (0, 1):  # moves (mars.py:95-111)
            idx = np.flatnonzero(~gone[:, k] & (ops[k] < 4))
            if len(idx):
                o = ops[k][idx]
                nx = x[idx, k] + _STEP_X[o]
                ny = y[idx, k] + _STEP_Y[o]
                leaving = nx == self.n
                ok = leaving | ((nx >= 0) & (nx < self.n) & (ny >= 0) & (ny < self.n))
                x[idx, k] = np.where(ok, nx, x[idx, k])
                y[idx, k] = np.where(ok & ~leaving, ny, y[idx, k])
                part = np.zeros(cnt)
                part[idx[leaving]] += 10.0
                reward += part
        for k in (0, 1):  # samples (mars.py:113-127)
            part = np.zeros(cnt)
            idx = np.flatnonzero(~gone[:, k] & (ops[k] == 4))
            if len(idx):
                part[idx] = -10.0
                rock = self.rock_at[x[idx, k], y[idx, k]]
                on = rock >= 0
                hit, rk = idx[on], rock[on]
                good = rocks[hit, rk]
                part[hit[good]] = 10.0
                rocks[hit[good], rk[good]] = False
            reward += part
        reading = []
        for k in (0, 1):  # sensor readings (mars.py:129-144)
            u = rng.derive(k).uniform()
            code = np.full(cnt, NULL, dtype=np.int64)
            idx = np.flatnonzero(~gone[:, k] & (ops[k] >= 5))
            if len(idx):
                rk = ops[k][idx] - 5
                d = np.sqrt((x[idx, k] - self.rock_x[rk]) ** 2.0 + (y[idx, k] - self.rock_y[rk]) ** 2.0)
                right = u[idx] < self.check_accuracy(d)
                code[idx] = np.where(rocks[idx, rk] == right, GOOD, BAD)
            reading.append(code)
        obs = reading[0] * 3 + reading[1]
        term = states.terminal | ((x[:, 0] == self.n) & (x[:, 1] == self.n))
        obs[term] = self.spec.terminal_obs
        stay = states.terminal
        if stay.any():
            x[stay], y[stay], rocks[stay] = states.x[stay], states.y[stay], states.rocks[stay]
            reward[stay] = 0.0
        return StepResult(MarsStates(x, y, rocks, term), obs, reward)

    def observation_log_likelihood(self, nxt: MarsStates, action: int, observation: int) -> np.ndarray:
        """mars.py:182-221."""
        if not 0 <= observation <= self.spec.terminal_obs:
            raise ValueError("invalid observation code")
        cnt = len(nxt)
        out = np.full(cnt, -np.inf)
        term = nxt.terminal
        if observation == self.spec.terminal_obs:
            out[term] = 0.0
            return out
        ops = (action // self.per_agent_ops, action % self.per_agent_ops)
        want = (observation // 3, observation % 3)
        logp = np.zeros(cnt)
        for k in (0, 1):
            op = ops[k]
            if op >= 5:
                rk = op - 5
                d = np.sqrt((nxt.x[:, k] - self.rock_x[rk]) ** 2.0 + (nxt.y[:, k] - self.rock_y[rk]) ** 2.0)
                acc = self.check_accuracy(d)
                good = nxt.rocks[:, rk]
                if want[k] == GOOD:
                    p = np.where(good, acc, 1.0 - acc)
                elif want[k] == BAD:
                    p = np.where(good, 1.0 - acc, acc)
                else:
                    p = np.zeros(cnt)
                p = np.where(~(nxt.x[:, k] == self.n), p, 1.0 if want[k] == NULL else 0.0)
            else:
                p = np.full(cnt, 1.0 if want[k] == NULL else 0.0)
            with np.errstate(divide="ignore"):
                logp += np.log(p)
        out[~term] = logp[~term]
        return out

    def value_heuristic(self, s: MarsStates) -> np.ndarray:
        """Exit bonus per active agent + nearest-agent discounted good rocks
        (mars.py:223-243)."""
        g = self.spec.discount
        h = np.zeros(len(s))
        active = s.x < self.n
        for k in (0, 1):
            h += np.where(active[:, k], 10.0 * g ** (self.n - s.x[:, k] - 1).astype(np.float64), 0.0)
        dist = np.abs(s.x[:, :, None] - self.rock_x[None, None, :]) + np.abs(s.y[:, :, None] - self.rock_y[None, None, :])
        dist = np.where(active[:, :, None], dist, np.iinfo(np.int64).max // 2)
        near = dist.min(axis=1).astype(np.float64)
        h += np.where(active.any(axis=1), (s.rocks * 10.0 * g ** near).sum(axis=1), 0.0)
        h[s.terminal] = 0.0
        return h

    def step_metrics(self, states: MarsStates, action: int, result) -> dict:
        ops = (action // self.per_agent_ops, action % self.per_agent_ops)
        good = bad = 0
        rocks = states.rocks[0].copy()
        for k in (0, 1):
            if ops[k] == 4 and states.x[0, k] < self.n and not states.terminal[0]:
                rk = self.rock_at[states.x[0, k], states.y[0, k]]
                if rk >= 0 and rocks[rk]:
                    good += 1
                    rocks[rk] = False
                else:
                    bad += 1
        return {"rocks_good": float(good), "rocks_bad": float(bad)}


# --------------------------------------------------------------------------- tabular


@dataclass(frozen=True)
class TabularPOMDP:
    """T[a, s, s'], Z[a, s', o], R[s, a] (tabular.py:19-63)."""

    transitions: np.ndarray
    observations: np.ndarray
    rewards: np.ndarray
    initial_belief: np.ndarray
    discount: float
    terminal_states: np.ndarray
    name: str = "tabular"
    max_steps: int = 100

    def __post_init__(self):
        t = np.asarray(self.transitions, dtype=np.float64)
        z = np.asarray(self.observations, dtype=np.float64)
        r = np.asarray(self.rewards, dtype=np.float64)
        b0 = np.asarray(self.initial_belief, dtype=np.float64)
        term = np.asarray(self.terminal_states, dtype=bool)
        na, ns, ns2 = t.shape
        if ns != ns2 or z.shape[0] != na or z.shape[1] != ns or r.shape != (ns, na):
            raise ValueError("inconsistent matrix shapes")
        if not np.allclose(t.sum(axis=2), 1.0, atol=1e-9):
            raise ValueError("transition rows must sum to 1")
        if not np.allclose(z.sum(axis=2), 1.0, atol=1e-9):
            raise ValueError("observation rows must sum to 1")
        if abs(b0.sum() - 1.0) > 1e-9 or b0.shape != (ns,):
            raise ValueError("initial belief must be a distribution over states")
        for name, val in (("transitions", t), ("observations", z), ("rewards", r),
                          ("initial_belief", b0), ("terminal_states", term)):
            object.__setattr__(self, name, val)

    n_states = property(lambda s: s.transitions.shape[1])
    n_actions = property(lambda s: s.transitions.shape[0])
    n_observations = property(lambda s: s.observations.shape[2])


@dataclass
class TabularStates:
    idx: np.ndarray
    terminal: np.ndarray

    def __len__(self) -> int:
        return len(self.idx)

    def take(self, indices) -> "TabularStates":
        i = np.asarray(indices, dtype=np.int64)
        return TabularStates(self.idx[i], self.terminal[i])


class TabularModel(ProblemModel):
    """Inverse-CDF stepping on cumsum(T) and cumsum(Z) (tabular.py:79-145)."""

    def __init__(self, pomdp: TabularPOMDP):
        self.pomdp = pomdp
        self.spec = ProblemSpec(pomdp.name, pomdp.n_actions, pomdp.n_observations, pomdp.discount, pomdp.max_steps)
        self._cum_t = np.cumsum(pomdp.transitions, axis=2)
        self._cum_z = np.cumsum(pomdp.observations, axis=2)
        with np.errstate(divide="ignore"):
            self._log_z = np.log(pomdp.observations)

    def states_from_indices(self, idx) -> TabularStates:
        i = np.asarray(idx, dtype=np.int64)
        return TabularStates(i, self.pomdp.terminal_states[i])

    def sample_initial_states(self, n: int, rng: RowRng) -> TabularStates:
        if n < 1:
            raise ValueError("n must be >= 1")
        u = rng.uniform(np.arange(n, dtype=np.int64))
        cum = np.cumsum(self.pomdp.initial_belief)
        return self.states_from_indices(np.minimum(np.searchsorted(cum, u, side="right"), len(cum) - 1))

    def step_batch(self, states: TabularStates, actions, rng) -> StepResult:
        check_step_inputs(self.spec, states, actions)
        act = np.asarray(actions, dtype=np.int64)
        s = states.idx
        u_s = rng.derive(0).uniform()
        nxt = np.minimum((self._cum_t[act, s] < u_s[:, None]).sum(axis=1), self.pomdp.n_states - 1)
        u_o = rng.derive(1).uniform()
        obs = np.minimum((self._cum_z[act, nxt] < u_o[:, None]).sum(axis=1),
                         self.pomdp.n_observations - 1).astype(np.int64)
        rew = self.pomdp.rewards[s, act].astype(np.float64)
        term = self.pomdp.terminal_states[nxt] | states.terminal
        obs[term] = self.spec.terminal_obs
        stay = states.terminal
        nxt = np.where(stay, s, nxt)
        rew[stay] = 0.0
        return StepResult(TabularStates(nxt, term), obs, rew)

    def observation_log_likelihood(self, nxt: TabularStates, action: int, observation: int) -> np.ndarray:
        if not 0 <= observation <= self.spec.terminal_obs:
            raise ValueError("invalid observation code")
        out = np.full(len(nxt), -np.inf)
        if observation == self.spec.terminal_obs:
            out[nxt.terminal] = 0.0
        else:
            live = ~nxt.terminal
            out[live] = self._log_z[action, nxt.idx[live], observation]
        return out


def tiger_model(listen_accuracy=0.85, reward_open_correct=10.0, reward_open_wrong=-100.0,
                reward_listen=-1.0, discount=0.95, max_steps=100) -> TabularModel:
    """Classic Tiger (tabular.py:148-190): 0 = listen, 1 = open left, 2 = open right."""
    acc = listen_accuracy
    t = np.zeros((3, 3, 3))
    t[0] = np.eye(3)
    t[1, :, 2] = 1.0
    t[2, :, 2] = 1.0
    z = np.zeros((3, 3, 2))
    z[0, 0] = (acc, 1 - acc)
    z[0, 1] = (1 - acc, acc)
    z[0, 2] = (0.5, 0.5)
    z[1:, :, :] = 0.5
    r = np.zeros((3, 3))
    r[0, 0] = r[1, 0] = reward_listen
    r[0, 1] = reward_open_wrong
    r[0, 2] = reward_open_correct
    r[1, 1] = reward_open_correct
    r[1, 2] = reward_open_wrong
    return TabularModel(TabularPOMDP(t, z, r, np.array([0.5, 0.5, 0.0]), discount,
                                     np.array([False, False, True]), "tiger", max_steps))


# --------------------------------------------------------------------------- Synthetic (NEW)

K_ACT = U64(0xD1B54A32D192ED03)
K_BRANCH = U64(0xABC98388FB8FAC03)
K_REWARD = U64(0x8CB92BA72F3D8DD7)
K_HEUR = U64(0x9FB21C651E98DF25)


@dataclass
class SyntheticStates:
    word: np.ndarray      # uint64 hidden state
    terminal: np.ndarray

    def __len__(self) -> int:
        return len(self.terminal)

    def take(self, idx) -> "SyntheticStates":
        i = np.asarray(idx, dtype=np.int64)
        return SyntheticStates(self.word[i], self.terminal[i])


class SyntheticModel(ProblemModel):
    """Integer-hash POMDP for the depth x width scaling sweep (BASELINE config 5).

    Hidden state is one 64-bit word.  With uniforms u_t, u_o, u_n from the
    model stream's derive(0/1/2):

        branch  = floor(u_t * branching)
        s'      = F(s + (a+1)*K_ACT + branch*K_BRANCH + salt)
        r       = 2 * unit(F(s ^ (a*K_REWARD + salt))) - 1          in [-1, 1)
        o       = (s' >> 17) % |O|   if u_o < obs_accuracy
                  min(floor(u_n * |O|), |O|-1)  otherwise
        term'   = term | ((s' >> 40) % 1000 < term_per_mille)
        h(s)    = 0.5 * unit(F(s + K_HEUR))  (0 on terminal)

    F = SplitMix64 finaliser, unit(h) = (h >> 11) * 2**-53, salt = F(seed + PHI).
    All operations are integer or exactly-rounded fp64, so a device port is
    bit-identical.
    """

    def __init__(self, n_actions: int = 16, n_obs: int = 8, branching: int = 4,
                 obs_accuracy: float = 0.8, term_per_mille: int = 10, seed: int = 0,
                 discount: float = 0.95, max_steps: int = 100):
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

    def sample_initial_states(self, n: int, rng: RowRng) -> SyntheticStates:
        if n < 1:
            raise ValueError("n must be >= 1")
        u = rng.derive(0).uniform(np.arange(n, dtype=np.int64))
        with np.errstate(over="ignore"):
            word = mix64((u * 2.0 ** 53).astype(U64) ^ self.salt)
        return SyntheticStates(word, np.zeros(n, dtype=bool))

    def step_batch(self, states: SyntheticStates, actions, rng) -> StepResult:
        check_step_inputs(self.spec, states, actions)
        act = np.asarray(actions, dtype=np.int64).astype(U64)
        s = states.word
        u_t = rng.derive(0).uniform()
        u_o = rng.derive(1).uniform()
        u_n = rng.derive(2).uniform()
        branch = np.floor(u_t * self.branching).astype(np.int64).astype(U64)
        with np.errstate(over="ignore"):
            nxt = mix64(s + (act + U64(1)) * K_ACT + branch * K_BRANCH + self.salt)
            rew = to_unit(mix64(s ^ (act * K_REWARD + self.salt))) * 2.0 - 1.0
        true_obs = ((nxt >> U64(17)) % U64(self.n_obs)).astype(np.int64)
        noise = np.minimum(np.floor(u_n * self.n_obs).astype(np.int64), self.n_obs - 1)
        obs = np.where(u_o < self.obs_accuracy, true_obs, noise)
        term = states.terminal | (((nxt >> U64(40)) % U64(1000)).astype(np.int64) < self.term_per_mille)
        obs[term] = self.spec.terminal_obs
        stay = states.terminal
        nxt = np.where(stay, s, nxt)
        rew[stay] = 0.0
        return StepResult(SyntheticStates(nxt, term), obs.astype(np.int64), rew)

    def value_heuristic(self, states: SyntheticStates) -> np.ndarray:
        with np.errstate(over="ignore"):
            h = 0.5 * to_unit(mix64(states.word + K_HEUR))
        h[states.terminal] = 0.0
        return h

    def observation_log_likelihood(self, nxt: SyntheticStates, action: int, observation: int) -> np.ndarray:
        if not 0 <= observation <= self.spec.terminal_obs:
            raise ValueError("invalid observation code")
        out = np.full(len(nxt), -np.inf)
        if observation == self.spec.terminal_obs:
            out[nxt.terminal] = 0.0
            return out
        true_obs = ((nxt.word >> U64(17)) % U64(self.n_obs)).astype(np.int64)
        # P(o) = acc * [o == true] + (1 - acc) * P(noise code == o)
        lo = np.ceil(observation / self.n_obs * 2 ** 53)  # exact bucket mass of floor(u*|O|)
        hi = np.ceil((observation + 1) / self.n_obs * 2 ** 53) if observation < self.n_obs - 1 else 2.0 ** 53
        p_noise = (hi - lo) * 2.0 ** -53
        p = self.obs_accuracy * (true_obs == observation) + (1.0 - self.obs_accuracy) * p_noise
        live = ~nxt.terminal
        with np.errstate(divide="ignore"):
            out[live] = np.log(p[live])
        return out


# --------------------------------------------------------------------------- Light-Dark (NEW)


@dataclass
class LightDarkStates:
    x: np.ndarray
    y: np.ndarray
    terminal: np.ndarray

    def __len__(self) -> int:
        return len(self.terminal)

    def take(self, idx) -> "LightDarkStates":
        i = np.asarray(idx, dtype=np.int64)
        return LightDarkStates(self.x[i], self.y[i], self.terminal[i])


# 8 compass moves then DECLARE (Light-Dark action set)
LD_DX = np.array([1, 1, 0, -1, -1, -1, 0, 1, 0], dtype=np.float64)
LD_DY = np.array([0, 1, 1, 1, 0, -1, -1, -1, 0], dtype=np.float64)
LD_DECLARE = 8


class LightDarkModel(ProblemModel):
    """2-D Light-Dark navigation with continuous observations (BASELINE config 4).

    State: position (x, y) in fp64.  Actions 0..7 move one ``step`` in the 8
    compass directions (reward -1); action 8 DECLAREs (reward +100 inside
    ``goal_radius`` of the origin, else -100) and terminates.  The observation
    is the next position plus Gaussian noise whose scale grows with the
    distance from the light column x = ``light_x``:

        sigma = sigma0 + sigma_slope * |x' - light_x|
        (ox, oy) = (x', y') + sigma * z,   z = rng.derive(0).normal(2)

    quantised per axis into ``bins`` cells of width ``bin_width`` centred on
    the origin and clipped at the border; the code is bx * bins + by (so
    |O| = bins^2, TERMINAL = bins^2).  Leaf heuristic: -(|x| + |y|).
    """

    def __init__(self, step: float = 1.0, light_x: float = 5.0, goal_radius: float = 1.0,
                 sigma0: float = 0.05, sigma_slope: float = 0.5, bin_width: float = 0.25,
                 bins: int = 64, discount: float = 0.95, max_steps: int = 60):
        if bins < 1 or bin_width <= 0:
            raise ValueError("need positive bins and bin width")
        self.step, self.light_x, self.goal_radius = float(step), float(light_x), float(goal_radius)
        self.sigma0, self.sigma_slope = float(sigma0), float(sigma_slope)
        self.bin_width, self.bins = float(bin_width), int(bins)
        self.spec = ProblemSpec("lightdark", 9, self.bins * self.bins, discount, max_steps)

    def sample_initial_states(self, n: int, rng: RowRng) -> LightDarkStates:
        """x ~ U[2, 6), y ~ U[-2, 2) from derive(0).uniform(rows, 2)."""
        if n < 1:
            raise ValueError("n must be >= 1")
        u = rng.derive(0).uniform(np.arange(n, dtype=np.int64), 2)
        return LightDarkStates(2.0 + 4.0 * u[:, 0], -2.0 + 4.0 * u[:, 1], np.zeros(n, dtype=bool))

    def _bin(self, v):
        b = np.floor(v / self.bin_width) + self.bins // 2
        return np.clip(b, 0, self.bins - 1).astype(np.int64)

    def step_batch(self, states: LightDarkStates, actions, rng) -> StepResult:
        check_step_inputs(self.spec, states, actions)
        act = np.asarray(actions, dtype=np.int64)
        nx = states.x + LD_DX[act] * self.step
        ny = states.y + LD_DY[act] * self.step
        declare = act == LD_DECLARE
        inside = states.x * states.x + states.y * states.y <= self.goal_radius * self.goal_radius
        rew = np.where(declare, np.where(inside, 100.0, -100.0), -1.0)
        z = rng.derive(0).normal(2)
        sigma = self.sigma0 + self.sigma_slope * np.abs(nx - self.light_x)
        obs = self._bin(nx + sigma * z[:, 0]) * self.bins + self._bin(ny + sigma * z[:, 1])
        term = states.terminal | declare
        obs[term] = self.spec.terminal_obs
        stay = states.terminal
        nx = np.where(stay, states.x, nx)
        ny = np.where(stay, states.y, ny)
        rew[stay] = 0.0
        return StepResult(LightDarkStates(nx, ny, term), obs.astype(np.int64), rew)

    def value_heuristic(self, s: LightDarkStates) -> np.ndarray:
        h = -(np.abs(s.x) + np.abs(s.y))
        h[s.terminal] = 0.0
        return h

    def observation_log_likelihood(self, nxt: LightDarkStates, action: int, observation: int) -> np.ndarray:
        """Bin mass of the Gaussian per axis (border bins absorb the tails)."""
        from math import erf, sqrt

        if not 0 <= observation <= self.spec.terminal_obs:
            raise ValueError("invalid observation code")
        out = np.full(len(nxt), -np.inf)
        if observation == self.spec.terminal_obs:
            out[nxt.terminal] = 0.0
            return out
        verf = np.vectorize(erf)
        sigma = self.sigma0 + self.sigma_slope * np.abs(nxt.x - self.light_x)

        def mass(center, b):
            lo = -np.inf if b == 0 else (b - self.bins // 2) * self.bin_width
            hi = np.inf if b == self.bins - 1 else (b + 1 - self.bins // 2) * self.bin_width
            cdf = lambda e: 0.5 * (1.0 + verf((e - center) / (sigma * sqrt(2.0))))
            return (1.0 if hi == np.inf else cdf(hi)) - (0.0 if lo == -np.inf else cdf(lo))

        p = mass(nxt.x, observation // self.bins) * mass(nxt.y, observation % self.bins)
        live = ~nxt.terminal
        with np.errstate(divide="ignore"):
            out[live] = np.log(p[live])
        return out


# --------------------------------------------------------------------------- Navigation


NAV_DEFAULT_MAP = "\n".join([
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
NAV_FREE, NAV_WALL, NAV_GATE, NAV_UNKNOWN = 0, 1, 2, 3
# neighbour / move order N, NE, E, SE, S, SW, W, NW; action 8 stays (navigation.py:42-47)
NAV_DR = np.array([-1, -1, 0, 1, 1, 1, 0, -1], dtype=np.int64)
NAV_DC = np.array([0, 1, 1, 1, 0, -1, -1, -1], dtype=np.int64)
NAV_STAY = 8


@dataclass
class NavStates:
    pos: np.ndarray        # flat cell, row * width + col
    occ: np.ndarray        # (n, n_unknown) occupancy of the unknown cells
    open_gate: np.ndarray  # which of the two gates is open
    terminal: np.ndarray

    def __len__(self) -> int:
        return len(self.pos)

    def take(self, idx) -> "NavStates":
        i = np.asarray(idx, dtype=np.int64)
        return NavStates(self.pos[i], self.occ[i], self.open_gate[i], self.terminal[i])


class NavigationModel(ProblemModel):
    """Grid navigation through a partially known obstacle field (navigation.py:1-251):
    hidden occupancy of the '?' cells and of which gate is open, an 8-bit noisy
    neighbour-occupancy reading per step, goal at the bottom."""

    def __init__(self, map_text: str = NAV_DEFAULT_MAP, p_obstacle: float = 0.25, sensor_accuracy: float = 0.9,
                 discount: float = 0.983, max_steps: int = 60):
        lines = [ln for ln in map_text.splitlines() if ln.strip()]
        self.height, self.width = len(lines), len(lines[0])
        if any(len(ln) != self.width for ln in lines):
            raise ValueError("map rows must have equal length")
        code = {"#": NAV_WALL, "|": NAV_GATE, "?": NAV_UNKNOWN, ".": NAV_FREE, "G": NAV_FREE}
        grid = np.array([[code.get(ch, -1) for ch in ln] for ln in lines], dtype=np.int64)
        if (grid < 0).any():
            raise ValueError("unknown map character")
        self.kind = grid.astype(np.int8)
        self.goal = np.array([[ch == "G" for ch in ln] for ln in lines])
        # per-cell index among the gates / among the unknown cells, in row-major order
        self.aux = np.full(grid.shape, -1, dtype=np.int64)
        for k in (NAV_GATE, NAV_UNKNOWN):
            cells = np.flatnonzero(grid.reshape(-1) == k)
            self.aux.reshape(-1)[cells] = np.arange(len(cells))
        self.n_gates = int((grid == NAV_GATE).sum())
        self.n_unknown = int((grid == NAV_UNKNOWN).sum())
        if self.n_gates != 2:
            raise ValueError("map must contain exactly two gates")
        self.start_cells = np.flatnonzero((grid[0] == NAV_FREE) & ~self.goal[0]).astype(np.int64)
        if not len(self.start_cells):
            raise ValueError("top border has no free start cells")
        self.p_obstacle, self.sensor_accuracy = p_obstacle, sensor_accuracy
        self.spec = ProblemSpec("navigation", 9, 256, discount, max_steps)
        self.goal_dist = self._goal_distances()

    def _goal_distances(self) -> np.ndarray:
        """8-connected BFS distance to the goal with walls blocking and gates / unknown
        cells optimistic (navigation.py:127-144)."""
        dist = np.full(self.kind.shape, np.inf)
        ring = [tuple(x) for x in np.argwhere(self.goal)]
        for r, c in ring:
            dist[r, c] = 0.0
        while ring:
            nxt = []
            for r, c in ring:
                for dr, dc in zip(NAV_DR, NAV_DC):
                    rr, cc = r + dr, c + dc
                    if 0 <= rr < self.height and 0 <= cc < self.width and self.kind[rr, cc] != NAV_WALL \
                            and dist[rr, cc] == np.inf:
                        dist[rr, cc] = dist[r, c] + 1
                        nxt.append((rr, cc))
            ring = nxt
        return dist

    def blocked(self, s: NavStates, r, c) -> np.ndarray:
        """Occupancy of target cells per row; off-map counts as occupied (navigation.py:146-162)."""
        off = (r < 0) | (r >= self.height) | (c < 0) | (c >= self.width)
        rr, cc = np.clip(r, 0, self.height - 1), np.clip(c, 0, self.width - 1)
        kind, aux = self.kind[rr, cc], self.aux[rr, cc]
        out = off | (kind == NAV_WALL) | (~off & (kind == NAV_GATE) & (aux != s.open_gate))
        unk = np.flatnonzero(~off & (kind == NAV_UNKNOWN))
        out[unk] |= s.occ[unk, aux[unk]]
        return out

    def neighbour_bits(self, s: NavStates) -> np.ndarray:
        r, c = s.pos // self.width, s.pos % self.width
        return np.stack([self.blocked(s, r + NAV_DR[i], c + NAV_DC[i]) for i in range(8)], axis=1)

    def sample_initial_states(self, n: int, rng: RowRng) -> NavStates:
        if n < 1:
            raise ValueError("n must be >= 1")
        rows = np.arange(n, dtype=np.int64)
        pos = self.start_cells[(rng.derive(0).uniform(rows) * len(self.start_cells)).astype(np.int64)]
        occ = rng.derive(1).uniform(rows, self.n_unknown) < self.p_obstacle
        gate = (rng.derive(2).uniform(rows) < 0.5).astype(np.int64)
        return NavStates(pos, occ, gate, np.zeros(n, dtype=bool))

    def step_batch(self, s: NavStates, actions, rng) -> StepResult:
        """navigation.py:172-213."""
        check_step_inputs(self.spec, s, actions)
        a = np.asarray(actions, dtype=np.int64)
        r, c = s.pos // self.width, s.pos % self.width
        move = a != NAV_STAY
        k = np.minimum(a, 7)
        tr = np.where(move, r + NAV_DR[k], r)
        tc = np.where(move, c + NAV_DC[k], c)
        hit = move & self.blocked(s, tr, tc)
        nr, nc = np.where(hit, r, tr), np.where(hit, c, tc)
        goal = self.goal[nr, nc] & move & ~hit
        rew = np.where(goal, 20.0, np.where(hit, -1.1, np.where(move, -0.1, -0.3)))
        term = s.terminal | goal
        nxt = NavStates(nr * self.width + nc, s.occ.copy(), s.open_gate.copy(), term)
        flips = rng.derive(0).uniform(8) >= self.sensor_accuracy
        obs = ((self.neighbour_bits(nxt) ^ flips) @ (1 << np.arange(8, dtype=np.int64))).astype(np.int64)
        obs[term] = self.spec.terminal_obs
        nxt.pos[s.terminal] = s.pos[s.terminal]
        rew = np.where(s.terminal, 0.0, rew)
        return StepResult(nxt, obs, rew)

    def observation_log_likelihood(self, nxt: NavStates, action: int, observation: int) -> np.ndarray:
        """matches * log(acc) + misses * log(1 - acc) over the 8 bits (navigation.py:215-239)."""
        if not 0 <= observation <= self.spec.terminal_obs:
            raise ValueError("invalid observation code")
        out = np.full(len(nxt), -np.inf)
        if observation == self.spec.terminal_obs:
            out[nxt.terminal] = 0.0
            return out
        want = ((observation >> np.arange(8)) & 1).astype(bool)
        live = ~nxt.terminal
        hits = (self.neighbour_bits(nxt) == want).sum(axis=1)[live]
        miss = 8 - hits
        with np.errstate(divide="ignore", invalid="ignore"):
            out[live] = hits * np.log(self.sensor_accuracy) + np.where(
                miss > 0, miss * np.log(1.0 - self.sensor_accuracy), 0.0)
        return out

    def value_heuristic(self, s: NavStates) -> np.ndarray:
        """Discounted goal bonus minus step costs at the optimistic distance (navigation.py:241-251)."""
        g = self.spec.discount
        d = np.maximum(self.goal_dist[s.pos // self.width, s.pos % self.width] - 1.0, 0.0)
        decay = g ** d
        h = 20.0 * decay - 0.1 * (1.0 - decay) / (1.0 - g)
        h[s.terminal] = 0.0
        return h


# --------------------------------------------------------------------------- CrowdNav

CROWD_DIRS = np.array([(0.0, 1.0), (1.0, 0.0), (0.0, -1.0), (-1.0, 0.0), (0.0, 0.0)])  # N E S W YELL
CROWD_YELL = 4


@dataclass
class CrowdStates:
    robot: np.ndarray      # (n, 2) float64 metres
    persons: np.ndarray    # (n, p, 2) float32 metres
    curious: np.ndarray    # (n, p) hidden traits
    tracked: np.ndarray    # (n, k) persons the sensor watches
    prev_dist: np.ndarray  # (n, k) their distances at the previous step
    last_code: np.ndarray  # (n,) observation emitted on entering the state
    terminal: np.ndarray

    def __len__(self) -> int:
        return len(self.robot)

    def take(self, idx) -> "CrowdStates":
        i = np.asarray(idx, dtype=np.int64)
        return CrowdStates(self.robot[i], self.persons[i], self.curious[i], self.tracked[i], self.prev_dist[i],
                           self.last_code[i], self.terminal[i])


class CrowdNavModel(ProblemModel):
    """Robot crossing a hall among a reactive crowd (crowdnav.py:1-241): hidden curious / shy
    traits, every person jitters, nearby people react; the observation is one bit per
    tracked person telling whether it closed distance."""

    def __init__(self, p_curious: float = 0.5, n_people: int = 300, n_tracked: int = 6, hall_width: float = 50.0,
                 hall_depth: float = 40.0, motion_noise: float = 0.05, react_prob: float = 0.9,
                 r_nearby: float = 4.0, v_curious: float = 0.3, v_shy: float = 0.8, v_back: float = 2.0,
                 collision_radius: float = 0.5, discount: float = 0.97, max_steps: int = 200):
        if not 0.0 <= p_curious <= 1.0:
            raise ValueError("p_curious must be in [0, 1]")
        self.p_curious, self.n_people, self.n_tracked = p_curious, n_people, n_tracked
        self.hall = np.array([hall_width, hall_depth])
        self.motion_noise, self.react_prob, self.r_nearby = motion_noise, react_prob, r_nearby
        self.v_curious, self.v_shy, self.v_back = v_curious, v_shy, v_back
        self.collision_radius = collision_radius
        self.spec = ProblemSpec("crowdnav", 5, 2 ** n_tracked, discount, max_steps)

    @staticmethod
    def _dist(persons, robot) -> np.ndarray:
        d = persons.astype(np.float64) - robot[:, None, :]
        return np.sqrt((d ** 2).sum(axis=2))

    def _track(self, robot, persons):
        dist = self._dist(persons, robot)
        tracked = np.argsort(dist, axis=1)[:, : self.n_tracked].astype(np.int64)
        return tracked, np.take_along_axis(dist, tracked, axis=1)

    def sample_initial_states(self, n: int, rng: RowRng) -> CrowdStates:
        if n < 1:
            raise ValueError("n must be >= 1")
        rows = np.arange(n, dtype=np.int64)
        robot = np.tile(np.array([self.hall[0] / 2.0, 0.0]), (n, 1))
        u = rng.derive(0).uniform(rows, self.n_people * 2).reshape(n, self.n_people, 2)
        persons = (u * self.hall).astype(np.float32)
        curious = rng.derive(1).uniform(rows, self.n_people) < self.p_curious
        tracked, prev = self._track(robot, persons)
        return CrowdStates(robot, persons, curious, tracked, prev, np.zeros(n, dtype=np.int64), np.zeros(n, dtype=bool))

    def step_batch(self, s: CrowdStates, actions, rng) -> StepResult:
        """crowdnav.py:120-186."""
        check_step_inputs(self.spec, s, actions)
        a = np.asarray(actions, dtype=np.int64)
        n, p = len(s), self.n_people
        robot = s.robot + CROWD_DIRS[a]
        entered = robot[:, 1] >= self.hall[1]
        robot = np.stack([np.clip(robot[:, 0], 0.0, self.hall[0]), np.clip(robot[:, 1], 0.0, self.hall[1])], axis=1)
        people = s.persons.astype(np.float64) + rng.derive(0).normal(p * 2).reshape(n, p, 2) * self.motion_noise
        diff = robot[:, None, :] - people
        dist = np.sqrt((diff ** 2).sum(axis=2))
        react = (dist < self.r_nearby) & (dist > 1e-9) & (rng.derive(1).uniform(p) < self.react_prob)
        unit = diff / np.maximum(dist, 1e-9)[:, :, None]
        speed = np.where(s.curious, self.v_curious, -self.v_shy)
        speed = np.where((a == CROWD_YELL)[:, None], -self.v_back, speed)
        people = people + react[:, :, None] * speed[:, :, None] * unit
        people[:, :, 0] = np.clip(people[:, :, 0], 0.0, self.hall[0])
        people[:, :, 1] = np.clip(people[:, :, 1], 0.0, self.hall[1])
        people = people.astype(np.float32)
        new_dist = self._dist(people, robot)
        bumped = (new_dist < self.collision_radius).any(axis=1)
        rew = -1.0 - 25.0 * (a == CROWD_YELL) - 200.0 * bumped + 1000.0 * entered
        tdist = np.take_along_axis(new_dist, s.tracked, axis=1)
        code = ((tdist < s.prev_dist) @ (1 << np.arange(self.n_tracked, dtype=np.int64))).astype(np.int64)
        term = s.terminal | entered
        obs = np.where(term, self.spec.terminal_obs, code)
        nxt = CrowdStates(robot, people, s.curious.copy(), s.tracked.copy(), tdist, code, term)
        old = s.terminal
        if old.any():
            nxt.robot[old], nxt.persons[old] = s.robot[old], s.persons[old]
            nxt.prev_dist[old], nxt.last_code[old] = s.prev_dist[old], s.last_code[old]
            rew = np.where(old, 0.0, rew)
        return StepResult(nxt, obs, rew)

    def observation_log_likelihood(self, nxt: CrowdStates, action: int, observation: int) -> np.ndarray:
        """Deterministic observation: 0 where the state emitted it, -inf elsewhere (crowdnav.py:188-201)."""
        if not 0 <= observation <= self.spec.terminal_obs:
            raise ValueError("invalid observation code")
        out = np.full(len(nxt), -np.inf)
        if observation == self.spec.terminal_obs:
            out[nxt.terminal] = 0.0
        else:
            out[~nxt.terminal & (nxt.last_code == observation)] = 0.0
        return out

    def value_heuristic(self, s: CrowdStates) -> np.ndarray:
        g = self.spec.discount
        decay = g ** np.maximum(np.ceil(self.hall[1] - s.robot[:, 1]) - 1.0, 0.0)
        h = 1000.0 * decay - (1.0 - decay) / (1.0 - g)
        h[s.terminal] = 0.0
        return h

    def refresh_executed(self, executed: CrowdStates) -> CrowdStates:
        tracked, prev = self._track(executed.robot, executed.persons)
        return CrowdStates(executed.robot, executed.persons, executed.curious, tracked, prev, executed.last_code,
                           executed.terminal)

    def reconcile_belief(self, particles: CrowdStates, executed: CrowdStates) -> CrowdStates:
        n = len(particles)
        rep = lambda x: np.repeat(x, n, axis=0)  # noqa: E731
        return CrowdStates(rep(executed.robot), rep(executed.persons), particles.curious, rep(executed.tracked),
                           rep(executed.prev_dist), rep(executed.last_code), rep(executed.terminal))
