"""Example ``CudaModel`` plug-ins (plugin.py): user ProblemModels written as CUDA.

* ``tabular_cuda_model(pomdp)`` -- any TabularPOMDP as a plug-in: its tables are uploaded
  to HBM once (``CudaModel(tables=...)``) and reached through pointers in ``Params``.  It restates
  envs/tabular.py:106-145 (the reference's TabularModel) operation for operation, so
  its plans equal the reference's trees bit for bit -- the plug-in path's parity check.
* ``corridor_cuda_model(length)`` -- a model that exists only as a plug-in: a robot in
  a 1-D corridor of unknown length-position with a noisy continuous range sensor
  (Gaussian, binned), reward at the door.  Shows floating-point states, normal draws
  and a non-trivial heuristic / observation likelihood.
"""

from __future__ import annotations

import numpy as np

from ..core import ProblemSpec
from ..plugin import CudaModel

TABULAR_SOURCE = r"""
// A TabularPOMDP of any size (envs/tabular.py:106-145); the tables live in HBM (CudaModel tables=).
struct Params {
  int32_t S, A, O, pad;
  const double* cum_t;      // [a][s][s'] cumulative transition rows
  const double* cum_z;      // [a][s'][o] cumulative observation rows
  const double* log_z;      // [a][s'][o] log Z
  const double* reward;     // [s][a]
  const int32_t* terminal;  // [s]
};
struct State {
  int32_t idx;
  int32_t terminal;
};
__device__ void step(const Params& P, State& s, int a, const RowDraws& rng, uint32_t& obs, double& reward) {
  const double us = rng.uniform(0);             // rng.derive(0).uniform()
  const double* ct = P.cum_t + ((size_t)a * P.S + s.idx) * P.S;
  int nxt = 0;
  for (int j = 0; j < P.S; ++j) nxt += ct[j] < us;
  nxt = nxt < P.S - 1 ? nxt : P.S - 1;
  const double uo = rng.uniform(1);             // rng.derive(1).uniform()
  const double* cz = P.cum_z + ((size_t)a * P.S + nxt) * P.O;
  int o = 0;
  for (int j = 0; j < P.O; ++j) o += cz[j] < uo;
  o = o < P.O - 1 ? o : P.O - 1;
  reward = P.reward[(size_t)s.idx * P.A + a];
  const bool term = P.terminal[nxt] || s.terminal;
  obs = term ? (uint32_t)P.O : (uint32_t)o;     // the terminal observation code is |O|
  if (s.terminal) {                             // absorbing
    reward = 0.0;
    return;
  }
  s.idx = nxt;
  s.terminal = term ? 1 : 0;
}
__device__ double heuristic(const Params&, const State&) { return 0.0; }
__device__ double obs_log_likelihood(const Params& P, const State& s, int a, uint32_t obs) {
  if (obs == (uint32_t)P.O) return s.terminal ? 0.0 : -INFINITY;
  if (s.terminal) return -INFINITY;
  return P.log_z[((size_t)a * P.S + s.idx) * P.O + obs];
}
"""

TAB_STATE = np.dtype([("idx", "<i4"), ("terminal", "<i4")])
TAB_PARAMS = np.dtype([("S", "<i4"), ("A", "<i4"), ("O", "<i4"), ("pad", "<i4"), ("cum_t", "<u8"), ("cum_z", "<u8"),
                       ("log_z", "<u8"), ("reward", "<u8"), ("terminal", "<u8")])


def tabular_cuda_model(pomdp) -> CudaModel:
    """A plug-in CudaModel of a TabularPOMDP (the reference's or ours), any size."""
    t = np.asarray(pomdp.transitions, dtype=np.float64)
    z = np.asarray(pomdp.observations, dtype=np.float64)
    A, S, O = t.shape[0], t.shape[1], z.shape[2]
    p = np.zeros((), dtype=TAB_PARAMS)
    p["S"], p["A"], p["O"] = S, A, O
    with np.errstate(divide="ignore"):
        log_z = np.log(z)
    term = np.asarray(pomdp.terminal_states, dtype=bool)
    tables = {"cum_t": np.cumsum(t, axis=2).reshape(-1), "cum_z": np.cumsum(z, axis=2).reshape(-1),
              "log_z": log_z.reshape(-1), "reward": np.asarray(pomdp.rewards, dtype=np.float64).reshape(-1),
              "terminal": term.astype(np.int32)}
    init = np.cumsum(np.asarray(pomdp.initial_belief, dtype=np.float64))

    def initial_states(n, rng):  # tabular.py sample_initial_states
        u = rng.uniform(np.arange(n, dtype=np.int64))
        idx = np.minimum(np.searchsorted(init, u, side="right"), len(init) - 1)
        out = np.zeros(n, dtype=TAB_STATE)
        out["idx"], out["terminal"] = idx, term[idx]
        return out

    spec = ProblemSpec(f"{pomdp.name}-cuda", A, O, float(pomdp.discount), int(pomdp.max_steps))
    return CudaModel(spec, TAB_STATE, TABULAR_SOURCE, p, initial_states=initial_states, tables=tables)


CORRIDOR_SOURCE = r"""
// 1-D corridor: position x in [0, L), door at L - 1.  Actions: 0 left, 1 right, 2 open door.
// Motion noise N(0, 0.1) per move; the range sensor reads the distance to the door plus
// N(0, sigma) noise, binned into nbins bins of width bin_w.
struct Params {
  double length, sigma, bin_w, move_noise;
  int32_t nbins, pad;
};
struct State {
  double x;
  int32_t terminal, pad;
};
__device__ int bin_of(const Params& P, double d) {
  int b = (int)floor(d / P.bin_w);
  return b < 0 ? 0 : (b >= P.nbins ? P.nbins - 1 : b);
}
__device__ void step(const Params& P, State& s, int a, const RowDraws& rng, uint32_t& obs, double& reward) {
  if (s.terminal) { obs = (uint32_t)P.nbins; reward = 0.0; return; }
  if (a == 2) {                                     // open: +10 at the door, -5 elsewhere; ends
    const bool at_door = fabs(s.x - (P.length - 1.0)) < 0.5;
    reward = at_door ? 10.0 : -5.0;
    s.terminal = 1;
    obs = (uint32_t)P.nbins;
    return;
  }
  const double dx = (a == 1 ? 1.0 : -1.0) + P.move_noise * rng.normal(0);
  s.x = fmin(fmax(s.x + dx, 0.0), P.length - 1.0);
  reward = -0.1;
  const double reading = (P.length - 1.0 - s.x) + P.sigma * rng.normal(1);
  obs = (uint32_t)bin_of(P, reading);
}
__device__ double heuristic(const Params& P, const State& s) {
  return s.terminal ? 0.0 : 10.0 * pow(0.95, fabs(P.length - 1.0 - s.x));
}
__device__ double obs_log_likelihood(const Params& P, const State& s, int, uint32_t obs) {
  if (obs == (uint32_t)P.nbins) return s.terminal ? 0.0 : -INFINITY;
  if (s.terminal) return -INFINITY;
  // mass of the reading's bin under N(distance, sigma); the end bins are open
  const double mu = P.length - 1.0 - s.x, k = 1.0 / (P.sigma * sqrt(2.0));
  const double lo = obs == 0 ? -INFINITY : obs * P.bin_w, hi = (int)obs == P.nbins - 1 ? INFINITY : (obs + 1) * P.bin_w;
  const double m = 0.5 * (erf((hi - mu) * k) - erf((lo - mu) * k));
  return m > 0.0 ? log(m) : -INFINITY;
}
"""

CORRIDOR_STATE = np.dtype([("x", "<f8"), ("terminal", "<i4"), ("pad", "<i4")])
CORRIDOR_PARAMS = np.dtype([("length", "<f8"), ("sigma", "<f8"), ("bin_w", "<f8"), ("move_noise", "<f8"),
                            ("nbins", "<i4"), ("pad", "<i4")])


def corridor_cuda_model(length: float = 20.0, sigma: float = 1.5, nbins: int = 16) -> CudaModel:
    p = np.zeros((), dtype=CORRIDOR_PARAMS)
    p["length"], p["sigma"], p["bin_w"], p["move_noise"], p["nbins"] = length, sigma, length / nbins, 0.1, nbins

    def initial_states(n, rng):  # x ~ U[0, L/2)
        out = np.zeros(n, dtype=CORRIDOR_STATE)
        out["x"] = rng.derive(0).uniform(np.arange(n, dtype=np.int64)) * (length / 2.0)
        return out

    spec = ProblemSpec("corridor-cuda", 3, nbins, 0.95, 60)
    return CudaModel(spec, CORRIDOR_STATE, CORRIDOR_SOURCE, p, initial_states=initial_states)


LEVELS_SOURCE = r"""
// "Levels": k hidden gauges (floats) drift with the action plus per-gauge Gaussian noise;
// the observation counts the gauges above 0, the reward is minus the gauges outside [-1, 1].
// A 520-byte record: the search steps it with a whole warp (VP_USER_COOP build, step_warp).
struct Params {
  int32_t k, horizon;
  double noise;
};
struct State {
  float level[128];
  int32_t t, terminal;
};
__device__ __forceinline__ double levels_delta(int a) { return a == 0 ? -0.5 : a == 1 ? -0.1 : a == 2 ? 0.1 : 0.5; }
__device__ __forceinline__ float levels_next(const Params& P, float v, int a, const RowDraws& rng, int i) {
  return (float)((double)v + levels_delta(a) + P.noise * rng.normal(0, (uint64_t)(i + 1)));
}
__device__ void step(const Params& P, State& s, int a, const RowDraws& rng, uint32_t& obs, double& reward) {
  if (s.terminal) { obs = (uint32_t)(P.k + 1); reward = 0.0; return; }
  int above = 0, out = 0;
  for (int i = 0; i < P.k; ++i) {
    const float v = levels_next(P, s.level[i], a, rng, i);
    s.level[i] = v;
    above += v > 0.0f;
    out += fabsf(v) > 1.0f;
  }
  s.t += 1;
  s.terminal = s.t >= P.horizon;
  reward = -(double)out;
  obs = s.terminal ? (uint32_t)(P.k + 1) : (uint32_t)above;
}
__device__ double heuristic(const Params& P, const State& s) {
  if (s.terminal) return 0.0;
  int out = 0;
  for (int i = 0; i < P.k; ++i) out += fabsf(s.level[i]) > 1.0f;
  return -0.5 * (double)out * (double)(P.horizon - s.t);
}
__device__ double obs_log_likelihood(const Params& P, const State& s, int, uint32_t obs) {
  if (obs == (uint32_t)(P.k + 1)) return s.terminal ? 0.0 : -INFINITY;
  if (s.terminal) return -INFINITY;
  int above = 0;
  for (int i = 0; i < P.k; ++i) above += s.level[i] > 0.0f;
  return (uint32_t)above == obs ? 0.0 : -INFINITY;
}
"""

LEVELS_COOP = r"""
#define VP_USER_COOP 1
""" + LEVELS_SOURCE + r"""
// the same step with the 32 lanes splitting the gauges (integer counts: any order is exact)
__device__ void step_warp(const Params& P, State& s, int a, const RowDraws& rng, bool, uint32_t& obs, double& reward) {
  const int lane = threadIdx.x & 31;
  const bool was_terminal = s.terminal;
  __syncwarp();
  if (was_terminal) { obs = (uint32_t)(P.k + 1); reward = 0.0; return; }
  int above = 0, out = 0;
  for (int i = lane; i < P.k; i += 32) {
    const float v = levels_next(P, s.level[i], a, rng, i);
    s.level[i] = v;
    above += v > 0.0f;
    out += fabsf(v) > 1.0f;
  }
  for (int o = 16; o; o >>= 1) {
    above += __shfl_xor_sync(0xffffffffu, above, o);
    out += __shfl_xor_sync(0xffffffffu, out, o);
  }
  __syncwarp();
  const int t = s.t + 1;
  const bool term = t >= P.horizon;
  if (lane == 0) { s.t = t; s.terminal = term; }
  __syncwarp();
  reward = -(double)out;
  obs = term ? (uint32_t)(P.k + 1) : (uint32_t)above;
}
"""

LEVELS_STATE = np.dtype([("level", "<f4", (128,)), ("t", "<i4"), ("terminal", "<i4")])
LEVELS_PARAMS = np.dtype([("k", "<i4"), ("horizon", "<i4"), ("noise", "<f8")])


def levels_cuda_model(k: int = 96, horizon: int = 20, noise: float = 0.3, coop: bool = True) -> CudaModel:
    """A large-record plug-in (520 B): ``coop`` builds the warp-cooperative form (one row per warp,
    the record in shared memory); ``coop=False`` the same dynamics one row per lane."""
    if not 1 <= k <= 128:
        raise ValueError("k must be in [1, 128]")
    p = np.zeros((), dtype=LEVELS_PARAMS)
    p["k"], p["horizon"], p["noise"] = k, horizon, noise

    def initial_states(n, rng):  # gauges ~ U[-1, 1)
        out = np.zeros(n, dtype=LEVELS_STATE)
        out["level"][:, :k] = (rng.derive(0).uniform(np.arange(n, dtype=np.int64), k) * 2.0 - 1.0).astype(np.float32)
        return out

    spec = ProblemSpec("levels-cuda", 4, k + 1, 0.95, horizon)
    return CudaModel(spec, LEVELS_STATE, LEVELS_COOP if coop else LEVELS_SOURCE, p, initial_states=initial_states)
