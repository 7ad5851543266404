"""Device descriptors (vp_model) and packed state records for problem models.

A ``DeviceModel`` binds one ProblemModel instance to:
* a ``VpModel`` ctypes struct (include/vpb200.h) with its constant tables
  uploaded to HBM (kept alive here);
* the packed per-row state record the kernels use (csrc/vp_models.cuh):

    MARS       16 B  {u8 x0, y0, x1, y1; u32 terminal; u64 rock bits}
    TABULAR     8 B  {i32 state index; i32 terminal}
    SYNTHETIC  16 B  {u64 word; u32 terminal; u32 pad}
    LIGHTDARK  24 B  {f64 x; f64 y; u32 terminal; u32 pad}
    NAVIGATION 24 B  {u64 occ[2]; i32 cell; u8 gate; u8 terminal; u16 pad}
    CROWDNAV 2704 B  {f64 robot[2]; f64 prev[8]; i32 code; u32 terminal; u16 tracked[8];
                      u32 curious bits[10]; f32 persons[320][2]}

Models are recognised either by a ``device_descriptor()`` method or, for
objects of the reference package (vecpomdp.envs.MarsModel / TabularModel),
by their public attributes, so the reference's own model objects plan on
the device unchanged.
"""

from __future__ import annotations

import ctypes as C
import weakref

import numpy as np

from .. import _lib
from ..core import check_step_inputs, StepResult
from ..rng import key_of, kind_of

MARS_DTYPE = np.dtype([("x0", "u1"), ("y0", "u1"), ("x1", "u1"), ("y1", "u1"), ("term", "<u4"), ("rocks", "<u8")])
TAB_DTYPE = np.dtype([("idx", "<i4"), ("term", "<i4")])
SYN_DTYPE = np.dtype([("word", "<u8"), ("term", "<u4"), ("pad", "<u4")])
LD_DTYPE = np.dtype([("x", "<f8"), ("y", "<f8"), ("term", "<u4"), ("pad", "<u4")])
NAV_DTYPE = np.dtype([("occ0", "<u8"), ("occ1", "<u8"), ("pos", "<i4"), ("gate", "u1"), ("term", "u1"),
                      ("pad", "<u2")])
CROWD_DTYPE = np.dtype([("robot", "<f8", (2,)), ("prev", "<f8", (8,)), ("code", "<i4"), ("term", "<u4"),
                        ("tracked", "<u2", (8,)), ("curious", "<u4", (10,)), ("persons", "<f4", (640,))])


def _torch():
    return _lib.torch_cuda()


class DeviceModel:
    """Descriptor + packer for one model instance."""

    def __init__(self, kind: int, spec, state_dtype: np.dtype, pack, unpack=None, pack_into=None):
        self.kind = kind
        self.spec = spec
        self.state_dtype = state_dtype
        self._pack = pack
        self._pack_into = pack_into
        self._unpack = unpack
        self.init_prefs_cache = {}  # eta -> initial PSI row (solver.initial_prefs)
        self.desc = _lib.VpModel()
        self.desc.kind = kind
        self.desc.action_count = spec.action_count
        self.desc.obs_arity = spec.observation_arity
        self.desc.state_bytes = state_dtype.itemsize
        self.desc.discount = float(spec.discount)
        self.tables = []  # device tensors referenced by desc
        self.lib = None  # the plug-in library of a CudaModel (plugin.py); None: the main library

    def call(self, name: str, *args):
        """A model-dependent entry point (vp_plan, vp_search, vp_sir_*, vp_model_*) on the library
        that carries this model."""
        _lib.call_on(self.lib, name, *args)

    @property
    def state_bytes(self) -> int:
        return self.state_dtype.itemsize

    def upload(self, arr: np.ndarray):
        torch = _torch()
        t = torch.from_numpy(np.ascontiguousarray(arr)).cuda()
        self.tables.append(t)
        return t.data_ptr()

    def pack(self, states) -> np.ndarray:
        return self._pack(states)

    def pack_into(self, states, dst: np.ndarray) -> int:
        """Pack ``states`` straight into the byte buffer ``dst`` (e.g. pinned host memory);
        returns the bytes written."""
        if self._pack_into is not None:
            return self._pack_into(states, dst)
        rec = self._pack(states)
        dst[: rec.nbytes] = rec.view(np.uint8).reshape(-1)
        return rec.nbytes

    def unpack(self, records: np.ndarray):
        if self._unpack is None:
            raise TypeError("this model's states cannot be rebuilt from device records")
        return self._unpack(records)

    def states_to_device(self, states):
        torch = _torch()
        rec = self.pack(states)
        return torch.from_numpy(rec.view(np.uint8).reshape(-1)).cuda()

    # -- device-backed ProblemModel pieces (used by the product model classes)
    def step(self, states, actions, rng):
        """step_batch on the device via vp_model_step (test hook + env step)."""
        torch = _torch()
        check_step_inputs(self.spec, states, actions)
        n = len(states)
        if n == 0:
            return StepResult(states, np.zeros(0, dtype=np.int64), np.zeros(0))
        st = self.states_to_device(states)
        acts = torch.as_tensor(np.asarray(actions, dtype=np.int32)).cuda()
        rows = torch.as_tensor(np.asarray(rng.rows, dtype=np.int64)).cuda()
        obs = torch.empty(n, dtype=torch.int32, device="cuda")
        rew = torch.empty(n, dtype=torch.float64, device="cuda")
        stream = torch.cuda.current_stream().cuda_stream
        self.desc.rng_kind = kind_of(rng)
        self.call("vp_model_step", C.byref(self.desc), st.data_ptr(), acts.data_ptr(), key_of(rng.rng),
                  rows.data_ptr(), n, obs.data_ptr(), rew.data_ptr(), stream)
        rec = st.cpu().numpy().view(self.state_dtype)
        o = obs.cpu().numpy().view(np.uint32).astype(np.int64)
        return StepResult(self.unpack(rec), o, rew.cpu().numpy())

    def heuristic(self, states) -> np.ndarray:
        torch = _torch()
        n = len(states)
        if n == 0:
            return np.zeros(0)
        st = self.states_to_device(states)
        out = torch.empty(n, dtype=torch.float64, device="cuda")
        self.call("vp_model_heuristic", C.byref(self.desc), st.data_ptr(), n, out.data_ptr(),
                  torch.cuda.current_stream().cuda_stream)
        return out.cpu().numpy()

    def obs_loglik(self, states, action: int, observation: int) -> np.ndarray:
        """observation_log_likelihood on the device via vp_model_obs_loglik."""
        torch = _torch()
        n = len(states)
        if n == 0:
            return np.zeros(0)
        st = self.states_to_device(states)
        out = torch.empty(n, dtype=torch.float64, device="cuda")
        self.call("vp_model_obs_loglik", C.byref(self.desc), st.data_ptr(), n, int(action), int(observation),
                  out.data_ptr(), torch.cuda.current_stream().cuda_stream)
        return out.cpu().numpy()


# ------------------------------------------------------------------ MARS


def _rock_bits(rocks: np.ndarray) -> np.ndarray:
    r = np.asarray(rocks, dtype=bool)
    if r.shape[1] > 64:
        raise ValueError("MARS device records hold at most 64 rocks")
    shifts = np.arange(r.shape[1], dtype=np.uint64)
    return np.bitwise_or.reduce(r.astype(np.uint64) << shifts[None, :], axis=1) if r.shape[1] else \
        np.zeros(len(r), dtype=np.uint64)


def mars_pack_into(states, dst: np.ndarray) -> int:
    """MarsStates -> 16-B records written into the byte buffer ``dst`` as two little-endian
    words {x0 | y0 << 8 | x1 << 16 | y1 << 24 | terminal << 32, rock bits}.  This runs on the
    host inside every e2e planning step, so it uses whole-vector integer ops on contiguous
    columns (no strided byte stores, no per-row bit packing)."""
    x = np.asarray(states.x)
    y = np.asarray(states.y)
    n = len(x)
    term, rk = np.asarray(states.terminal), np.asarray(states.rocks)
    if (x.dtype == y.dtype == np.int64 and term.dtype == rk.dtype == np.bool_ and x.shape == y.shape == (n, 2)
            and term.shape == (n,) and rk.ndim == 2 and rk.shape[0] == n and rk.shape[1] <= 64
            and all(a.flags["C_CONTIGUOUS"] for a in (x, y, term, rk))):
        # the library's host packer (vp_pack_mars_states): the same words, ~4x faster
        _lib.call("vp_pack_mars_states", x.ctypes.data, y.ctypes.data, term.ctypes.data, rk.ctypes.data, n,
                  rk.shape[1], dst.ctypes.data)
        return 16 * n
    out = dst[: 16 * n].view(np.uint64).reshape(n, 2)
    t = np.left_shift(y, 8, dtype=np.int64)
    t |= x
    w0 = t[:, 1] << 16
    w0 |= t[:, 0]
    w0 |= np.asarray(states.terminal).astype(np.int64) << 32
    out[:, 0] = w0
    r = np.asarray(states.rocks, dtype=bool)
    m = r.shape[1]
    if m > 64:
        raise ValueError("MARS device records hold at most 64 rocks")
    if m == 0:
        out[:, 1] = 0
    elif m <= 24:  # sums of distinct 2^k < 2^24 are exact in float32: one mat-vec
        out[:, 1] = r.astype(np.float32) @ np.exp2(np.arange(m, dtype=np.float32))
    elif m <= 52:
        out[:, 1] = r.astype(np.float64) @ np.exp2(np.arange(m))
    else:
        out[:, 1] = np.packbits(np.pad(r, ((0, 0), (0, 64 - m))), axis=1, bitorder="little").view("<u8")[:, 0]
    return 16 * n


def mars_pack(states) -> np.ndarray:
    n = len(np.asarray(states.x))
    out = np.empty(16 * n, dtype=np.uint8)
    mars_pack_into(states, out)
    return out.view(MARS_DTYPE)


def mars_descriptor(model, unpack=None) -> DeviceModel:
    """vp_model for a MarsModel (reference envs/mars.py:44-80 attributes)."""
    n, m = int(model.n), int(model.m)
    if n > 254 or m > 64:
        raise ValueError("MARS device model supports n <= 254 and m <= 64")
    dm = DeviceModel(_lib.VP_MODEL_MARS, model.spec, MARS_DTYPE, mars_pack, unpack, mars_pack_into)
    d = dm.desc
    d.mars_n, d.mars_m, d.mars_ops = n, m, int(model.per_agent_ops)
    d.mars_half_eff = float(model.half_efficiency_distance)
    rock_at = np.asarray(model.rock_at, dtype=np.int64).astype(np.int8).reshape(-1)  # [x, y] -> x*n + y
    d.mars_rock_at = dm.upload(rock_at)
    # the generative model's only transcendental terms, tabulated with the reference's own numpy
    # arithmetic (bit-exact by construction): sensor accuracy by |dx|, |dy| and gamma**k
    dxy = np.arange(n + 1, dtype=np.int64)
    dist = np.sqrt(dxy[:, None] ** 2.0 + dxy[None, :] ** 2.0)
    d.mars_acc = dm.upload(np.ascontiguousarray(model.check_accuracy(dist.reshape(-1)), dtype=np.float64))
    d.mars_gpow = dm.upload(model.spec.discount ** np.arange(2 * n + 2, dtype=np.float64))
    for i in range(m):
        d.mars_rock_x[i] = int(model.rock_x[i])
        d.mars_rock_y[i] = int(model.rock_y[i])
    return dm


# ------------------------------------------------------------------ TABULAR


def tab_pack(states) -> np.ndarray:
    rec = np.zeros(len(states.idx), dtype=TAB_DTYPE)
    rec["idx"] = np.asarray(states.idx)
    rec["term"] = np.asarray(states.terminal, dtype=bool)
    return rec


def tabular_descriptor(model, unpack=None) -> DeviceModel:
    """vp_model for a TabularModel (reference envs/tabular.py:79-92)."""
    p = model.pomdp
    t = np.asarray(p.transitions, dtype=np.float64)
    z = np.asarray(p.observations, dtype=np.float64)
    dm = DeviceModel(_lib.VP_MODEL_TABULAR, model.spec, TAB_DTYPE, tab_pack, unpack)
    d = dm.desc
    d.tab_states = t.shape[1]
    d.tab_obs = z.shape[2]
    d.tab_cum_t = dm.upload(np.cumsum(t, axis=2).reshape(-1))
    d.tab_cum_z = dm.upload(np.cumsum(z, axis=2).reshape(-1))
    d.tab_reward = dm.upload(np.asarray(p.rewards, dtype=np.float64).reshape(-1))
    d.tab_terminal = dm.upload(np.asarray(p.terminal_states, dtype=np.uint8))
    with np.errstate(divide="ignore"):
        d.tab_log_z = dm.upload(np.log(z).reshape(-1))  # SIR likelihood (tabular.py observation model)
    return dm


# ------------------------------------------------------------------ SYNTHETIC


def syn_pack(states) -> np.ndarray:
    rec = np.zeros(len(states.word), dtype=SYN_DTYPE)
    rec["word"] = np.asarray(states.word, dtype=np.uint64)
    rec["term"] = np.asarray(states.terminal, dtype=bool)
    return rec


def synthetic_descriptor(model, unpack=None) -> DeviceModel:
    dm = DeviceModel(_lib.VP_MODEL_SYNTHETIC, model.spec, SYN_DTYPE, syn_pack, unpack)
    d = dm.desc
    d.syn_branching = int(model.branching)
    d.syn_term_per_mille = int(model.term_per_mille)
    d.syn_obs_accuracy = float(model.obs_accuracy)
    d.syn_salt = int(model.salt) & ((1 << 64) - 1)
    return dm


# ------------------------------------------------------------------ LIGHTDARK


def ld_pack(states) -> np.ndarray:
    rec = np.zeros(len(states.x), dtype=LD_DTYPE)
    rec["x"] = np.asarray(states.x, dtype=np.float64)
    rec["y"] = np.asarray(states.y, dtype=np.float64)
    rec["term"] = np.asarray(states.terminal, dtype=bool)
    return rec


def lightdark_descriptor(model, unpack=None) -> DeviceModel:
    dm = DeviceModel(_lib.VP_MODEL_LIGHTDARK, model.spec, LD_DTYPE, ld_pack, unpack)
    d = dm.desc
    d.ld_step, d.ld_light_x, d.ld_goal_radius = float(model.step), float(model.light_x), float(model.goal_radius)
    d.ld_sigma0, d.ld_sigma_slope = float(model.sigma0), float(model.sigma_slope)
    d.ld_bin_width, d.ld_bins = float(model.bin_width), int(model.bins)
    return dm


# ------------------------------------------------------------------ NAVIGATION


def nav_pack(states) -> np.ndarray:
    occ = np.asarray(states.occ, dtype=bool)
    if occ.shape[1] > 128:
        raise ValueError("Navigation device records hold at most 128 unknown cells")
    bits = np.packbits(np.pad(occ, ((0, 0), (0, 128 - occ.shape[1]))), axis=1, bitorder="little")
    rec = np.zeros(len(occ), dtype=NAV_DTYPE)
    words = bits.view("<u8")
    rec["occ0"], rec["occ1"] = words[:, 0], words[:, 1]
    rec["pos"] = np.asarray(states.pos)
    rec["gate"] = np.asarray(states.open_gate)
    rec["term"] = np.asarray(states.terminal, dtype=bool)
    return rec


def nav_unpacker(n_unknown: int, states_cls):
    def unpack(rec):
        words = np.stack([rec["occ0"], rec["occ1"]], axis=1).astype("<u8")
        occ = np.unpackbits(words.view(np.uint8), axis=1, bitorder="little")[:, :n_unknown].astype(bool)
        return states_cls(rec["pos"].astype(np.int64), occ, rec["gate"].astype(np.int64), rec["term"].astype(bool))
    return unpack


def navigation_descriptor(model, unpack=None) -> DeviceModel:
    """vp_model for a NavigationModel (reference envs/navigation.py:62-121 attributes)."""
    if model.n_unknown > 128:
        raise ValueError("Navigation device records hold at most 128 unknown cells")
    if unpack is None:  # a reference model object: rebuild records as the product's NavStates
        from .navigation import NavStates

        unpack = nav_unpacker(int(model.n_unknown), NavStates)
    dm = DeviceModel(_lib.VP_MODEL_NAVIGATION, model.spec, NAV_DTYPE, nav_pack, unpack)
    d = dm.desc
    d.nav_h, d.nav_w, d.nav_unknown = int(model.height), int(model.width), int(model.n_unknown)
    d.nav_kind = dm.upload(np.asarray(model.kind, dtype=np.int8).reshape(-1))
    d.nav_aux = dm.upload(np.asarray(model.aux, dtype=np.int64).astype(np.int16).reshape(-1))
    d.nav_goal = dm.upload(np.asarray(model.goal, dtype=np.uint8).reshape(-1))
    # the heuristic and the sensor logs with the reference's own numpy arithmetic (bit-exact)
    g = model.spec.discount
    dist = np.asarray(model.goal_dist if hasattr(model, "goal_dist") else model._goal_dist)
    decay = g ** np.maximum(dist - 1.0, 0.0)
    d.nav_heur = dm.upload((20.0 * decay - 0.1 * (1.0 - decay) / (1.0 - g)).reshape(-1))
    d.nav_acc = float(model.sensor_accuracy)
    d.nav_log_acc = float(np.log(model.sensor_accuracy))
    with np.errstate(divide="ignore"):
        d.nav_log_miss = float(np.log(1.0 - model.sensor_accuracy))
    return dm


# ------------------------------------------------------------------ CROWDNAV


def crowd_pack_into(states, dst: np.ndarray) -> int:
    """CrowdStates -> 2704-B records written straight into the byte buffer ``dst`` (pinned host
    memory on the e2e path: one pass over the 2.7 KB records, no temporary copy)."""
    n = len(np.asarray(states.robot))
    rec = dst[: n * CROWD_DTYPE.itemsize].view(CROWD_DTYPE)
    _crowd_fill(states, rec)
    return n * CROWD_DTYPE.itemsize


def crowd_pack(states) -> np.ndarray:
    rec = np.zeros(len(np.asarray(states.robot)), dtype=CROWD_DTYPE)
    _crowd_fill(states, rec)
    return rec


def _crowd_fill(states, rec) -> None:
    persons = np.asarray(states.persons, dtype=np.float32)
    n, p = persons.shape[:2]
    k = np.asarray(states.tracked).shape[1]
    if p > _lib.CROWD_MAX_PEOPLE or k > _lib.CROWD_MAX_TRACKED:
        raise ValueError(f"CrowdNav device records hold at most {_lib.CROWD_MAX_PEOPLE} people and "
                         f"{_lib.CROWD_MAX_TRACKED} tracked persons")
    if k < _lib.CROWD_MAX_TRACKED:
        rec["prev"][:, k:] = 0.0
        rec["tracked"][:, k:] = 0
    if p < _lib.CROWD_MAX_PEOPLE:
        rec["persons"][:, 2 * p:] = 0.0
    rec["robot"] = np.asarray(states.robot, dtype=np.float64)
    rec["prev"][:, :k] = np.asarray(states.prev_dist, dtype=np.float64)
    rec["code"] = np.asarray(states.last_code)
    rec["term"] = np.asarray(states.terminal, dtype=bool)
    rec["tracked"][:, :k] = np.asarray(states.tracked)
    cur = np.pad(np.asarray(states.curious, dtype=bool), ((0, 0), (0, _lib.CROWD_MAX_PEOPLE - p)))
    rec["curious"] = np.packbits(cur, axis=1, bitorder="little").view("<u4")
    rec["persons"][:, : 2 * p] = persons.reshape(n, 2 * p)


def crowd_unpacker(n_people: int, n_tracked: int, states_cls):
    def unpack(rec):
        n = len(rec)
        bits = np.ascontiguousarray(rec["curious"]).view(np.uint8)
        curious = np.unpackbits(bits, axis=1, bitorder="little")[:, :n_people].astype(bool)
        persons = np.ascontiguousarray(rec["persons"][:, : 2 * n_people]).reshape(n, n_people, 2)
        return states_cls(np.array(rec["robot"]), persons, curious, rec["tracked"][:, :n_tracked].astype(np.int64),
                          np.array(rec["prev"][:, :n_tracked]), rec["code"].astype(np.int64), rec["term"].astype(bool))
    return unpack


def crowdnav_descriptor(model, unpack=None) -> DeviceModel:
    """vp_model for a CrowdNavModel (reference envs/crowdnav.py:54-91 attributes)."""
    if model.n_people > _lib.CROWD_MAX_PEOPLE or model.n_tracked > _lib.CROWD_MAX_TRACKED:
        raise ValueError(f"CrowdNav device records hold at most {_lib.CROWD_MAX_PEOPLE} people and "
                         f"{_lib.CROWD_MAX_TRACKED} tracked persons")
    if unpack is None:  # a reference model object: rebuild records as the product's CrowdStates
        from .crowdnav import CrowdStates

        unpack = crowd_unpacker(int(model.n_people), int(model.n_tracked), CrowdStates)
    dm = DeviceModel(_lib.VP_MODEL_CROWDNAV, model.spec, CROWD_DTYPE, crowd_pack, unpack, crowd_pack_into)
    d = dm.desc
    hall = np.asarray(model.hall, dtype=np.float64)
    d.crowd_people, d.crowd_tracked = int(model.n_people), int(model.n_tracked)
    d.crowd_hall_w, d.crowd_hall_d = float(hall[0]), float(hall[1])
    d.crowd_noise, d.crowd_react, d.crowd_r_nearby = (float(model.motion_noise), float(model.react_prob),
                                                      float(model.r_nearby))
    d.crowd_v_curious, d.crowd_v_shy, d.crowd_v_back = float(model.v_curious), float(model.v_shy), float(model.v_back)
    d.crowd_collision = float(model.collision_radius)
    # heuristic per remaining-row count with the reference's own numpy arithmetic (bit-exact)
    g = model.spec.discount
    decay = g ** np.arange(int(np.ceil(hall[1])) + 1, dtype=np.float64)
    heur = 1000.0 * decay - (1.0 - decay) / (1.0 - g)
    d.crowd_heur, d.crowd_heur_len = dm.upload(heur), len(heur)
    return dm


_BY_NAME = {
    "MarsModel": mars_descriptor,
    "TabularModel": tabular_descriptor,
    "SyntheticModel": synthetic_descriptor,
    "LightDarkModel": lightdark_descriptor,
    "NavigationModel": navigation_descriptor,
    "CrowdNavModel": crowdnav_descriptor,
}
_CACHE: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()
# ProblemModel methods the device re-implements (core.py:84-142): search / SIR step, leaf value,
# SIR likelihood.  reference_log_probs, the initial-state sampler and the belief hooks run on the host.
_DEVICE_METHODS = frozenset({"step_batch", "value_heuristic", "observation_log_likelihood"})


def device_model(model) -> DeviceModel:
    """The (cached) DeviceModel of any supported ProblemModel instance."""
    try:
        return _CACHE[model]
    except (KeyError, TypeError):
        pass
    mro = type(model).__mro__
    if hasattr(model, "device_descriptor"):
        # the class providing the descriptor binds the dynamics of the classes from it upward
        known = next(i for i, c in enumerate(mro) if "device_descriptor" in vars(c))
    else:
        # the model's class or its nearest known base (subclasses of the reference's models,
        # e.g. with another reference policy, keep their device layout)
        known = next((i for i, c in enumerate(mro) if c.__name__ in _BY_NAME), None)
        if known is None:
            raise TypeError(f"no device model for {type(model).__name__}; supported: {sorted(_BY_NAME)} -- or state "
                            f"its dynamics in CUDA as a paper_2510_27191_b200.CudaModel plug-in")
    # a subclass that changes the dynamics the device runs (the generative step, the leaf
    # heuristic, the SIR likelihood) must not silently plan with its base's device model
    for c in mro[:known]:
        bad = sorted(set(vars(c)) & _DEVICE_METHODS)
        if bad:
            raise TypeError(f"{type(model).__name__} overrides {', '.join(bad)} of {mro[known].__name__} "
                            f"(in {c.__name__}); the device runs {mro[known].__name__}'s dynamics -- give the "
                            f"model its own device_descriptor() or keep those methods")
    dm = model.device_descriptor() if hasattr(model, "device_descriptor") else _BY_NAME[mro[known].__name__](model)
    try:
        _CACHE[model] = dm
    except TypeError:
        pass
    return dm
