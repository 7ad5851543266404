"""Device forward search (API mirror of /root/reference/pkg/src/vecpomdp/search.py).

``search(tree, model, batch, d_max, eta, rng)`` descends every row of the
batch ``d_max - batch.depth`` levels in ONE kernel launch (``vp_search``):
per level the rows draw actions from the softmax of their belief's PSI row,
step the device generative model and extend the tree through the two hash
indexes, without a grid barrier or a host round trip (csrc/vp_phases.cuh).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .envs._device import device_model
from .rng import key_of, kind_of

SITE_ACTION = 0
SITE_MODEL = 1


def _torch():
    return _lib.torch_cuda()


class Workspace:
    """Per-row scratch of n simulation rows: start states, leaf list and traces."""

    def __init__(self, n: int, max_levels: int, state_bytes: int, trace: bool = False, stats: bool = False):
        if n < 1:
            raise ValueError("n_parallel must be >= 1")
        if n >= 1 << 24:
            raise ValueError("n_parallel must be < 2**24")
        torch = _torch()
        dev = "cuda"
        L = max(1, int(max_levels))
        if L > 255:
            raise ValueError("d_max must be <= 255")
        self.n, self.max_levels, self.state_bytes, self.trace = n, L, state_bytes, trace
        i32 = dict(dtype=torch.int32, device=dev)
        self.states = torch.empty(n * state_bytes + 16, dtype=torch.uint8, device=dev)
        self.leaves = torch.empty(n, **i32)
        self.leaf_count = torch.zeros(2, **i32)
        self.leaf_belief = torch.empty(n, **i32)
        self.leaf_value = torch.empty(n, dtype=torch.float64, device=dev)
        self.stats = torch.zeros(16, dtype=torch.int64, device=dev)
        self.last_pass = 0
        s = _lib.VpWork()
        s.n, s.max_levels = n, L
        for name in ("states", "leaves", "leaf_count", "leaf_belief", "leaf_value"):
            setattr(s, name, getattr(self, name).data_ptr())
        if trace:
            self.trace_action = torch.empty(L * n, **i32)
            self.trace_obs = torch.empty(L * n, **i32)
            self.trace_anode = torch.empty(L * n, **i32)
            self.trace_belief = torch.empty(L * n, **i32)
            self.trace_reward = torch.empty(L * n, dtype=torch.float64, device=dev)
            for name in ("trace_action", "trace_obs", "trace_anode", "trace_belief", "trace_reward"):
                setattr(s, name, getattr(self, name).data_ptr())
        self.struct = s
        self.enable_stats(stats)

    def enable_stats(self, on: bool):
        """Traffic counters (vp_work.stats) -- off on the timed path."""
        self.struct.stats = self.stats.data_ptr() if on else None

    def fits(self, n: int, levels: int, state_bytes: int, trace: bool) -> bool:
        return (self.n == n and self.max_levels >= levels and self.state_bytes == state_bytes
                and (self.trace or not trace))

    def traces(self, tree, depth0: int, d_max: int) -> list:
        """Per-level host copies of the traced columns (like oracle.search(trace=)),
        node ids in reference numbering."""
        n = self.n
        out = []
        for lvl in range(depth0, d_max):
            sl = slice(lvl * n, (lvl + 1) * n)
            out.append({"actions": self.trace_action[sl].cpu().numpy().astype(np.int64),
                        "observations": self.trace_obs[sl].cpu().numpy().view(np.uint32).astype(np.int64),
                        "action_nodes": tree.to_reference_actions(self.trace_anode[sl]).cpu().numpy(),
                        "next_beliefs": tree.to_reference_beliefs(self.trace_belief[sl]).cpu().numpy()})
        return out


@dataclass
class SearchBatch:
    """Frontier of a search call (search.py:26-37)."""

    belief_indices: np.ndarray
    states: object
    depth: int = 0

    def __post_init__(self):
        self.belief_indices = np.asarray(self.belief_indices, dtype=np.int64)
        if len(self.belief_indices) != len(self.states):
            raise ValueError("belief_indices and states must have equal length")


class LeafResult:
    """Device frontier after a search (search.py:40-43); host arrays on demand
    (belief ids in reference numbering)."""

    def __init__(self, tree, work: Workspace, depth0: int, d_max: int, pass_: int, generation: int):
        self.tree, self.work = tree, work
        self.depth0, self.d_max, self.pass_, self.generation = depth0, d_max, pass_, generation

    @property
    def leaf_belief_indices(self) -> np.ndarray:
        return self.tree.to_reference_beliefs(self.work.leaf_belief.to(_torch().int64)).cpu().numpy()

    @property
    def heuristic_values(self) -> np.ndarray:
        return self.work.leaf_value.cpu().numpy().copy()


def run_search(tree, dm, work: Workspace, search_key: int, depth0: int, d_max: int, pass_: int, inject=None,
               start=None, particles=None, cumw=None, m: int = 0, draw_key: int = 0):
    """Launch one device search (no host synchronisation).  With ``particles``
    the rows draw their start states from the belief inside the kernel."""
    args = _lib.VpSearchArgs()
    args.search_key = search_key
    args.depth0, args.d_max, args.pass_ = depth0, d_max, pass_
    args.inject_actions = inject.data_ptr() if inject is not None else None
    args.start_beliefs = start.data_ptr() if start is not None else None
    if particles is not None:
        args.particles, args.cum_weights, args.m, args.draw_key = particles.data_ptr(), cumw.data_ptr(), m, draw_key
    if pass_ != work.last_pass + 1:
        work.leaf_count.zero_()  # the leaf-list parity chain restarts (fresh tree or another tree)
    work.last_pass = pass_
    stream = _torch().cuda.current_stream().cuda_stream
    dm.call("vp_search", C.byref(tree.struct), C.byref(dm.desc), C.byref(work.struct), C.byref(args), stream)
    tree._scratch_dirty = True


def search(tree, model, batch: SearchBatch, d_max: int, eta: float, rng, *, inject_actions=None,
           trace: bool = False) -> LeafResult:
    """Descend ``d_max - batch.depth`` levels expanding ``tree`` in place (search.py:86-119).

    ``inject_actions`` (test hook): a (d_max, n) array of actions replacing the
    softmax draws level by level (the "identical injected sample streams" of
    the parity contract).
    """
    torch = _torch()
    if eta <= 0:
        raise ValueError("eta must be positive")
    if batch.depth > d_max:
        raise ValueError("batch.depth must not exceed d_max")
    dm = device_model(model)
    n = len(batch.belief_indices)
    bi = batch.belief_indices
    if n and (bi.min() < 0 or bi.max() >= tree.counts()[0]):
        raise ValueError("invalid belief index in batch")
    tree.set_eta(eta)
    tree.clear_pass_scratch()
    levels = max(d_max, 1)
    work = getattr(tree, "_api_work", None)
    if work is None or not work.fits(n, levels, dm.state_bytes, trace):
        work = Workspace(n, levels, dm.state_bytes, trace)
        tree._api_work = work
    nb, na = tree.extent()
    grow = n * (d_max - batch.depth)
    tree.ensure_capacity(nb + grow, na + grow)
    rec = dm.pack(batch.states)
    work.states[: rec.nbytes].copy_(torch.from_numpy(rec.view(np.uint8).reshape(-1)))
    start = tree.to_device_beliefs(bi).to(torch.int32)
    inject = None
    if inject_actions is not None:
        arr = np.zeros((levels, n), dtype=np.int32)
        arr[: d_max] = np.asarray(inject_actions, dtype=np.int32).reshape(d_max, n)
        inject = torch.from_numpy(arr.reshape(-1)).cuda()
    pass_ = tree.next_pass()
    dm.desc.rng_kind = kind_of(rng)
    run_search(tree, dm, work, key_of(rng), batch.depth, d_max, pass_, inject, start)
    leaves = LeafResult(tree, work, batch.depth, d_max, pass_, tree.generation)
    tree.last_search = leaves
    return leaves


def search_recorded(tree, model, actions, observations, rewards, leaf_values) -> LeafResult:
    """A search pass from the root whose rows' trajectories are given: (d, n) actions,
    observations and rewards and n leaf values (VP_SEARCH_INSERT, the insert half of a
    sharded pass).  The rows extend the tree exactly as search.py:106-119 would had they
    drawn these samples (append_actions / append_beliefs, rewards and visits, the leaf
    frontier), so ``backup(tree, leaves, d, ...)`` applies Alg. 3 to them -- the hook the
    backup acceptance test (SPEC ACCEPTANCE 1) builds its random trees with."""
    torch = _torch()
    act = np.ascontiguousarray(np.asarray(actions, dtype=np.int32))
    obs = np.ascontiguousarray(np.asarray(observations, dtype=np.int64))
    rew = np.ascontiguousarray(np.asarray(rewards, dtype=np.float64))
    leaf = np.ascontiguousarray(np.asarray(leaf_values, dtype=np.float64))
    if act.ndim != 2 or obs.shape != act.shape or rew.shape != act.shape or leaf.shape != (act.shape[1],):
        raise ValueError("actions / observations / rewards must be (d, n) and leaf_values (n,)")
    d, n = act.shape
    A = tree.action_count
    if d < 1 or n < 1:
        raise ValueError("need at least one level and one row")
    if act.min() < 0 or act.max() >= A:
        raise ValueError("invalid action")
    if obs.min() < 0 or obs.max() > model.spec.observation_arity:
        raise ValueError("invalid observation code")
    dm = device_model(model)
    if dm.desc.action_count != A:
        raise ValueError("model and tree differ in action count")
    tree.clear_pass_scratch()
    work = getattr(tree, "_api_work", None)
    if work is None or not work.fits(n, d, dm.state_bytes, False):
        work = Workspace(n, d, dm.state_bytes, False)
        tree._api_work = work
    nb, na = tree.extent()
    tree.ensure_capacity(nb + n * d, na + n * d)
    dev = {k: torch.from_numpy(v.reshape(-1)).cuda() for k, v in
           (("a", act), ("o", obs.astype(np.uint32).view(np.int32)), ("r", rew), ("h", leaf))}
    pass_ = tree.next_pass()
    args = _lib.VpSearchArgs()
    args.depth0, args.d_max, args.pass_ = 0, d, pass_
    args.mode = _lib.VP_SEARCH_INSERT
    args.inject_actions, args.inject_obs = dev["a"].data_ptr(), dev["o"].data_ptr()
    args.inject_reward, args.inject_leaf = dev["r"].data_ptr(), dev["h"].data_ptr()
    if pass_ != work.last_pass + 1:
        work.leaf_count.zero_()
    work.last_pass = pass_
    stream = torch.cuda.current_stream()
    dm.call("vp_search", C.byref(tree.struct), C.byref(dm.desc), C.byref(work.struct), C.byref(args),
            stream.cuda_stream)
    stream.synchronize()  # the injected columns are temporaries
    tree._scratch_dirty = True
    leaves = LeafResult(tree, work, 0, d, pass_, tree.generation)
    tree.last_search = leaves
    return leaves


def softmax_rows(pref_rows, eta: float, *, precision: str = "fp64"):
    """Row softmax of eta * PSI (search.py:46-54), computed from the device CDF."""
    if eta <= 0:
        raise ValueError("eta must be positive")
    from .backup import log_sum_exp_rows

    rows = np.asarray(pref_rows, dtype=np.float64)
    lse = log_sum_exp_rows(rows, eta, precision=precision, exact=precision == "fp64")
    return np.exp(eta * (rows - lse[..., None]))


def sample_actions(policies_or_prefs, uniforms, groups=None, *, eta: float = 1.0, precision: str = "fp64",
                   exact: bool = True) -> np.ndarray:
    """Device categorical draws: row ``groups[i]`` of softmax(eta * prefs) with
    uniform ``uniforms[i]`` (the draw of search.py:57-83 given its uniforms)."""
    torch = _torch()
    rows = np.ascontiguousarray(np.atleast_2d(np.asarray(policies_or_prefs, dtype=np.float64)))
    u = np.asarray(uniforms, dtype=np.float64)
    g = np.zeros(len(u), dtype=np.int32) if groups is None else np.asarray(groups, dtype=np.int32)
    dt = torch.float64 if precision == "fp64" else torch.float32
    dev_rows = torch.from_numpy(rows).to(dt).cuda()
    dtype_code = 1 if precision == "fp64" else 0
    if not exact:
        from .backup import log_sum_exp_rows

        lse = torch.from_numpy(np.atleast_1d(log_sum_exp_rows(rows.astype(np.float64) if precision == "fp64"
                                                              else rows.astype(np.float32).astype(np.float64),
                                                              eta, precision=precision, exact=False))).cuda()
    out = torch.empty(len(u), dtype=torch.int32, device="cuda")
    dev_g = torch.from_numpy(g).cuda()  # keep every operand alive until the kernel has run
    dev_u = torch.from_numpy(u).cuda()
    _lib.call("vp_sample_rows", dev_rows.data_ptr(), dtype_code, int(exact), rows.shape[0], rows.shape[1],
              float(eta), None if exact else lse.data_ptr(), dev_g.data_ptr(), dev_u.data_ptr(), len(u),
              out.data_ptr(), torch.cuda.current_stream().cuda_stream)
    return out.cpu().numpy().astype(np.int64)
