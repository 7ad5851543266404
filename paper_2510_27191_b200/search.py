"""Device forward search (API mirror of /root/reference/pkg/src/vecpomdp/search.py).

``search(tree, model, batch, d_max, eta, rng)`` descends every row of the
batch ``d_max - batch.depth`` levels in one ``vp_search`` call: per level the
rows draw actions from the softmax of their belief's PSI row, step the device
generative model and extend the tree through the two hash indexes, all
without a host round trip (csrc/vp_kernels.cu, K1..K4).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .envs._device import device_model
from .rng import key_of

SITE_ACTION = 0
SITE_MODEL = 1


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_2510_27191_b200 needs a CUDA device (B200, sm_100a); there is no CPU fallback")
    return torch


class Workspace:
    """Per-row scratch and per-level distinct lists for n simulation rows."""

    def __init__(self, n: int, max_levels: int, state_bytes: int, trace: bool = False):
        if n < 1:
            raise ValueError("n_parallel must be >= 1")
        torch = _torch()
        dev = "cuda"
        L = max(1, int(max_levels))
        self.n, self.max_levels, self.state_bytes, self.trace = n, L, state_bytes, trace
        i32 = dict(dtype=torch.int32, device=dev)
        self.states = torch.empty(n * state_bytes + 16, dtype=torch.uint8, device=dev)
        self.slot_a = torch.empty(n, **i32)
        self.slot_b = torch.empty(n, **i32)
        self.obs = torch.empty(n, **i32)
        self.reward = torch.empty(n, dtype=torch.float64, device=dev)
        self.action = torch.empty(n, **i32)
        self.flist = torch.empty((L + 1) * n, **i32)
        self.fcount = torch.zeros(L + 1, **i32)
        self.plist = torch.empty(L * n, **i32)
        self.pcount = torch.zeros(L, **i32)
        self.level_base = torch.zeros(2 * (L + 1), **i32)
        tiles = (n + _lib.VP_SCAN_TILE - 1) // _lib.VP_SCAN_TILE
        self.scan_status = torch.zeros(tiles, dtype=torch.int64, device=dev)
        self.scan_ticket = torch.zeros(2, **i32)
        self.leaf_belief = torch.empty(n, **i32)
        self.leaf_value = torch.empty(n, dtype=torch.float64, device=dev)
        self.stats = torch.zeros(8, dtype=torch.int64, device=dev)
        s = _lib.VpWork()
        s.n, s.max_levels = n, L
        for name in ("states", "slot_a", "slot_b", "obs", "reward", "action", "flist", "fcount", "plist",
                     "pcount", "level_base", "scan_status", "scan_ticket", "leaf_belief", "leaf_value", "stats"):
            setattr(s, name, getattr(self, name).data_ptr())
        if trace:
            self.trace_action = torch.empty(L * n, **i32)
            self.trace_obs = torch.empty(L * n, **i32)
            self.trace_anode = torch.empty(L * n, **i32)
            self.trace_belief = torch.empty(L * n, **i32)
            for name in ("trace_action", "trace_obs", "trace_anode", "trace_belief"):
                setattr(s, name, getattr(self, name).data_ptr())
        self.struct = s

    def fits(self, n: int, levels: int, state_bytes: int, trace: bool) -> bool:
        return (self.n == n and self.max_levels >= levels and self.state_bytes == state_bytes
                and (self.trace or not trace))

    def traces(self, depth0: int, d_max: int) -> list:
        """Per-level host copies of the traced columns (like oracle.search(trace=))."""
        n = self.n
        out = []
        cols = {k: getattr(self, "trace_" + k).cpu().numpy() for k in ("action", "obs", "anode", "belief")}
        for lvl in range(depth0, d_max):
            sl = slice(lvl * n, (lvl + 1) * n)
            out.append({"actions": cols["action"][sl].astype(np.int64),
                        "observations": cols["obs"][sl].view(np.uint32).astype(np.int64),
                        "action_nodes": cols["anode"][sl].astype(np.int64),
                        "next_beliefs": cols["belief"][sl].astype(np.int64)})
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
    """Device frontier after a search (search.py:40-43); host arrays on demand."""

    def __init__(self, tree, work: Workspace, depth0: int, d_max: int, stamp_base: int, generation: int):
        self.tree, self.work = tree, work
        self.depth0, self.d_max, self.stamp_base, self.generation = depth0, d_max, stamp_base, generation

    @property
    def leaf_belief_indices(self) -> np.ndarray:
        return self.work.leaf_belief.cpu().numpy().astype(np.int64)

    @property
    def heuristic_values(self) -> np.ndarray:
        return self.work.leaf_value.cpu().numpy().copy()


def run_search(tree, dm, work: Workspace, search_key: int, depth0: int, d_max: int, stamp_base: int,
               iteration: int = 0, inject=None, start=None):
    """Launch one device search (no host synchronisation)."""
    args = _lib.VpSearchArgs()
    args.search_key = search_key
    args.depth0, args.d_max = depth0, d_max
    args.stamp_base, args.iteration = stamp_base, iteration
    args.inject_actions = inject.data_ptr() if inject is not None else None
    args.start_beliefs = start.data_ptr() if start is not None else None
    stream = _torch().cuda.current_stream().cuda_stream
    _lib.call("vp_search", C.byref(tree.struct), C.byref(dm.desc), C.byref(work.struct), C.byref(args), stream)


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
    levels = max(d_max, 1)
    work = getattr(tree, "_api_work", None)
    if work is None or not work.fits(n, levels, dm.state_bytes, trace):
        work = Workspace(n, levels, dm.state_bytes, trace)
        tree._api_work = work
    nb, na, _ = tree.counts()
    grow = n * (d_max - batch.depth)
    tree.ensure_capacity(nb + grow, na + grow)
    rec = dm.pack(batch.states)
    work.states[: rec.nbytes].copy_(torch.from_numpy(rec.view(np.uint8).reshape(-1)))
    start = torch.from_numpy(bi.astype(np.int32)).cuda()
    inject = None
    if inject_actions is not None:
        arr = np.zeros((levels, n), dtype=np.int32)
        arr[: d_max] = np.asarray(inject_actions, dtype=np.int32).reshape(d_max, n)
        inject = torch.from_numpy(arr.reshape(-1)).cuda()
    stamp = tree.next_stamp_base(levels)
    run_search(tree, dm, work, key_of(rng), batch.depth, d_max, stamp, 0, inject, start)
    leaves = LeafResult(tree, work, batch.depth, d_max, stamp, tree.generation)
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
