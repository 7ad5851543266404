"""Device PORPP backup (API mirror of /root/reference/pkg/src/vecpomdp/backup.py).

``backup(tree, leaves, d_max, eta, gamma)`` runs Alg. 3 on the device in ONE
kernel (csrc/vp_phases.cuh backup_warp): leaf means and counts, then a
bottom-up completion wave -- an action's Q and PSI scatter happen when its
last valued child delivers, a belief's LSE when its last visited action
completes.  That is the reference's level order restricted to each subtree:
every node is updated after all of its valued children, exactly once, and
the valued sets are the nodes the search visited (SURVEY.md section 0
finding 2), so no depth scan is needed.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib


def _torch():
    return _lib.torch_cuda()


def run_backup(tree, work, pass_: int, gamma: float):
    stream = _torch().cuda.current_stream().cuda_stream
    _lib.call("vp_backup", C.byref(tree.struct), C.byref(work.struct), pass_, float(gamma), stream)
    tree._scratch_dirty = False


def backup(tree, leaves, d_max: int, eta: float, gamma: float) -> None:
    """In-place preference backup after a device ``search`` (backup.py:75-114)."""
    if eta <= 0:
        raise ValueError("eta must be positive")
    if getattr(leaves, "tree", None) is not tree or leaves.generation != tree.generation:
        raise ValueError("device backup consumes the LeafResult of the latest device search on this tree")
    if tree.last_search is not leaves:
        raise ValueError("leaves are stale: another search ran on this tree since")
    if d_max != leaves.d_max:
        raise ValueError("d_max must match the search that produced the leaves")
    tree.set_eta(eta)
    run_backup(tree, leaves.work, leaves.pass_, gamma)
    tree.last_search = None


def log_sum_exp_rows(pref_rows, eta: float, *, precision: str = "fp64", exact: bool = True) -> np.ndarray:
    """(1/eta) log sum exp(eta * PSI) per row on the device (backup.py:34-41)."""
    if eta <= 0:
        raise ValueError("eta must be positive")
    torch = _torch()
    rows = np.ascontiguousarray(np.atleast_2d(np.asarray(pref_rows, dtype=np.float64)))
    if precision == "fp32":
        exact = False
    dt = torch.float64 if precision == "fp64" else torch.float32
    dev = torch.from_numpy(rows).to(dt).cuda()
    out = torch.empty(rows.shape[0], dtype=torch.float64, device="cuda")
    _lib.call("vp_lse_rows", dev.data_ptr(), 1 if precision == "fp64" else 0, int(exact), rows.shape[0],
              rows.shape[1], float(eta), out.data_ptr(), torch.cuda.current_stream().cuda_stream)
    res = out.cpu().numpy()
    return res if np.ndim(pref_rows) > 1 else res[0]


class LevelValues:
    """Per-belief values of one level (backup.py:25-31): distinct beliefs, their values and
    visit weights (device tensors; host arrays through the properties)."""

    def __init__(self, belief_indices, values, visit_weights):
        self._b, self._v, self._w = belief_indices, values, visit_weights

    @property
    def belief_indices(self) -> np.ndarray:
        return self._b.cpu().numpy()

    @property
    def values(self) -> np.ndarray:
        return self._v.cpu().numpy()

    @property
    def visit_weights(self) -> np.ndarray:
        return self._w.cpu().numpy()


def aggregate_leaves(leaves) -> LevelValues:
    """backup.py:44-51 on the device: per distinct leaf belief, N = rows that ended there and
    V = their mean heuristic value (sums by device reductions: equal to numpy's bincount up to
    the order of floating-point additions)."""
    torch = _torch()
    ids = torch.as_tensor(np.asarray(leaves.leaf_belief_indices, dtype=np.int64), device="cuda")
    h = torch.as_tensor(np.asarray(leaves.heuristic_values, dtype=np.float64), device="cuda")
    if ids.shape != h.shape:
        raise ValueError("leaf ids and heuristic values differ in length")
    distinct, grp = torch.unique(ids, sorted=True, return_inverse=True)
    n = torch.zeros(len(distinct), dtype=torch.float64, device="cuda").index_add_(0, grp, torch.ones_like(h))
    total = torch.zeros(len(distinct), dtype=torch.float64, device="cuda").index_add_(0, grp, h)
    return LevelValues(distinct, total / n, n)


def action_q_values(tree, action_rows, child: LevelValues, gamma: float) -> np.ndarray:
    """backup.py:54-72 on the device tree: Q(a) = reward_sum / visits + gamma * sum(V N) / sum(N)
    over a's valued children (reference ids in; ValueError for an action without valued child)."""
    torch = _torch()
    t = tree.tables()  # reference-ordered columns (parent_action of the children, action stats)
    acts = torch.as_tensor(np.asarray(action_rows, dtype=np.int64), device="cuda")
    kids = torch.as_tensor(np.asarray(child.belief_indices, dtype=np.int64), device="cuda")
    v = torch.as_tensor(np.asarray(child.values, dtype=np.float64), device="cuda")
    w = torch.as_tensor(np.asarray(child.visit_weights, dtype=np.float64), device="cuda")
    par = torch.as_tensor(t["parent_action"], device="cuda")[kids]
    na = len(t["action_id"])
    num = torch.zeros(na, dtype=torch.float64, device="cuda").index_add_(0, par, v * w)
    den = torch.zeros(na, dtype=torch.float64, device="cuda").index_add_(0, par, w)
    if bool((den[acts] <= 0).any()):
        raise ValueError("action node without valued children")
    reward = torch.as_tensor(t["action_reward_sum"], device="cuda")[acts]
    visits = torch.as_tensor(t["action_visits"], device="cuda").to(torch.float64)[acts]
    return (reward / visits + gamma * num[acts] / den[acts]).cpu().numpy()
