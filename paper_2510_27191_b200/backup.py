"""Device PORPP backup (API mirror of /root/reference/pkg/src/vecpomdp/backup.py).

``backup(tree, leaves, d_max, eta, gamma)`` runs Alg. 3 level-synchronously on
the device (csrc/vp_kernels.cu k_backup_*): leaf means and counts, then for
d = d_max..1 the action Q values and PSI scatter over the distinct action
nodes of level d-1 followed by the LSE of their parent beliefs.  The visited
sets come from the per-level lists the device search recorded (the
reference's valued(d) equals the beliefs visited at search level d, SURVEY.md
section 0 finding 2), so no depth scan is needed.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_2510_27191_b200 needs a CUDA device (B200, sm_100a); there is no CPU fallback")
    return torch


def run_backup(tree, work, depth0: int, d_max: int, gamma: float, stamp_base: int):
    stream = _torch().cuda.current_stream().cuda_stream
    _lib.call("vp_backup", C.byref(tree.struct), C.byref(work.struct), depth0, d_max, float(gamma), stamp_base,
              stream)


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
    run_backup(tree, leaves.work, leaves.depth0, d_max, gamma, leaves.stamp_base)
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
