"""Structure-of-arrays belief tree resident in HBM (device mirror of
/root/reference/pkg/src/vecpomdp/tree.py:100-378).

Layout (all device tensors, row-indexed):

    B   b_parent_action i32 | b_parent_obs u32 | b_depth i32 | b_ckey i64
    PSI psi [cap_dense, stride] fp32 (fast) or fp64 (parity), row-major, rows
        padded to 16 B.  Parity mode: row b is belief b's (b_flags bit 0 = row
        still lazily equal to init, bit 1 = row not yet written).  Fast mode: a
        belief's row is the initial row overlaid with <= 4 realised cells kept in
        its 32-B record b_rec {dense_pass, dense_row, action+1 [4], value [4]};
        only beliefs with more than 4 action children own a dense row
        (cap_dense = cap_actions // 5 + 2 rows bound them); b_nact counts the
        children, a_slot is an action's child index
        b_lse f64 (cached LSE of the row) | b_value f64, b_rows i32, b_acc 16 B (pass scratch)
    A   a_parent_belief i32 | a_action i32 | a_reward f64 | a_visits i32 | a_ckey i64
        a_rows i32, a_acc 16 B (pass scratch)
    two open-addressing hash indexes of 16-byte slots, load factor <= 1/2:
        (belief << 32 | action) -> action row, (action row << 32 | obs) -> belief row

Row 0 is the root (parent fields -1).  The device numbers new rows in the
order warps create them; each row carries its creation key (pass, level,
first row), and sorting by it gives the reference's first-occurrence ids
(tree.py:10-12).  Every host-facing accessor (``tables``, ``serialize``,
traces, search frontiers) speaks reference ids; the permutation is computed
on the device (one sort per table) when something is exported.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .core import ROOT_SENTINEL

PRECISIONS = {"fp32": _lib.VP_PSI_F32, "fp64": _lib.VP_PSI_F64}


def _torch():
    return _lib.torch_cuda()


def _pow2_at_least(x: int) -> int:
    p = 1
    while p < x:
        p <<= 1
    return p


def _stream():
    return _torch().cuda.current_stream().cuda_stream


class DeviceTree:
    """B / A / PSI tables of one planning step on the current CUDA device."""

    def __init__(self, action_count: int, init_prefs=None, *, eta: float = 2.0, precision: str = "fp32",
                 exact: bool = False, cap_beliefs: int = 4096, cap_actions: int = 4096, cap_dense: int = 0):
        if action_count < 1:
            raise ValueError("action_count must be >= 1")
        if precision not in PRECISIONS:
            raise ValueError(f"precision must be one of {sorted(PRECISIONS)}")
        if exact and precision != "fp64":
            raise ValueError("exact (numpy-order) mode requires precision='fp64'")
        torch = _torch()
        self.action_count = action_count
        self.precision = precision
        self.exact = bool(exact)
        self.eta = float(eta)
        self.generation = 0
        self.pass_cursor = 0       # last search pass run on this tree (creation keys use it)
        self._canon_cache = None
        self._scratch_dirty = False  # a search ran without its backup
        self.last_search = None
        self._psi_dtype = torch.float32 if precision == "fp32" else torch.float64
        self._counters = torch.zeros(_lib.VP_COUNTERS, dtype=torch.int32, device="cuda")
        self._init_lse = torch.zeros(1, dtype=torch.float64, device="cuda")
        self._init_prefs = torch.zeros(action_count, dtype=torch.float64, device="cuda")
        # PSI rows padded to 16 bytes so they can be TMA bulk-copied (csrc K1)
        per16 = 4 if precision == "fp32" else 2
        self.psi_stride = (action_count + per16 - 1) // per16 * per16
        self._init_cdf = torch.zeros(action_count, dtype=self._psi_dtype, device="cuda")
        self._host_counts = (C.c_int32 * 5)()  # live b, live a, overflow, id extents
        self.cap_beliefs = 0
        self.cap_actions = 0
        self.overlay_slots = 0 if self.exact else _lib.VP_OVERLAY_SLOTS
        self._allocate(max(16, cap_beliefs), max(16, cap_actions), min_dense=cap_dense)
        self.reset(init_prefs, eta)

    # ------------------------------------------------------------------ storage
    def dense_rows_for(self, cap_b: int, cap_a: int) -> int:
        """PSI rows the arena needs: one per belief in parity mode; in fast mode one per
        belief with more than ``overlay_slots`` action children (each owns >= slots + 1 of
        the cap_a actions) plus the root."""
        return cap_b if self.exact else cap_a // (self.overlay_slots + 1) + 2

    def _allocate(self, cap_b: int, cap_a: int, keep_b: int = 0, keep_a: int = 0, keep_dense: int = 0,
                  min_dense: int = 0):
        torch = _torch()
        dev = "cuda"
        A = self.action_count
        if getattr(self, "dense_on_demand", False) and getattr(self, "cap_dense", 0):
            cap_d = max(self.cap_dense, min_dense, keep_dense, 1)  # grown separately (ensure_dense)
        else:
            cap_d = max(self.dense_rows_for(cap_b, cap_a), min_dense, keep_dense, 1)
        rec_words = 8 if self.precision == "fp32" else 12  # sizeof(Rec<PsiT>) / 4 (32 / 48 bytes)

        def col(old, shape, dtype, keep, fill=None):
            # accumulators start at zero and creation keys unset (-1 = ~0): node creation
            # on the device relies on rows beyond the counts being in that state
            new = torch.empty(shape, dtype=dtype, device=dev) if fill is None else \
                torch.full(shape if isinstance(shape, tuple) else (shape,), fill, dtype=dtype, device=dev)
            if old is not None and keep:
                new[:keep] = old[:keep]
            return new

        g = lambda name: getattr(self, name, None)  # noqa: E731
        self.b_parent_action = col(g("b_parent_action"), cap_b, torch.int32, keep_b)
        self.b_parent_obs = col(g("b_parent_obs"), cap_b, torch.int32, keep_b)
        self.b_parent_belief = col(g("b_parent_belief"), cap_b, torch.int32, keep_b)
        self.b_parent_act = col(g("b_parent_act"), cap_b, torch.int32, keep_b)
        self.b_depth = col(g("b_depth"), cap_b, torch.int32, keep_b)
        self.psi = col(g("psi"), (cap_d, self.psi_stride), self._psi_dtype, keep_b if self.exact else keep_dense)
        # fast mode: the softmax CDF of each dense row (rebuilt by the backup)
        self.psi_cdf = col(g("psi_cdf"), (1 if self.exact else cap_d, self.psi_stride), self._psi_dtype,
                           0 if self.exact else keep_dense)
        self.dense_meta = col(g("dense_meta"), (1 if self.exact else cap_d, 2), torch.int64, 0, 0)
        self.b_lse = col(g("b_lse"), cap_b, torch.float64, keep_b)
        self.b_value = col(g("b_value"), cap_b, torch.float64, keep_b, 0)
        self.b_rows = col(g("b_rows"), cap_b, torch.int32, keep_b, 0)
        self.b_acc = col(g("b_acc"), (cap_b, 2), torch.int64, keep_b, 0)
        self.b_flags = col(g("b_flags"), cap_b, torch.int32, keep_b)
        self.b_rec = col(g("b_rec"), (cap_b, rec_words), torch.int32, keep_b, 0)
        self.b_nact = col(g("b_nact"), cap_b, torch.int32, keep_b, 0)
        self.b_ckey = col(g("b_ckey"), cap_b, torch.int64, keep_b, -1)
        self.a_parent_belief = col(g("a_parent_belief"), cap_a, torch.int32, keep_a)
        self.a_action = col(g("a_action"), cap_a, torch.int32, keep_a)
        self.a_reward = col(g("a_reward"), cap_a, torch.float64, keep_a, 0)
        self.a_visits = col(g("a_visits"), cap_a, torch.int32, keep_a, 0)
        self.a_rows = col(g("a_rows"), cap_a, torch.int32, keep_a, 0)
        self.a_acc = col(g("a_acc"), (cap_a, 2), torch.int64, keep_a, 0)
        self.a_ckey = col(g("a_ckey"), cap_a, torch.int64, keep_a, -1)
        self.a_slot = col(g("a_slot"), cap_a, torch.int32, keep_a, 0)
        ha = _pow2_at_least(2 * cap_a)
        hb = _pow2_at_least(2 * cap_b)
        self.hash_a = torch.empty((ha, 2), dtype=torch.int64, device=dev)
        self.hash_b = torch.empty((hb, 2), dtype=torch.int64, device=dev)
        self.cap_beliefs, self.cap_actions, self.cap_dense = cap_b, cap_a, cap_d
        s = _lib.VpTree()
        s.cap_beliefs, s.cap_actions, s.action_count = cap_b, cap_a, A
        s.psi_dtype = PRECISIONS[self.precision]
        s.exact = int(self.exact)
        s.hmask_a, s.hmask_b = ha - 1, hb - 1
        s.psi_stride = self.psi_stride
        for name in ("b_parent_action", "b_parent_obs", "b_parent_belief", "b_parent_act", "b_depth", "psi", "b_lse", "b_value", "b_rows", "b_acc",
                     "b_flags", "b_rec", "b_nact", "b_ckey", "a_parent_belief", "a_action", "a_reward", "a_visits",
                     "a_rows", "a_acc", "a_ckey", "a_slot", "hash_a", "hash_b", "psi_cdf", "dense_meta"):
            setattr(s, name, getattr(self, name).data_ptr())
        s.cap_dense = cap_d
        s.overlay_slots = self.overlay_slots
        s.bkey_mode = getattr(self, "bkey_mode", 0)
        s.init_uniform = getattr(self, "_init_uniform", 0)  # (a regrown arena keeps it)
        s.counters = self._counters.data_ptr()
        s.init_prefs = self._init_prefs.data_ptr()
        s.init_lse = self._init_lse.data_ptr()
        s.init_cdf = self._init_cdf.data_ptr()
        s.eta = self.eta
        self.struct = s

    def set_belief_key_mode(self, mode: int):
        """0: belief index keyed by (action row, obs) -- any |A|, any obs < 2^32; 1: keyed by
        (belief, action, obs) so the search issues a level's two claims together (needs
        |A| <= 4096 and obs codes < 2^20).  Only on an empty index (right after reset)."""
        if mode not in (0, 1):
            raise ValueError("belief key mode must be 0 or 1")
        self.bkey_mode = mode
        self.struct.bkey_mode = mode

    def set_eta(self, eta: float, *, refresh: bool = True):
        """Change eta.  On a live tree the cached per-row LSEs and the initial row's LSE / CDF
        depend on eta, so ``refresh`` recomputes them on the device (the reference tree is
        eta-free: search / backup take eta per call, search.py:86, backup.py:75)."""
        if eta <= 0:
            raise ValueError("eta must be positive")
        changed = float(eta) != self.eta
        self.eta = float(eta)
        self.struct.eta = self.eta
        if changed and refresh:
            _lib.call("vp_tree_set_eta", C.byref(self.struct), _stream())

    def reset(self, init_prefs=None, eta: float | None = None, device_init: bool = True):
        """Fresh tree (tree.py:103-132): root row, no actions, init PSI row.

        ``device_init=False`` leaves the device-side reset to a following
        ``vp_plan`` call (which starts every planning step with it)."""
        torch = _torch()
        if eta is not None:
            self.set_eta(eta, refresh=False)  # the reset below recomputes everything
        A = self.action_count
        base = np.zeros(A) if init_prefs is None else np.asarray(init_prefs, dtype=np.float64)
        if base.shape != (A,) or not np.all(np.isfinite(base)):
            raise ValueError("init_prefs must be a finite vector of length |A|")
        if getattr(self, "init_prefs", None) is None or not np.array_equal(self.init_prefs, base):
            self._init_prefs.copy_(torch.from_numpy(base))
        self.init_prefs = base
        self._init_uniform = self.struct.init_uniform = int(bool(np.all(base == base[0])))
        self.generation += 1
        self.pass_cursor = 0
        self._canon_cache = None
        self._scratch_dirty = False
        self.last_search = None
        if device_init:
            _lib.call("vp_tree_init", C.byref(self.struct), _stream())

    def counts(self):
        """(n_beliefs, n_actions, overflow) -- synchronises the stream."""
        _lib.call("vp_tree_counts", C.byref(self.struct), self._host_counts, _stream())
        return int(self._host_counts[0]), int(self._host_counts[1]), int(self._host_counts[2])

    def extent(self):
        """(belief, action) id extents: the device columns in use.  A search numbers nodes
        statically (row r creating at level l takes extent + l n + r), so ids below the
        extents that no node took are holes (creation key ~0)."""
        self.counts()
        return int(self._host_counts[3]), int(self._host_counts[4])

    def ensure_capacity(self, need_beliefs: int, need_actions: int, limit: int | None = None):
        """Grow (geometric, tree.py:90-97) so the next search cannot overflow."""
        if getattr(self, "dense_on_demand", False) and not self.exact:  # one dense row per new action at most
            self.ensure_dense(self.n_dense() + max(0, need_actions - self.extent()[1]))
        if need_beliefs <= self.cap_beliefs and need_actions <= self.cap_actions:
            return False
        nb, na = self.extent()
        cap_b = max(self.cap_beliefs, 16)
        while cap_b < need_beliefs:
            cap_b *= 2
        cap_a = max(self.cap_actions, 16)
        while cap_a < need_actions:
            cap_a *= 2
        if limit is not None:  # never past what the caller can still use (a fixed budget's total)
            cap_b, cap_a = max(min(cap_b, limit), need_beliefs), max(min(cap_a, limit), need_actions)
        self._allocate(cap_b, cap_a, keep_b=nb, keep_a=na, keep_dense=self.n_dense())
        _lib.call("vp_tree_rehash", C.byref(self.struct), _stream())
        return True

    def ensure_dense(self, need_rows: int) -> bool:
        """Fast mode, iterative plans: grow the dense PSI pool (rows, their CDF rows and CDF
        requests; geometric) so the next pass cannot run out -- a pass makes at most one dense
        row per new action node.  Only the pool is reallocated."""
        if self.exact or need_rows <= self.cap_dense:
            return False
        torch = _torch()
        used = self.n_dense()
        cap = max(self.cap_dense, 16)
        while cap < need_rows:
            cap *= 2
        for name, width, dt in (("psi", self.psi_stride, self._psi_dtype), ("psi_cdf", self.psi_stride, self._psi_dtype),
                                ("dense_meta", 2, torch.int64)):
            old = getattr(self, name)
            new = torch.zeros((cap, width), dtype=dt, device="cuda") if name == "dense_meta" else \
                torch.empty((cap, width), dtype=dt, device="cuda")
            new[:used] = old[:used]
            setattr(self, name, new)
            setattr(self.struct, name, new.data_ptr())
        self.cap_dense = self.struct.cap_dense = cap
        return True

    def dense_bytes_per_row(self) -> int:
        return 2 * self.psi_stride * self._psi_dtype.itemsize + 16

    def n_dense(self) -> int:
        """PSI rows in use (parity mode: the belief count)."""
        if self.exact:
            return self.extent()[0]
        return int(self._counters[_lib.VP_COUNTER_DENSE].item())

    def next_pass(self) -> int:
        """Pass number of the next search on this tree (ckey order, leaf-list parity)."""
        self.pass_cursor += 1
        self._canon_cache = None
        return self.pass_cursor

    def clear_pass_scratch(self):
        """Zero the per-pass counters after a search that was never backed up."""
        if not self._scratch_dirty:
            return
        nb, na = self.extent()
        for t in (self.b_rows, self.b_value, self.b_acc):
            t[:nb].zero_()
        for t in (self.a_rows, self.a_acc):
            t[:na].zero_()
        self._scratch_dirty = False

    def canonical(self):
        """(b_order, b_rank, a_order, a_rank) device tensors: ``order[k]`` is the
        device row of reference id k, ``rank[row]`` its reference id."""
        nb, na, _ = self.counts()
        hb, ha = int(self._host_counts[3]), int(self._host_counts[4])
        key = (self.generation, self.pass_cursor, nb, na, hb, ha)
        if self._canon_cache is not None and self._canon_cache[0] == key:
            return self._canon_cache[1]
        torch = _torch()
        out = []
        for ck, cnt, ext in ((self.b_ckey, nb, hb), (self.a_ckey, na, ha)):
            # holes keep ckey ~0 (-1 as int64) and sort first; live keys are >= 0
            order = torch.argsort(ck[:ext], stable=True).to(torch.int64)[ext - cnt:]
            rank = torch.full((ext,), -1, device=order.device, dtype=torch.int64)
            rank[order] = torch.arange(cnt, device=order.device, dtype=torch.int64)
            out += [order, rank]
        self._canon_cache = (key, tuple(out))
        return self._canon_cache[1]

    def to_reference_beliefs(self, rows):
        """Device belief rows -> reference belief ids (numpy or torch input)."""
        torch = _torch()
        _, brank, _, _ = self.canonical()
        t = torch.as_tensor(np.asarray(rows, dtype=np.int64) if not torch.is_tensor(rows) else rows,
                            device="cuda").to(torch.int64)
        return brank[t]

    def to_reference_actions(self, rows):
        torch = _torch()
        _, _, _, arank = self.canonical()
        t = torch.as_tensor(np.asarray(rows, dtype=np.int64) if not torch.is_tensor(rows) else rows,
                            device="cuda").to(torch.int64)
        return arank[t]

    def to_device_beliefs(self, ids):
        """Reference belief ids -> device rows."""
        torch = _torch()
        border, _, _, _ = self.canonical()
        t = torch.as_tensor(np.asarray(ids, dtype=np.int64), device="cuda")
        return border[t]

    # ------------------------------------------------------------------ host-level mutation (tree.py:180-265)
    def _append(self, fn: str, ids_dev, labels, extra, n: int):
        torch = _torch()
        out = torch.empty(n, dtype=torch.int32, device="cuda")
        args = [C.byref(self.struct), ids_dev.data_ptr(), labels.data_ptr()]
        if extra is not None:
            args.append(extra.data_ptr())
        _lib.call(fn, *args, n, self.next_pass(), out.data_ptr(), _stream())
        return out

    def append_actions(self, belief_indices, actions, rewards) -> np.ndarray:
        """tree.py:180-218 on the device: resolve (belief, action) edges -- new nodes numbered
        n_actions + rank in first-occurrence order -- and add each row's reward and one visit.
        Reference ids in and out."""
        torch = _torch()
        b = np.asarray(belief_indices, dtype=np.int64)
        a = np.asarray(actions, dtype=np.int64)
        r = np.asarray(rewards, dtype=np.float64)
        if not (len(b) == len(a) == len(r)):
            raise ValueError("append_actions: batch lengths differ")
        nb, na, _ = self.counts()
        if len(b) and (b.min() < 0 or b.max() >= nb):
            raise ValueError("append_actions: invalid belief index")
        if len(a) and (a.min() < 0 or a.max() >= self.action_count):
            raise ValueError("append_actions: actions must be in [0, |A|)")
        if not len(b):
            return np.zeros(0, dtype=np.int64)
        self.ensure_capacity(nb, na + len(b))
        dev_b = self.to_device_beliefs(b).to(torch.int32)
        out = self._append("vp_tree_append_actions", dev_b, torch.from_numpy(a.astype(np.int32)).cuda(),
                           torch.from_numpy(r).cuda(), len(b))
        if self.counts()[2]:
            raise _lib.CapacityError("action table overflow")
        _lib.call("vp_tree_build_cdfs", C.byref(self.struct), _stream())  # rows made dense by the edit
        return self.to_reference_actions(out.to(torch.int64)).cpu().numpy()

    def append_beliefs(self, action_node_indices, observations) -> np.ndarray:
        """tree.py:220-256 on the device: resolve (action node, observation) edges; new beliefs
        get depth = parent depth + 1 and the initial PSI row (lazily).  Reference ids in and out."""
        torch = _torch()
        x = np.asarray(action_node_indices, dtype=np.int64)
        o = np.asarray(observations, dtype=np.int64)
        if len(x) != len(o):
            raise ValueError("append_beliefs: batch lengths differ")
        nb, na, _ = self.counts()
        if len(x) and (x.min() < 0 or x.max() >= na):
            raise ValueError("append_beliefs: invalid action-node index")
        if len(o) and (o.min() < 0 or o.max() >= 1 << 32):
            raise ValueError("pair entries must be in [0, 2**32)")
        if not len(x):
            return np.zeros(0, dtype=np.int64)
        self.ensure_capacity(nb + len(x), na)
        _, _, aorder, _ = self.canonical()
        dev_x = aorder[torch.from_numpy(x).cuda()].to(torch.int32)
        out = self._append("vp_tree_append_beliefs", dev_x, torch.from_numpy(o.astype(np.uint32).view(np.int32)).cuda(),
                           None, len(x))
        if self.counts()[2]:
            raise _lib.CapacityError("belief table overflow")
        return self.to_reference_beliefs(out.to(torch.int64)).cpu().numpy()

    def nodes_at_depth(self, d: int):
        """Beliefs at depth d with their parent action and grandparent belief (tree.py:258-265),
        reference ids."""
        if d < 1:
            raise ValueError("nodes_at_depth requires d >= 1")
        t = self.tables()
        bel = np.flatnonzero(t["depth"] == d)
        par = t["parent_action"][bel]
        grand = t["action_parent_belief"][par] if len(par) else par
        return bel, par, grand

    @classmethod
    def deserialize(cls, text: str, *, eta: float = 2.0, precision: str = "fp32") -> "DeviceTree":
        """Inverse of ``serialize`` (tree.py:322-368): the B / A / P rows become device columns
        (reference ids = device ids), the hash indexes are rebuilt on the device."""
        torch = _torch()
        b_rows, a_rows, p_rows = [], [], []
        for line in text.splitlines():
            if not line.strip():
                continue
            parts = line.split("\t")
            if parts[0] == "B":
                b_rows.append([int(v) for v in parts[1:5]])
            elif parts[0] == "A":
                a_rows.append((int(parts[1]), int(parts[2]), int(parts[3]), float(parts[4]), int(parts[5])))
            elif parts[0] == "P":
                p_rows.append((int(parts[1]), [float(v) for v in parts[3:]]))
            else:
                raise ValueError(f"unknown row tag {parts[0]!r}")
        if not b_rows or b_rows[0][0] != 0:
            raise ValueError("serialized tree must start with belief row 0")
        A = len(p_rows[0][1])
        nb, na = len(b_rows), len(a_rows)
        tree = cls(A, eta=eta, precision=precision, cap_beliefs=max(16, nb), cap_actions=max(16, na),
                   cap_dense=nb)
        prefs = np.zeros((nb, A))
        for row, vals in p_rows:
            prefs[row] = vals
        pa = np.array([r[1] for r in b_rows], dtype=np.int64)
        apb = np.array([r[1] for r in a_rows], dtype=np.int64)
        act = np.array([r[2] for r in a_rows], dtype=np.int64)
        dev = lambda v, dt: torch.as_tensor(np.asarray(v), device="cuda").to(dt)  # noqa: E731
        tree.b_parent_action[:nb] = dev(np.where(pa >= 0, pa, -1), torch.int32)
        tree.b_parent_obs[:nb] = dev(np.array([r[2] for r in b_rows], dtype=np.int64).astype(np.uint32).view(np.int32),
                                     torch.int32)
        tree.b_depth[:nb] = dev([r[3] for r in b_rows], torch.int32)
        tree.b_parent_belief[:nb] = dev(np.where(pa >= 0, apb[np.maximum(pa, 0)] if na else -1, -1), torch.int32)
        tree.b_parent_act[:nb] = dev(np.where(pa >= 0, act[np.maximum(pa, 0)] if na else 0, 0), torch.int32)
        tree.psi[:nb, :A] = dev(prefs, tree._psi_dtype)
        tree.b_lse[:nb] = dev(np.max(eta * prefs, axis=1) / eta
                              + np.log(np.exp(eta * prefs - np.max(eta * prefs, axis=1)[:, None]).sum(axis=1)) / eta,
                              torch.float64)
        tree.b_flags[:nb] = 0  # every row is written
        if not tree.exact:  # fast mode: every belief owns its dense row (row = id)
            tree.b_rec[:nb] = 0
            tree.b_rec[:nb, 0] = 1
            tree.b_rec[:nb, 1] = torch.arange(nb, device="cuda", dtype=torch.int32)
            tree.b_nact[:nb] = tree.overlay_slots + 1
            tree._counters[_lib.VP_COUNTER_DENSE] = nb
        tree.b_ckey[:nb] = torch.arange(nb, device="cuda", dtype=torch.int64)  # canonical order = ids
        if na:
            tree.a_parent_belief[:na] = dev(apb, torch.int32)
            tree.a_action[:na] = dev(act, torch.int32)
            tree.a_reward[:na] = dev([r[3] for r in a_rows], torch.float64)
            tree.a_visits[:na] = dev([r[4] for r in a_rows], torch.int32)
            tree.a_ckey[:na] = torch.arange(na, device="cuda", dtype=torch.int64)
        tree._counters[0], tree._counters[_lib.VP_COUNTER_ACTIONS], tree._counters[2] = nb, na, 0
        tree._counters[_lib.VP_COUNTER_LIVE_B], tree._counters[_lib.VP_COUNTER_LIVE_A] = nb, na
        _lib.call("vp_tree_rehash", C.byref(tree.struct), _stream())
        _lib.call("vp_tree_build_cdfs", C.byref(tree.struct), _stream())  # every row is dense here
        tree.pass_cursor = 1
        tree._canon_cache = None
        return tree

    # ------------------------------------------------------------------ reference-style accessors
    @property
    def n_beliefs(self) -> int:
        return self.counts()[0]

    @property
    def n_actions(self) -> int:
        return self.counts()[1]

    # the reference's column properties (tree.py:136-166), host arrays in reference order
    parent_action = property(lambda s: s.tables()["parent_action"])
    parent_obs = property(lambda s: s.tables()["parent_obs"])
    depth = property(lambda s: s.tables()["depth"])
    prefs = property(lambda s: s.tables()["prefs"])
    action_parent_belief = property(lambda s: s.tables()["action_parent_belief"])
    action_id = property(lambda s: s.tables()["action_id"])
    action_reward_sum = property(lambda s: s.tables()["action_reward_sum"])
    action_visits = property(lambda s: s.tables()["action_visits"])

    def tables(self) -> dict:
        """All columns as host numpy arrays (int64 / float64 like the reference),
        rows in reference (first-occurrence) order."""
        torch = _torch()
        nb, na, _ = self.counts()
        border, brank, aorder, arank = self.canonical()
        hb, ha = int(self._host_counts[3]), int(self._host_counts[4])  # (canonical() refreshed them)
        pa = self.b_parent_action[:hb].to(torch.int64)[border]
        pa = torch.where(pa >= 0, arank[pa.clamp(min=0)], pa)
        obs = self.b_parent_obs[:hb][border].cpu().numpy().view(np.uint32).astype(np.int64)
        if nb:
            obs[0] = ROOT_SENTINEL
        prefs = self._prefs_rows(hb)[border].cpu().numpy().astype(np.float64)
        apb = brank[self.a_parent_belief[:ha].to(torch.int64)[aorder]] if na else torch.zeros(0, dtype=torch.int64)
        return {
            "parent_action": pa.cpu().numpy(),
            "parent_obs": obs,
            "depth": self.b_depth[:hb][border].cpu().numpy().astype(np.int64),
            "prefs": prefs,
            "action_parent_belief": apb.cpu().numpy().astype(np.int64),
            "action_id": self.a_action[:ha][aorder].cpu().numpy().astype(np.int64),
            "action_reward_sum": self.a_reward[:ha][aorder].cpu().numpy().copy(),
            "action_visits": self.a_visits[:ha][aorder].cpu().numpy().astype(np.int64),
        }


    def _prefs_rows(self, nb: int):
        """[nb, |A|] PSI rows in device order, the dtype of the tree."""
        torch = _torch()
        A = self.action_count
        init = self._init_prefs.to(self._psi_dtype)[None, :]
        if self.exact:  # lazily initialised rows read as the initial row (tree.py:253)
            fresh = (self.b_flags[:nb] & 1).bool()[:, None]
            return torch.where(fresh, init, self.psi[:nb, :A])
        rec = self.b_rec[:nb]
        dense_pass, dense_row = rec[:, 0], rec[:, 1].to(torch.int64)
        act = rec[:, 2:4].contiguous().view(torch.int16).to(torch.int64) & 0xFFFF  # action + 1, 0 = empty
        val = rec[:, 4:].contiguous().view(self._psi_dtype)[:, : self.overlay_slots]
        rows = init.expand(nb, A).clone()
        dense = dense_pass != 0
        if bool(dense.any()):
            rows[dense] = self.psi[dense_row[dense], :A]
        for k in range(self.overlay_slots):
            m = (act[:, k] > 0) & ~dense
            if bool(m.any()):
                idx = torch.nonzero(m).squeeze(1)
                rows[idx, act[idx, k] - 1] = val[idx, k]
        return rows

    def root_prefs(self) -> np.ndarray:
        return self.psi[0, : self.action_count].cpu().numpy().astype(np.float64)

    def stats(self) -> dict:
        nb, na, _ = self.counts()
        return {"belief_rows": nb, "action_rows": na}

    def validate(self):
        """Full-table invariants (tree.py:269-291) on the downloaded tables."""
        t = self.tables()
        nb, na = len(t["depth"]), len(t["action_id"])
        assert nb >= 1 and t["parent_action"][0] == ROOT_SENTINEL
        assert t["parent_obs"][0] == ROOT_SENTINEL and t["depth"][0] == 0
        if nb > 1:
            pa = t["parent_action"][1:]
            assert pa.min() >= 0 and pa.max() < na
            keys = (pa << 32) | t["parent_obs"][1:]
            assert len(np.unique(keys)) == nb - 1, "duplicate belief edge"
            assert np.all(t["depth"][1:] == t["depth"][t["action_parent_belief"][pa]] + 1)
        if na:
            pb = t["action_parent_belief"]
            assert pb.min() >= 0 and pb.max() < nb
            assert len(np.unique((pb << 32) | t["action_id"])) == na, "duplicate action edge"
            assert t["action_visits"].min() >= 1
            assert np.all(np.isfinite(t["action_reward_sum"]))
        assert np.all(np.isfinite(t["prefs"]))

    def serialize(self) -> str:
        """Text dump in the reference format (tree.py:298-320)."""
        t = self.tables()
        out = ["B\t%d\t%d\t%d\t%d" % (i, t["parent_action"][i], t["parent_obs"][i], t["depth"][i])
               for i in range(len(t["depth"]))]
        out += ["A\t%d\t%d\t%d\t%r\t%d" % (i, t["action_parent_belief"][i], t["action_id"][i],
                                          float(t["action_reward_sum"][i]), t["action_visits"][i])
                for i in range(len(t["action_id"]))]
        out += ["P\t%d\t%d\t%s" % (i, i, "\t".join(repr(float(v)) for v in t["prefs"][i]))
                for i in range(len(t["depth"]))]
        return "\n".join(out) + "\n"


class TreeHandle:
    """What ``PlanOutcome.tree`` holds when the planner reuses pooled storage:
    valid until the pool's next ``plan()`` resets the tree (then it raises
    instead of silently showing the next step's tree)."""

    def __init__(self, tree: DeviceTree):
        self._tree = tree
        self._generation = tree.generation

    def __getattr__(self, name):
        tree = self.__dict__["_tree"]
        if tree.generation != self.__dict__["_generation"]:
            raise RuntimeError("this plan's device tree was recycled by a later plan() call; "
                               "pass keep_tree=True to keep it")
        return getattr(tree, name)


def match_or_append_pairs(existing_keys, query_keys):
    """tree.py:71-87 on the device: resolve (k, 2) integer pairs against a table whose row
    index is the pair's position, appending unseen ones -- new rows k, k+1, ... in
    first-occurrence order of the batch.  Returns (row per query, number of new rows)."""
    torch = _torch()
    ex = np.asarray(existing_keys, dtype=np.int64).reshape(-1, 2)
    q = np.asarray(query_keys, dtype=np.int64).reshape(-1, 2)
    for arr in (ex, q):
        if arr.size and (arr.min() < 0 or arr.max() >= 1 << 32):
            raise ValueError("pair entries must be in [0, 2**32)")
    enc = lambda a: (torch.as_tensor(a[:, 0], device="cuda") << 32) | torch.as_tensor(a[:, 1], device="cuda")  # noqa: E731
    k = len(ex)
    if not len(q):
        return np.zeros(0, dtype=np.int64), 0
    qk = enc(q)
    uq, inv = torch.unique(qk, sorted=True, return_inverse=True)
    row = torch.full((len(uq),), -1, dtype=torch.int64, device="cuda")
    if k:
        ek = enc(ex)
        es, eo = torch.sort(ek, stable=True)
        pos = torch.searchsorted(es, uq).clamp(max=k - 1)
        hit = es[pos] == uq
        row = torch.where(hit, eo[pos], row)
    miss = row < 0
    first = torch.full((len(uq),), len(q), dtype=torch.int64, device="cuda")
    first.scatter_reduce_(0, inv, torch.arange(len(q), device="cuda"), reduce="amin")
    order = torch.argsort(torch.where(miss, first, torch.full_like(first, len(q) + 1)), stable=True)
    n_new = int(miss.sum())
    rank = torch.empty_like(order)
    rank[order] = torch.arange(len(uq), device="cuda")
    row = torch.where(miss, k + rank, row)
    return row[inv].cpu().numpy(), n_new


def init_tree(spec, init_prefs=None, *, eta: float = 2.0, precision: str = "fp32", exact: bool = False,
              cap_beliefs: int = 4096, cap_actions: int = 4096) -> DeviceTree:
    """Device counterpart of tree.init_tree (tree.py:370-378)."""
    return DeviceTree(spec.action_count, init_prefs, eta=eta, precision=precision, exact=exact,
                      cap_beliefs=cap_beliefs, cap_actions=cap_actions)
