"""Columnar belief tree (oracle restatement -- test infrastructure only).

Restates /root/reference/pkg/src/vecpomdp/tree.py:

* belief table B: parent action row, parent observation, depth; root is row 0
  with -1 sentinels (tree.py:114-120);
* action table A: parent belief row, action id, reward sum, visit count
  (tree.py:122-126);
* preference table PSI: one |A|-row per belief (tree.py:119);
* edge keys are (first << 32) | second (tree.py:25-36);
* unseen keys of a batch get consecutive ids in FIRST-OCCURRENCE order of the
  batch, duplicates share one id (tree.py:44-68).

The edge index keeps a sorted (key, row) pair of arrays, as the reference
does, so the CPU baseline built from this oracle has the reference's cost
profile.
"""

from __future__ import annotations

import numpy as np

SENTINEL = -1
_SHIFT = np.int64(32)
_LIMIT = np.int64(1) << _SHIFT


def pack_edge(first, second) -> np.ndarray:
    """(first << 32) | second with range checks (tree.py:25-36)."""
    hi = np.asarray(first, dtype=np.int64)
    lo = np.asarray(second, dtype=np.int64)
    if hi.size and (min(hi.min(), lo.min()) < 0 or max(hi.max(), lo.max()) >= _LIMIT):
        raise ValueError("pair entries must be in [0, 2**32)")
    return (hi << _SHIFT) | lo


def unpack_edge(keys):
    k = np.asarray(keys, dtype=np.int64)
    return k >> _SHIFT, k & (_LIMIT - 1)


class EdgeIndex:
    """Sorted key -> row map with first-occurrence batch resolution."""

    def __init__(self):
        self.keys = np.empty(0, dtype=np.int64)
        self.rows = np.empty(0, dtype=np.int64)

    def resolve(self, queries: np.ndarray, next_row: int):
        """Rows for each query; new keys numbered from next_row (tree.py:44-68)."""
        uniq, first_at, back = np.unique(queries, return_index=True, return_inverse=True)
        n_known = len(self.keys)
        where = np.searchsorted(self.keys, uniq)
        found = np.zeros(len(uniq), dtype=bool)
        if n_known:
            clipped = np.minimum(where, n_known - 1)
            found = (where < n_known) & (self.keys[clipped] == uniq)
        out = np.empty(len(uniq), dtype=np.int64)
        if n_known:
            out[found] = self.rows[clipped[found]]
        missing = np.flatnonzero(~found)
        missing = missing[np.argsort(first_at[missing], kind="stable")]
        out[missing] = next_row + np.arange(len(missing), dtype=np.int64)
        return out[back], uniq[missing]

    def add(self, new_keys: np.ndarray, first_row: int):
        """Merge keys whose rows are first_row, first_row+1, ... (tree.py:170-178)."""
        if not len(new_keys):
            return
        order = np.argsort(new_keys, kind="stable")
        ins = np.searchsorted(self.keys, new_keys[order])
        self.keys = np.insert(self.keys, ins, new_keys[order])
        self.rows = np.insert(self.rows, ins, first_row + order.astype(np.int64))


def match_or_append_pairs(existing_keys, query_keys):
    """Pure batch resolution against an explicit pair table (tree.py:71-87)."""
    ex = np.asarray(existing_keys, dtype=np.int64).reshape(-1, 2)
    q = np.asarray(query_keys, dtype=np.int64).reshape(-1, 2)
    idx = EdgeIndex()
    idx.add(pack_edge(ex[:, 0], ex[:, 1]), 0)
    rows, new = idx.resolve(pack_edge(q[:, 0], q[:, 1]), len(ex))
    return rows, len(new)


def _ensure(arr: np.ndarray, need: int) -> np.ndarray:
    """Geometric capacity growth (tree.py:90-97)."""
    if need <= len(arr):
        return arr
    grown = np.empty((max(need, 2 * len(arr), 16),) + arr.shape[1:], dtype=arr.dtype)
    grown[: len(arr)] = arr
    return grown


class ColumnarTree:
    """B / A / PSI tables of one planning step (tree.py:100-132)."""

    def __init__(self, action_count: int, init_prefs=None):
        if action_count < 1:
            raise ValueError("action_count must be >= 1")
        base = np.zeros(action_count) if init_prefs is None else np.asarray(init_prefs, dtype=np.float64)
        if base.shape != (action_count,) or not np.all(np.isfinite(base)):
            raise ValueError("init_prefs must be a finite vector of length |A|")
        self.action_count = action_count
        self.init_prefs = base
        self.n_beliefs = 1
        self.n_actions = 0
        self._pa = np.full(16, SENTINEL, dtype=np.int64)
        self._po = np.full(16, SENTINEL, dtype=np.int64)
        self._dep = np.zeros(16, dtype=np.int64)
        self._psi = np.zeros((16, action_count))
        self._psi[0] = base
        self._apb = np.empty(16, dtype=np.int64)
        self._aid = np.empty(16, dtype=np.int64)
        self._arew = np.empty(16)
        self._avis = np.empty(16, dtype=np.int64)
        self._aindex = EdgeIndex()
        self._bindex = EdgeIndex()

    # trimmed views (tree.py:136-166)
    parent_action = property(lambda s: s._pa[: s.n_beliefs])
    parent_obs = property(lambda s: s._po[: s.n_beliefs])
    depth = property(lambda s: s._dep[: s.n_beliefs])
    prefs = property(lambda s: s._psi[: s.n_beliefs])
    action_parent_belief = property(lambda s: s._apb[: s.n_actions])
    action_id = property(lambda s: s._aid[: s.n_actions])
    action_reward_sum = property(lambda s: s._arew[: s.n_actions])
    action_visits = property(lambda s: s._avis[: s.n_actions])

    def append_actions(self, beliefs, actions, rewards) -> np.ndarray:
        """Resolve (belief, action) edges; accumulate reward/visits (tree.py:180-218)."""
        b = np.asarray(beliefs, dtype=np.int64)
        a = np.asarray(actions, dtype=np.int64)
        r = np.asarray(rewards, dtype=np.float64)
        if not (len(b) == len(a) == len(r)):
            raise ValueError("append_actions: batch lengths differ")
        if len(b) and (b.min() < 0 or b.max() >= self.n_beliefs):
            raise ValueError("append_actions: invalid belief index")
        rows, fresh = self._aindex.resolve(pack_edge(b, a), self.n_actions)
        if len(fresh):
            lo, hi = self.n_actions, self.n_actions + len(fresh)
            self._apb = _ensure(self._apb, hi)
            self._aid = _ensure(self._aid, hi)
            self._arew = _ensure(self._arew, hi)
            self._avis = _ensure(self._avis, hi)
            self._apb[lo:hi], self._aid[lo:hi] = unpack_edge(fresh)
            self._arew[lo:hi] = 0.0
            self._avis[lo:hi] = 0
            self.n_actions = hi
            self._aindex.add(fresh, lo)
        np.add.at(self._arew, rows, r)
        np.add.at(self._avis, rows, 1)
        return rows

    def append_beliefs(self, action_nodes, observations) -> np.ndarray:
        """Resolve (action node, observation) edges (tree.py:220-256)."""
        an = np.asarray(action_nodes, dtype=np.int64)
        ob = np.asarray(observations, dtype=np.int64)
        if len(an) != len(ob):
            raise ValueError("append_beliefs: batch lengths differ")
        if len(an) and (an.min() < 0 or an.max() >= self.n_actions):
            raise ValueError("append_beliefs: invalid action-node index")
        rows, fresh = self._bindex.resolve(pack_edge(an, ob), self.n_beliefs)
        if len(fresh):
            lo, hi = self.n_beliefs, self.n_beliefs + len(fresh)
            self._pa = _ensure(self._pa, hi)
            self._po = _ensure(self._po, hi)
            self._dep = _ensure(self._dep, hi)
            self._psi = _ensure(self._psi, hi)
            pa, obs = unpack_edge(fresh)
            self._pa[lo:hi] = pa
            self._po[lo:hi] = obs
            self._dep[lo:hi] = self._dep[self._apb[pa]] + 1
            self._psi[lo:hi] = self.init_prefs
            self.n_beliefs = hi
            self._bindex.add(fresh, lo)
        return rows

    def nodes_at_depth(self, d: int):
        """Beliefs at depth d with parent / grandparent rows (tree.py:258-265)."""
        if d < 1:
            raise ValueError("nodes_at_depth requires d >= 1")
        bel = np.flatnonzero(self.depth == d)
        par = self.parent_action[bel]
        grand = self.action_parent_belief[par] if len(par) else par
        return bel, par, grand

    def validate(self):
        """Full-table invariants (tree.py:269-291)."""
        nb, na = self.n_beliefs, self.n_actions
        assert nb >= 1 and self.parent_action[0] == SENTINEL
        assert self.parent_obs[0] == SENTINEL and self.depth[0] == 0
        if nb > 1:
            pa = self.parent_action[1:]
            assert pa.min() >= 0 and pa.max() < na
            assert len(np.unique(pack_edge(pa, self.parent_obs[1:]))) == nb - 1
            assert np.all(self.depth[1:] == self.depth[self.action_parent_belief[pa]] + 1)
        if na:
            pb = self.action_parent_belief
            assert pb.min() >= 0 and pb.max() < nb
            assert len(np.unique(pack_edge(pb, self.action_id))) == na
            assert self.action_visits.min() >= 1
            assert np.all(np.isfinite(self.action_reward_sum))
        assert np.all(np.isfinite(self.prefs))

    def stats(self) -> dict:
        return {"belief_rows": self.n_beliefs, "action_rows": self.n_actions}

    def tables(self) -> dict:
        """All columns as plain arrays (the diff medium used by the tests)."""
        return {
            "parent_action": self.parent_action.copy(),
            "parent_obs": self.parent_obs.copy(),
            "depth": self.depth.copy(),
            "prefs": self.prefs.copy(),
            "action_parent_belief": self.action_parent_belief.copy(),
            "action_id": self.action_id.copy(),
            "action_reward_sum": self.action_reward_sum.copy(),
            "action_visits": self.action_visits.copy(),
        }

    def serialize(self) -> str:
        """Tab-separated text dump in the reference's format (tree.py:298-320)."""
        out = ["B\t%d\t%d\t%d\t%d" % (i, self._pa[i], self._po[i], self._dep[i])
               for i in range(self.n_beliefs)]
        out += ["A\t%d\t%d\t%d\t%r\t%d" % (i, self._apb[i], self._aid[i], float(self._arew[i]), self._avis[i])
                for i in range(self.n_actions)]
        out += ["P\t%d\t%d\t%s" % (i, i, "\t".join(repr(float(v)) for v in self._psi[i]))
                for i in range(self.n_beliefs)]
        return "\n".join(out) + "\n"


def init_tree(spec, init_prefs=None) -> ColumnarTree:
    """tree.py:370-378."""
    return ColumnarTree(spec.action_count, init_prefs)
