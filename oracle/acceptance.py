"""Acceptance oracles of the reference (SPEC.md ACCEPTANCE CRITERIA 1, 4, 5) --
TEST INFRASTRUCTURE ONLY (never imported by the product).

Restates /root/reference/pkg/src/vecpomdp/oracle.py:

* ``PathTree`` + ``serial_backup`` (oracle.py:37-97, 124-173): the per-node,
  per-level preference backup over a linked tree.  Nodes are keyed by their
  path from the root -- a tuple (a1, o1, a2, o2, ...) -- so trees built in
  different orders (episode by episode, level by level, on the device) compare
  node by node without renumbering.
* ``exact_value_iteration`` (oracle.py:212-310): finite-horizon optimal value of
  a tabular POMDP as a set of alpha vectors; each backup is the cross-sum over
  observations of the back-projected vectors, pruned to the vectors that are
  strictly best somewhere on the belief simplex (an LP witness per candidate,
  Lark's filter; scipy HiGHS).
* ``exact_bayes_filter`` (oracle.py:313-323): b'(s') ∝ Z[a, s', o] Σ_s T[a, s, s'] b(s).

Parity: pinned against the real reference's outputs by
tests/golden/make_golden.py (``acceptance.npz``; tests/test_oracle_golden.py).
"""

from __future__ import annotations

import math

import numpy as np


# ------------------------------------------------------------------ serial backup (SPEC #1)


class PathTree:
    """Beliefs and actions keyed by their root path (oracle.py:37-97).

    belief path: (a1, o1, ..., ad, od); action path: belief path + (a,).
    """

    def __init__(self, action_count: int, init_prefs=None):
        self.A = action_count
        self.init = np.zeros(action_count) if init_prefs is None else np.asarray(init_prefs, dtype=np.float64)
        self.prefs = {(): self.init.astype(np.float64).tolist()}
        self.reward = {}   # action path -> reward sum
        self.visits = {}   # action path -> lifetime visits
        self.children = {}  # action path -> list of child belief paths (creation order)

    def add_row(self, actions, observations, rewards):
        """One simulated row: the path's nodes are created on first sight, each
        traversed action gains the row's reward and one visit (tree.py:180-256)."""
        b = ()
        for a, o, r in zip(actions, observations, rewards):
            x = b + (int(a),)
            if x not in self.reward:
                self.reward[x], self.visits[x], self.children[x] = 0.0, 0, []
            self.reward[x] += float(r)
            self.visits[x] += 1
            c = x + (int(o),)
            if c not in self.prefs:
                self.prefs[c] = self.init.tolist()
                self.children[x].append(c)
            b = c
        return b


def _lse(prefs, eta: float) -> float:
    top = max(prefs)
    return top + math.log(math.fsum(math.exp(eta * (p - top)) for p in prefs)) / eta


def serial_backup(tree: PathTree, leaves, d_max: int, eta: float, gamma: float) -> None:
    """oracle.py:124-173 over a PathTree; ``leaves`` = [(belief path, heuristic)].

    Level d = d_max..1: the valued beliefs at depth d (the leaves of this batch,
    then the parents valued at the level below) determine their parent actions;
    Q(x) = R(x)/visits(x) + gamma * Σ V N / Σ N over x's valued children; every
    parent belief b is shifted by Q - LSE_pre(b) on its valued actions, then
    V(b) = LSE_post(b), N(b) = Σ lifetime visits of those actions.
    """
    value, weight = {}, {}
    sums, counts = {}, {}
    for path, h in leaves:
        sums[path] = sums.get(path, 0.0) + float(h)
        counts[path] = counts.get(path, 0) + 1
    for path in counts:
        value[path] = sums[path] / counts[path]
        weight[path] = float(counts[path])
    for d in range(d_max, 0, -1):
        level = [p for p in weight if len(p) == 2 * d and weight[p] > 0]
        if not level:
            continue
        acts = sorted({p[:-1] for p in level})
        q = {}
        for x in acts:
            kids = [c for c in tree.children[x] if weight.get(c, 0.0) > 0]
            num = sum(value[c] * weight[c] for c in kids)
            den = sum(weight[c] for c in kids)
            q[x] = tree.reward[x] / tree.visits[x] + gamma * num / den
        parents = sorted({x[:-1] for x in acts})
        pre = {b: _lse(tree.prefs[b], eta) for b in parents}
        for x in acts:
            tree.prefs[x[:-1]][x[-1]] += q[x] - pre[x[:-1]]
        for b in parents:
            value[b] = _lse(tree.prefs[b], eta)
            weight[b] = float(sum(tree.visits[x] for x in acts if x[:-1] == b))


def random_tree_case(rng: np.random.Generator, max_beliefs: int = 50, max_actions: int = 6):
    """One random backup case in the SPEC #1 family (depth <= 4, <= 50 beliefs, |A| <= 6,
    random rewards / heuristics): 1-3 passes of n rows x d levels of (action, observation,
    reward) and a leaf heuristic per row.  Returns (A, passes) with passes a list of
    dicts {d, actions[d, n], observations[d, n], rewards[d, n], leaf[n]}."""
    A = int(rng.integers(2, max_actions + 1))
    O = int(rng.integers(1, 4))
    n_pass = int(rng.integers(1, 4))
    passes, budget = [], max_beliefs - 1
    for k in range(n_pass):
        d = int(rng.integers(1, 5))
        n = int(rng.integers(1, max(2, budget // d) + 1))
        n = max(1, min(n, budget // d))
        if budget < d:
            break
        budget -= n * d
        p = rng.dirichlet(np.full(A, 0.7))  # concentrated policies share nodes
        passes.append({
            "d": d,
            "actions": rng.choice(A, size=(d, n), p=p).astype(np.int32),
            "observations": rng.integers(0, O, size=(d, n)).astype(np.int32),
            "rewards": np.round(rng.uniform(-5.0, 5.0, size=(d, n)), 3),
            "leaf": np.round(rng.normal(0.0, 10.0, size=n), 3),
        })
    return A, passes


def serial_run(A: int, passes, eta: float, gamma: float) -> PathTree:
    """The case's passes applied to a PathTree: each pass inserts its rows, then one
    serial_backup with the rows' leaves."""
    tree = PathTree(A)
    for p in passes:
        leaves = []
        for r in range(p["actions"].shape[1]):
            path = tree.add_row(p["actions"][:, r], p["observations"][:, r], p["rewards"][:, r])
            leaves.append((path, p["leaf"][r]))
        serial_backup(tree, leaves, p["d"], eta, gamma)
    return tree


def belief_paths(parent_action, parent_obs, action_parent_belief, action_id):
    """Root paths of every belief of a columnar tree (tree.py column layout)."""
    paths = [()]
    for b in range(1, len(parent_action)):
        x = int(parent_action[b])
        paths.append(paths[int(action_parent_belief[x])] + (int(action_id[x]), int(parent_obs[b])))
    return paths


# ------------------------------------------------------------------ exact value iteration (SPEC #4)


class AlphaSet:
    """max over alpha vectors, each tagged with its first action (oracle.py:212-224)."""

    def __init__(self, alphas: np.ndarray, actions: np.ndarray):
        self.alphas, self.actions = alphas, actions

    def value(self, belief) -> float:
        return float(np.max(self.alphas @ np.asarray(belief, dtype=np.float64)))

    def action(self, belief) -> int:
        return int(self.actions[int(np.argmax(self.alphas @ np.asarray(belief, dtype=np.float64)))])

    def q_values(self, belief) -> np.ndarray:
        """Best value per first action (−inf for an action without a vector)."""
        v = self.alphas @ np.asarray(belief, dtype=np.float64)
        out = np.full(int(self.actions.max()) + 1, -np.inf)
        np.maximum.at(out, self.actions, v)
        return out


def _witness(v: np.ndarray, others: np.ndarray, tol: float):
    """A belief where v beats every vector of ``others`` by more than tol, or None
    (maximise delta s.t. (w - v)·b + delta <= 0, b in the simplex)."""
    from scipy.optimize import linprog

    s = len(v)
    c = np.zeros(s + 1)
    c[-1] = -1.0
    a_ub = np.hstack([others - v[None, :], np.ones((len(others), 1))])
    a_eq = np.hstack([np.ones((1, s)), np.zeros((1, 1))])
    res = linprog(c, A_ub=a_ub, b_ub=np.zeros(len(others)), A_eq=a_eq, b_eq=[1.0],
                  bounds=[(0.0, 1.0)] * s + [(None, None)], method="highs")
    if not res.success:
        raise RuntimeError(f"pruning LP failed: {res.message}")
    return res.x[:s] if -res.fun > tol else None


def prune(alphas: np.ndarray, tags: np.ndarray, tol: float = 1e-9):
    """Lark's filter: keep the vectors that are strictly best at some belief."""
    _, first = np.unique(np.round(alphas, 12), axis=0, return_index=True)
    order = np.sort(first)
    alphas, tags = alphas[order], tags[order]
    todo = list(range(len(alphas)))
    kept = []
    while todo:
        if not kept:
            kept.append(todo.pop(0))
            continue
        b = _witness(alphas[todo[0]], alphas[kept], tol)
        if b is None:
            todo.pop(0)
            continue
        best = todo[int(np.argmax(alphas[todo] @ b))]  # the winner at the witness is undominated
        todo.remove(best)
        kept.append(best)
    kept.sort()
    return alphas[kept], tags[kept]


def exact_value_iteration(pomdp, horizon: int, max_vectors: int = 20_000) -> AlphaSet:
    """oracle.py:259-310: V_{t+1} = max_a [R(:, a) + Σ_o γ proj_{a,o}(V_t)] by cross-sums."""
    T = np.asarray(pomdp.transitions, dtype=np.float64)   # [a, s, s']
    Z = np.asarray(pomdp.observations, dtype=np.float64)  # [a, s', o]
    R = np.asarray(pomdp.rewards, dtype=np.float64)       # [s, a]
    g = float(pomdp.discount)
    S, nA, nO = T.shape[1], T.shape[0], Z.shape[2]
    alphas = np.zeros((1, S))
    tags = np.zeros(1, dtype=np.int64)
    for _ in range(horizon):
        pool, pool_tags = [], []
        for a in range(nA):
            acc = R[:, a][None, :]
            for o in range(nO):
                # proj[k](s) = γ Σ_s' T[a, s, s'] Z[a, s', o] alpha_k(s')
                proj = g * (alphas * Z[a][:, o][None, :]) @ T[a].T
                acc = (acc[:, None, :] + proj[None, :, :]).reshape(-1, S)
                if len(acc) > max_vectors:
                    raise RuntimeError("cross-sum too large for exact enumeration")
                if len(acc) > 64:
                    acc, _ = prune(acc, np.zeros(len(acc), dtype=np.int64))
            pool.append(acc)
            pool_tags.append(np.full(len(acc), a, dtype=np.int64))
        alphas, tags = prune(np.concatenate(pool), np.concatenate(pool_tags))
    return AlphaSet(alphas, tags)


# ------------------------------------------------------------------ exact Bayes filter (SPEC #5)


def exact_bayes_filter(pomdp, belief, action: int, observation: int) -> np.ndarray:
    """oracle.py:313-323."""
    b = np.asarray(belief, dtype=np.float64)
    pred = np.asarray(pomdp.transitions, dtype=np.float64)[action].T @ b
    post = np.asarray(pomdp.observations, dtype=np.float64)[action][:, observation] * pred
    z = post.sum()
    if z <= 0.0:
        raise ValueError(f"observation {observation} is impossible after action {action}")
    return post / z
