"""The acceptance oracles' restatement (oracle/acceptance.py) against the REAL
reference's outputs (tests/golden/acceptance.npz, written by make_golden.py from
/root/reference/pkg/src/vecpomdp/oracle.py) -- CPU.

* serial_backup (oracle.py:124-173) on 24 random trees of the SPEC #1 family;
* exact_value_iteration (oracle.py:259-310) on Tiger, horizons 1-8;
* exact_bayes_filter (oracle.py:313-323) on 10 random 2-state chains x 10 steps.

Also: the level-synchronous oracle backup (oracle/backup.py, the reference's
vectorised Alg. 3) equals the serial backup on the SPEC #1 cases -- SPEC
ACCEPTANCE 1 for the oracle itself.
"""

import numpy as np
import pytest

import oracle
from oracle import acceptance as acc
from golden_cases import load

G = load("acceptance")


def test_serial_backup_equals_reference():
    for k in range(24):
        A, passes = acc.random_tree_case(np.random.default_rng(1000 + k))
        tree = acc.serial_run(A, passes, eta=2.0, gamma=0.9)
        paths = sorted(tree.prefs)
        want_paths = [tuple(int(v) for v in row if v >= 0) for row in G[f"tree{k}_paths"]]
        assert paths == want_paths
        got = np.array([tree.prefs[p] for p in paths])
        np.testing.assert_allclose(got, G[f"tree{k}_prefs"], rtol=0, atol=1e-12)


def columnar_run(A, passes, eta, gamma):
    """The case through the oracle's columnar tree + vectorised backup (tree.py, backup.py)."""
    t = oracle.ColumnarTree(A)
    for p in passes:
        d, n = p["actions"].shape
        b = np.zeros(n, dtype=np.int64)
        for lvl in range(d):
            x = t.append_actions(b, p["actions"][lvl].astype(np.int64), p["rewards"][lvl])
            b = t.append_beliefs(x, p["observations"][lvl].astype(np.int64))
        leaves = oracle.LeafResult(b, p["leaf"].astype(np.float64))
        oracle.backup(t, leaves, d, eta, gamma)
    return t


def test_vectorised_oracle_backup_matches_serial_on_200_random_trees():
    """SPEC ACCEPTANCE 1 for the oracle restatement: every PSI entry within 1e-6."""
    worst = 0.0
    for k in range(200):
        A, passes = acc.random_tree_case(np.random.default_rng(k))
        serial = acc.serial_run(A, passes, 2.0, 0.9)
        col = columnar_run(A, passes, 2.0, 0.9)
        paths = acc.belief_paths(col.parent_action, col.parent_obs, col.action_parent_belief, col.action_id)
        assert sorted(paths) == sorted(serial.prefs)
        for i, p in enumerate(paths):
            worst = max(worst, float(np.max(np.abs(col.prefs[i] - np.array(serial.prefs[p])))))
    assert worst <= 1e-6, worst


@pytest.mark.parametrize("h", [1, 2, 3, 5, 8])
def test_exact_value_iteration_equals_reference(h):
    tiger = oracle.tiger_model()
    v = acc.exact_value_iteration(tiger.pomdp, h)
    beliefs = G["vi_beliefs"]
    vals = np.array([v.value(b) for b in beliefs])
    np.testing.assert_allclose(vals, G[f"vi_h{h}_values"], rtol=1e-9, atol=1e-9)
    acts = np.array([v.action(b) for b in beliefs])
    # ties between actions (equal values at a boundary belief) may pick either vector
    q = np.array([v.q_values(b) for b in beliefs])
    for i, (a, want) in enumerate(zip(acts, G[f"vi_h{h}_actions"])):
        assert a == want or abs(q[i, a] - q[i, want]) < 1e-9


def test_exact_bayes_filter_equals_reference():
    for k in range(10):
        pomdp = oracle.TabularPOMDP(G[f"chain{k}_T"], G[f"chain{k}_Z"], G[f"chain{k}_R"], np.array([0.5, 0.5]),
                                    0.95, np.array([False, False]), "chain", 50)
        b = np.array([0.5, 0.5])
        for (a, o), want in zip(G[f"chain{k}_seq"], G[f"chain{k}_post"]):
            b = acc.exact_bayes_filter(pomdp, b, int(a), int(o))
            np.testing.assert_allclose(b, want, rtol=0, atol=1e-15)
    with pytest.raises(ValueError):
        z = np.zeros((1, 2, 2))
        z[..., 0] = 1.0
        p = oracle.TabularPOMDP(np.ones((1, 2, 2)) / 2, z, np.zeros((2, 1)), np.array([0.5, 0.5]), 0.9,
                                np.array([False, False]))
        acc.exact_bayes_filter(p, [0.5, 0.5], 0, 1)


@pytest.mark.parametrize("case", __import__("golden_cases").SERIAL_CASES)
def test_oracle_width1_search_equals_reference_serial_search(case):
    """SPEC ACCEPTANCE 2 for the oracle: its vectorized search + backup at n_p = 1 rebuild the
    reference's serial_search_backup tree (integer fields exact, floats within 1e-9)."""
    from golden_cases import parse_tree_text, serial_search_build

    n, m, seed = case[:3]
    want_i, want_f = parse_tree_text(str(load("serial_search")[f"mars{n}_{m}_s{seed}"]))
    tree = serial_search_build(oracle, case, lambda model: oracle.tree.init_tree(model.spec))
    got_i, got_f = parse_tree_text(tree.serialize())
    assert got_i == want_i
    np.testing.assert_allclose(got_f, want_f, rtol=0, atol=1e-9)
