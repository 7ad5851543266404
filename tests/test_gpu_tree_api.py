"""The reference's tree / backup utility surface on the device:
match_or_append_pairs, BeliefTree.append_actions / append_beliefs / nodes_at_depth /
serialize / deserialize, aggregate_leaves, action_q_values -- against the reference's golden
vectors and the oracle restatement, on identical inputs."""

import numpy as np
import pytest

import oracle
import paper_2510_27191_b200 as vp
from golden_cases import load

pytestmark = pytest.mark.gpu


def test_match_or_append_pairs_equals_reference_golden():
    g = load("formulas")
    rows, n_new = vp.match_or_append_pairs(g["moa_existing"], g["moa_query"])
    np.testing.assert_array_equal(rows, g["moa_rows"])
    assert n_new == int(g["moa_new"][0])
    rows, n_new = vp.match_or_append_pairs(np.zeros((0, 2), dtype=np.int64), [[5, 1], [2, 2], [5, 1], [0, 9]])
    np.testing.assert_array_equal(rows, [0, 1, 0, 2])
    assert n_new == 3
    with pytest.raises(ValueError):
        vp.match_or_append_pairs([[0, 0]], [[-1, 0]])


def _grow_both(A, steps, seed):
    """The same random append sequence on the oracle tree and the device tree."""
    ot = oracle.ColumnarTree(A)
    dt = vp.DeviceTree(A, precision="fp64", cap_beliefs=16, cap_actions=16)
    g = np.random.default_rng(seed)
    for _ in range(steps):
        nb = ot.n_beliefs
        k = int(g.integers(1, 300))
        b = g.integers(0, nb, size=k)
        a = g.integers(0, A, size=k)
        r = g.integers(-5, 6, size=k).astype(np.float64)
        xo = ot.append_actions(b, a, r)
        xd = dt.append_actions(b, a, r)
        np.testing.assert_array_equal(xd, xo)
        o = g.integers(0, 4, size=k)
        co = ot.append_beliefs(xo, o)
        cd = dt.append_beliefs(xd, o)
        np.testing.assert_array_equal(cd, co)
    return ot, dt


@pytest.mark.parametrize("seed", [0, 1])
def test_appends_equal_oracle_tables(seed):
    ot, dt = _grow_both(A=7, steps=6, seed=seed)
    want, got = ot.tables(), dt.tables()
    for k in ("parent_action", "parent_obs", "depth", "action_parent_belief", "action_id", "action_visits"):
        np.testing.assert_array_equal(got[k], want[k], err_msg=k)
    np.testing.assert_array_equal(got["action_reward_sum"], want["action_reward_sum"])  # integer rewards: exact
    np.testing.assert_array_equal(got["prefs"], want["prefs"])
    dt.validate()
    for k in ("parent_action", "depth", "prefs", "action_id", "action_visits"):  # column properties
        np.testing.assert_array_equal(getattr(dt, k), getattr(ot, k), err_msg=k)
    for d in (1, 2, 3):
        for x, y in zip(dt.nodes_at_depth(d), ot.nodes_at_depth(d)):
            np.testing.assert_array_equal(x, y)
    with pytest.raises(ValueError):
        dt.nodes_at_depth(0)
    with pytest.raises(ValueError):
        dt.append_actions([0, 1], [0], [0.0, 0.0])
    with pytest.raises(ValueError):
        dt.append_beliefs([dt.n_actions], [0])


def test_serialize_deserialize_round_trip():
    model = oracle.MarsModel(4, 3, layout_seed=0)
    belief = oracle.ParticleBelief.from_model(model, 500, oracle.RowRng.from_seed(0).derive(3))
    out = vp.plan(belief, model, oracle.SolverConfig(n_parallel=256, iterations=5), oracle.RowRng.from_seed(0),
                  precision="fp64", keep_tree=True)
    text = out.tree.serialize()
    back = vp.DeviceTree.deserialize(text, precision="fp64")
    assert back.serialize() == text
    back.validate()
    # the rebuilt hash indexes resolve the existing edges to their ids and append past them
    t = back.tables()
    np.testing.assert_array_equal(back.append_actions(t["action_parent_belief"][:50], t["action_id"][:50],
                                                      np.zeros(50)), np.arange(50))
    assert back.append_beliefs([0], [7]) == [t["depth"].shape[0]]


def test_aggregate_leaves_and_q_values_equal_oracle():
    ot, dt = _grow_both(A=5, steps=4, seed=3)

    class Leaves:
        pass

    g = np.random.default_rng(9)
    deep = np.flatnonzero(ot.depth == ot.depth.max())
    leaves = Leaves()
    leaves.leaf_belief_indices = g.choice(deep, size=2000)
    leaves.heuristic_values = g.normal(size=2000)
    lo, ld = oracle.aggregate_leaves(leaves), vp.aggregate_leaves(leaves)
    np.testing.assert_array_equal(ld.belief_indices, lo.belief_indices)
    np.testing.assert_array_equal(ld.visit_weights, lo.visit_weights)
    np.testing.assert_allclose(ld.values, lo.values, rtol=1e-13, atol=1e-15)
    acts = np.unique(ot.parent_action[lo.belief_indices])
    qo = oracle.action_q_values(ot, acts, lo, 0.95)
    qd = vp.action_q_values(dt, acts, ld, 0.95)
    np.testing.assert_allclose(qd, qo, rtol=1e-13, atol=1e-13)
    with pytest.raises(ValueError):
        vp.action_q_values(dt, [0], ld, 0.95)  # the root's first action has no valued child here


def _dense_cdf_errors(tree, eta):
    """Max |psi_cdf - normalised cumsum(softmax(eta psi))| over every dense row of a fast-mode tree,
    with the cached LSE of the row's belief (what the next pass's draws read)."""
    import torch

    nb = tree.extent()[0]
    rec = tree.b_rec[:nb]
    dense = torch.nonzero(rec[:, 0] != 0).squeeze(1)
    rows = rec[dense, 1].to(torch.int64)
    A = tree.action_count
    psi = tree.psi[rows, :A].double()
    lse = tree.b_lse[dense]
    p = torch.exp(eta * (psi - lse[:, None]))
    want = torch.cumsum(p, dim=1) / p.sum(dim=1, keepdim=True)
    got = tree.psi_cdf[rows, :A].double()
    return len(rows), float((got - want).abs().max()) if len(rows) else 0.0


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_dense_rows_cdf_rows_are_current(precision):
    """After a fast-mode plan every dense PSI row's CDF row (rebuilt by the CDF kernel after each
    backup that changed the row) is the softmax CDF of the row under its cached LSE; after
    deserialize / append_actions (host-level edits) vp_tree_build_cdfs makes them so."""
    model = vp.MarsModel(7, 8, layout_seed=1)
    belief = vp.ParticleBelief.from_model(model, 500, vp.RowRng.from_seed(1).derive(3))
    out = vp.plan(belief, model, vp.SolverConfig(n_parallel=2048, iterations=6), vp.RowRng.from_seed(1),
                  precision=precision, keep_tree=True)
    n, err = _dense_cdf_errors(out.tree, 2.0)
    assert n > 10
    assert err < (1e-5 if precision == "fp32" else 1e-12), err
    back = vp.DeviceTree.deserialize(out.tree.serialize(), precision=precision)
    n2, err2 = _dense_cdf_errors(back, back.eta)
    assert n2 == len(back.tables()["depth"]) and err2 < (1e-5 if precision == "fp32" else 1e-12), err2
