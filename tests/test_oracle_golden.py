"""Pin the CPU oracle against golden vectors produced by the real reference.

CPU-only.  If any of these fail the oracle is not trustworthy and every GPU
parity claim built on it is void.
"""

import numpy as np
import pytest

import oracle
from golden_cases import CROWD_CASES, CROWD_FIELDS, INT_COLUMNS, load, manifest, plan_inputs, tree_columns


def test_rng_streams_match_reference():
    g = load("rng")
    rows = g["rows"]
    i = 0
    for s in [0, 1, 42, 2**63 + 5, 123456789]:
        r = oracle.RowRng.from_seed(s)
        for path in [(), (0,), (1, 0), (3, 5, 7), (2, 11)]:
            d = r.derive(*path)
            assert int(d.key) == int(g["keys"][i])
            np.testing.assert_array_equal(d.uniform(rows), g["uniform"][i])
            np.testing.assert_array_equal(d.uniform(rows, 3), g["uniform_k3"][i])
            np.testing.assert_array_equal(d.normal(rows, 2), g["normal_k2"][i])
            i += 1
    assert oracle.RowRng.from_seed(12).derive(4).uniform1() == g["uniform1"][0]


def test_rng_contract_examples():
    # pkg/tests/test_rng.py:6-61 restated against the oracle
    with pytest.raises(ValueError):
        oracle.RowRng.from_seed(1).derive(-1)
    rng = oracle.RowRng.from_seed(9).derive(1)
    np.testing.assert_array_equal(rng.uniform(np.arange(4)), rng.uniform(np.arange(4096))[:4])
    b = oracle.RowRng.from_seed(3).derive(7).bind([5, 6])
    np.testing.assert_array_equal(b.uniform(), oracle.RowRng.from_seed(3).derive(7).uniform(np.array([5, 6])))


def test_formula_vectors():
    g = load("formulas")
    np.testing.assert_array_equal(oracle.log_sum_exp_rows(g["lse_in"], 2.0), g["lse_eta2"])
    np.testing.assert_array_equal(oracle.softmax_rows(g["lse_in"], 2.0), g["softmax_eta2"])
    rng = oracle.RowRng.from_seed(3).derive(9)
    got = oracle.sample_actions(g["sa_pol"], rng.bind(np.arange(300)), groups=g["sa_groups"])
    np.testing.assert_array_equal(got, g["sa_multi"])
    got1 = oracle.sample_actions(g["sa_pol"][:1], rng.bind(np.arange(300)), groups=np.zeros(300, dtype=np.int64))
    np.testing.assert_array_equal(got1, g["sa_single"])
    rows, n_new = oracle.match_or_append_pairs(g["moa_existing"], g["moa_query"])
    np.testing.assert_array_equal(rows, g["moa_rows"])
    assert n_new == int(g["moa_new"][0])


def test_spec_appendix_c_examples():
    # SPEC.md:154-157, 163-166, 227-230, 285-288, 294-297, 303-306
    rows, n_new = oracle.match_or_append_pairs(np.zeros((0, 2)), [(0, 3), (0, 3), (0, 5)])
    assert list(rows) == [0, 0, 1] and n_new == 2
    rows, n_new = oracle.match_or_append_pairs([(0, 3)], [(0, 3)])
    assert list(rows) == [0] and n_new == 0
    t = oracle.ColumnarTree(4)
    t.append_actions([0, 0, 0], [2, 2, 2], [1.0, 1.0, 4.0])
    assert t.action_visits[0] == 3 and t.action_reward_sum[0] == 6.0
    np.testing.assert_allclose(oracle.softmax_rows([[0.0, np.log(2.0)]], 1.0), [[1 / 3, 2 / 3]])
    np.testing.assert_allclose(oracle.softmax_rows([[1.0] * 4], 2.0), [[0.25] * 4])
    assert abs(oracle.log_sum_exp_rows([[3.0] * 4], 2.0)[0] - (3.0 + np.log(4) / 2)) < 1e-12
    assert abs(oracle.log_sum_exp_rows([[1.0, 2.0]], 1.0)[0] - 2.31326) < 1e-5
    lv = oracle.aggregate_leaves(oracle.LeafResult(np.array([7, 7]), np.array([4.0, 6.0])))
    assert lv.values[0] == 5.0 and lv.visit_weights[0] == 2.0


@pytest.mark.parametrize("name", sorted(manifest()["plans"]))
def test_oracle_plan_matches_reference(name):
    case = manifest()["plans"][name]
    g = load(name)
    for run in case["runs"]:
        s = run["seed"]
        model, belief, cfg, rng = plan_inputs(case, s)
        out = oracle.plan(belief, model, cfg, rng)
        assert out.chosen_action == run["chosen_action"]
        assert out.tree_stats == run["tree_stats"]
        assert out.final_d_max == run["final_d_max"]
        cols = tree_columns(out.tree.tables())
        for k in INT_COLUMNS:
            np.testing.assert_array_equal(cols[k], g[f"s{s}_{k}"].astype(cols[k].dtype), err_msg=k)
        np.testing.assert_array_equal(cols["action_reward_sum"], g[f"s{s}_action_reward_sum"])
        np.testing.assert_array_equal(cols["prefs_root"], g[f"s{s}_prefs_root"])
        np.testing.assert_allclose(cols["prefs_row_sum"], g[f"s{s}_prefs_row_sum"], rtol=0, atol=1e-12)
        if f"s{s}_prefs" in g:
            np.testing.assert_array_equal(cols["prefs"], g[f"s{s}_prefs"])
        out.tree.validate()


def test_oracle_episode_matches_reference():
    recs = manifest()["episodes"]["episode_mars4_3"]
    cfg = oracle.SolverConfig(n_parallel=64, iterations=4, particles=500)
    for r in recs:
        got = oracle.run_episode(oracle.MarsModel(n=4, m=3, layout_seed=r["seed"]), cfg, seed=r["seed"])
        assert got.steps == r["steps"] and got.terminal_reason == r["reason"]
        assert got.discounted_return == r["return"]


def test_oracle_crowdnav_episodes_match_reference():
    """Closed loop with CrowdNav's refresh / reconcile hooks (crowdnav.py:199-224)."""
    cfg = oracle.SolverConfig(n_parallel=128, iterations=4, particles=300)
    for r in manifest()["episodes"]["episode_crowdnav40"]:
        got = oracle.run_episode(oracle.CrowdNavModel(n_people=40, hall_depth=8.0, max_steps=15), cfg, seed=r["seed"])
        assert (got.steps, got.terminal_reason, got.degenerate_updates) == (r["steps"], r["reason"], r["degenerate"])
        assert got.discounted_return == r["return"]


def test_navigation_model_vectors():
    """oracle.NavigationModel vs the reference's navigation.py (steps, likelihoods, heuristic)."""
    g = load("nav_steps")
    m = oracle.NavigationModel()
    st = m.sample_initial_states(400, oracle.RowRng.from_seed(21))
    np.testing.assert_array_equal(st.pos, g["pos0"])
    np.testing.assert_array_equal(st.occ, g["occ0"])
    np.testing.assert_array_equal(st.open_gate, g["gate0"])
    for t in range(8):
        res = m.step_batch(st, g[f"a{t}"], oracle.RowRng.from_seed(40 + t).bind(np.arange(400)))
        np.testing.assert_array_equal(res.next_states.pos, g[f"pos{t + 1}"])
        np.testing.assert_array_equal(res.next_states.terminal, g[f"term{t + 1}"])
        np.testing.assert_array_equal(res.observations, g[f"obs{t + 1}"])
        np.testing.assert_array_equal(res.rewards, g[f"rew{t + 1}"])
        a, o = (int(v) for v in g[f"llobs{t + 1}"])
        np.testing.assert_array_equal(m.observation_log_likelihood(res.next_states, a, o), g[f"ll{t + 1}"])
        np.testing.assert_array_equal(m.value_heuristic(res.next_states), g[f"h{t + 1}"])
        st = res.next_states


@pytest.mark.parametrize("tag,people,n,steps", CROWD_CASES)
def test_crowdnav_model_vectors(tag, people, n, steps):
    """oracle.CrowdNavModel vs the reference's crowdnav.py (sampler, steps, likelihoods,
    heuristic, tracking refresh)."""
    g = load("crowd_steps")
    m = oracle.CrowdNavModel(n_people=people)
    st = m.sample_initial_states(n, oracle.RowRng.from_seed(31))
    for f in CROWD_FIELDS:
        np.testing.assert_array_equal(getattr(st, f), g[f"{tag}_{f}0"], err_msg=f)
    for t in range(steps):
        res = m.step_batch(st, g[f"{tag}_a{t}"], oracle.RowRng.from_seed(50 + t).bind(np.arange(n)))
        for f in ("robot", "prev_dist", "last_code", "terminal"):
            np.testing.assert_array_equal(getattr(res.next_states, f), g[f"{tag}_{f}{t + 1}"], err_msg=f)
        np.testing.assert_array_equal(res.observations, g[f"{tag}_obs{t + 1}"])
        np.testing.assert_array_equal(res.rewards, g[f"{tag}_rew{t + 1}"])
        a, o = (int(v) for v in g[f"{tag}_llobs{t + 1}"])
        np.testing.assert_array_equal(m.observation_log_likelihood(res.next_states, a, o), g[f"{tag}_ll{t + 1}"])
        np.testing.assert_array_equal(m.value_heuristic(res.next_states), g[f"{tag}_h{t + 1}"])
        st = res.next_states
    np.testing.assert_array_equal(st.persons, g[f"{tag}_persons_end"])
    r = m.refresh_executed(st.take([2]))
    np.testing.assert_array_equal(r.tracked, g[f"{tag}_refresh_tracked"])
    np.testing.assert_array_equal(r.prev_dist, g[f"{tag}_refresh_prev"])
