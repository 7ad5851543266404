"""User ProblemModels as device plug-ins (plugin.py; the reference plans any ProblemModel,
core.py:84-142).  The tabular plug-in restates the reference's TabularModel in a user's
CUDA source; compiled into a plug-in build it must plan Tiger exactly like the built-in
model and the reference:

* step / observation likelihood: bit-exact against the oracle's Tiger;
* fp64 parity-mode plans equal the REFERENCE's golden Tiger trees in every integer column
  (and, on Philox streams, the oracle's trees);
* the device SIR through the plug-in equals the oracle SIR;
* a plug-in-only model (corridor: continuous state, normal draws) plans and runs episodes.
"""

import numpy as np
import pytest

import oracle
import paper_2510_27191_b200 as vp
from paper_2510_27191_b200.envs.plugin_examples import corridor_cuda_model, tabular_cuda_model
from golden_cases import INT_COLUMNS, load, manifest, plan_inputs
from oracle.rng import PhiloxRowRng

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tiger():
    return tabular_cuda_model(oracle.tiger_model().pomdp)


def test_plugin_step_and_likelihood_equal_oracle(tiger):
    om = oracle.tiger_model()
    g = np.random.default_rng(3)
    n = 4096
    idx = g.integers(0, 3, n)
    states = om.states_from_indices(idx)
    acts = g.integers(0, 3, n)
    rng = oracle.RowRng.from_seed(8).derive(2).bind(np.arange(n) * 7 + 1)
    want = om.step_batch(states, acts, rng)
    got = tiger.step_batch(states, acts, rng)
    np.testing.assert_array_equal(got.next_states.idx, want.next_states.idx)
    np.testing.assert_array_equal(got.next_states.terminal, want.next_states.terminal)
    np.testing.assert_array_equal(got.observations, want.observations)
    np.testing.assert_array_equal(got.rewards, want.rewards)
    for a in range(3):
        for o in range(3):
            np.testing.assert_array_equal(tiger.observation_log_likelihood(want.next_states, a, o),
                                          om.observation_log_likelihood(want.next_states, a, o))
    np.testing.assert_array_equal(tiger.value_heuristic(states), np.zeros(n))


@pytest.mark.parametrize("rng_kind", ["splitmix64", "philox"])
def test_plugin_fp64_exact_plan_equals_reference(tiger, rng_kind):
    case = manifest()["plans"]["plan_tiger"]
    g = load("plan_tiger")
    for run in case["runs"]:
        s = run["seed"]
        om, belief, cfg, rng = plan_inputs(case, s)
        if rng_kind == "philox":
            rng = PhiloxRowRng(rng.key)
            want = oracle.plan(belief, om, cfg, rng)
            stats, cols, chosen = want.tree_stats, want.tree.tables(), want.chosen_action
        else:  # the reference's own golden tree
            stats, chosen = run["tree_stats"], run["chosen_action"]
            cols = {k: g[f"s{s}_{k}"] for k in INT_COLUMNS}
        out = vp.plan(belief, tiger, cfg, rng, precision="fp64", exact=True, keep_tree=True)
        assert out.tree_stats == stats
        t = out.tree.tables()
        for k in INT_COLUMNS:
            np.testing.assert_array_equal(t[k], np.asarray(cols[k]).astype(np.int64), err_msg=f"s{s} {k}")
        assert out.chosen_action == chosen
        if rng_kind == "splitmix64":
            np.testing.assert_allclose(t["prefs"][0], g[f"s{s}_prefs_root"], rtol=1e-9, atol=1e-9)


def test_plugin_fp32_plan_equals_builtin(tiger):
    om = oracle.tiger_model()
    belief = oracle.ParticleBelief.from_model(om, 2000, oracle.RowRng.from_seed(4).derive(3))
    cfg = oracle.SolverConfig(n_parallel=4096, iterations=8)
    rng = oracle.RowRng.from_seed(4).derive(1, 0)
    a = vp.plan(belief, tiger, cfg, rng, keep_tree=True)
    b = vp.plan(belief, vp.tiger_model(), cfg, rng, keep_tree=True)
    assert a.tree_stats == b.tree_stats and a.chosen_action == b.chosen_action
    ta, tb = a.tree.tables(), b.tree.tables()
    for k in INT_COLUMNS:
        np.testing.assert_array_equal(ta[k], tb[k])
    np.testing.assert_array_equal(ta["prefs"], tb["prefs"])


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_plugin_device_sir_equals_oracle(tiger, seed):
    om = oracle.tiger_model()
    belief = oracle.ParticleBelief.from_model(om, 3000, oracle.RowRng.from_seed(seed).derive(3))
    rng = oracle.RowRng.from_seed(seed).derive(2, 1)
    want = oracle.sir_update(belief, om, 0, 1, rng, max_retries=3)
    got = vp.sir_update(vp.DeviceBelief.from_host(belief, tiger), tiger, 0, 1, rng, max_retries=3)
    assert (got.retries, got.degenerate) == (want.retries, want.degenerate)
    np.testing.assert_array_equal(got.belief.states.idx, want.belief.states.idx)


def test_plugin_episodes_match_builtin(tiger):
    cfg = vp.SolverConfig(n_parallel=1024, iterations=6, particles=1000)
    for seed in range(3):
        a = vp.run_episode(tiger, cfg, seed=seed, precision="fp64")
        b = vp.run_episode(vp.tiger_model(), cfg, seed=seed, precision="fp64")
        assert (a.steps, a.terminal_reason) == (b.steps, b.terminal_reason)
        assert a.discounted_return == pytest.approx(b.discounted_return, abs=1e-12)


def test_plugin_only_model_plans_and_runs():
    m = corridor_cuda_model()
    belief = vp.ParticleBelief.from_model(m, 2000, vp.RowRng.from_seed(1).derive(3))
    cfg = vp.SolverConfig(n_parallel=8192, iterations=10)
    out = vp.plan(belief, m, cfg, vp.RowRng.from_seed(1).derive(1, 0), keep_tree=True)
    out.tree.validate()
    assert out.tree.tables()["action_visits"].sum() == cfg.n_parallel * sum(range(1, 11))
    assert 0 <= out.chosen_action < 3
    rec = vp.run_episode(m, vp.SolverConfig(n_parallel=4096, iterations=8, particles=2000), seed=3)
    assert np.isfinite(rec.discounted_return) and rec.steps >= 1
    p = vp.run_episode(m, vp.SolverConfig(n_parallel=4096, iterations=8, particles=2000), seed=3, rng_kind="philox")
    assert np.isfinite(p.discounted_return)


@pytest.mark.parametrize("world", [2, 4])
def test_plugin_sharded_plan_equals_reference(tiger, world):
    """The sharded planner routes the plug-in's trajectory / insert passes to its library too."""
    case = manifest()["plans"]["plan_tiger"]
    g = load("plan_tiger")
    run = case["runs"][0]
    s = run["seed"]
    om, belief, cfg, rng = plan_inputs(case, s)
    out = vp.ShardedPlanner(world=world, precision="fp64", exact=True).plan(belief, tiger, cfg, rng, keep_tree=True)
    assert out.tree_stats == run["tree_stats"]
    t = out.tree.tables()
    for k in INT_COLUMNS:
        np.testing.assert_array_equal(t[k], g[f"s{s}_{k}"].astype(np.int64), err_msg=k)
    assert out.chosen_action == run["chosen_action"]


def test_plugin_with_reference_policy(tiger):
    """reference_log_probs (core.py:109-112) of a plug-in shape the initial PSI rows like a built-in's."""
    om = oracle.tiger_model()
    logp = np.log(np.array([0.6, 0.2, 0.2]))
    from paper_2510_27191_b200.envs.plugin_examples import TAB_PARAMS

    biased = vp.CudaModel(tiger.spec, tiger.state_dtype, tiger.source, tiger.params.view(TAB_PARAMS),
                          reference_log_probs=logp, tables=tiger.tables)

    class BiasedTiger(oracle.TabularModel):
        def reference_log_probs(self):
            return logp.copy()

    ob = BiasedTiger(om.pomdp)
    belief = oracle.ParticleBelief.from_model(om, 1000, oracle.RowRng.from_seed(6).derive(3))
    cfg = oracle.SolverConfig(n_parallel=512, iterations=6)
    rng = oracle.RowRng.from_seed(6).derive(1, 0)
    want = oracle.plan(belief, ob, cfg, rng)
    out = vp.plan(belief, biased, cfg, rng, precision="fp64", exact=True, keep_tree=True)
    assert out.tree_stats == want.tree_stats and out.chosen_action == want.chosen_action
    t, w = out.tree.tables(), want.tree.tables()
    for k in INT_COLUMNS:
        np.testing.assert_array_equal(t[k], np.asarray(w[k]).astype(np.int64), err_msg=k)


def _random_pomdp(S, A, O, seed):
    g = np.random.default_rng(seed)
    t = g.dirichlet(np.ones(S) * 0.3, size=(A, S))
    z = g.dirichlet(np.ones(O) * 0.5, size=(A, S))
    term = np.zeros(S, dtype=bool)
    term[-1] = True
    t[:, -1, :] = 0.0
    t[:, -1, -1] = 1.0
    b0 = np.ones(S) / (S - 1)
    b0[-1] = 0.0
    return oracle.TabularPOMDP(t, z, g.normal(size=(S, A)), b0, 0.95, term, "random", 60)


def test_large_tabular_plugin_with_hbm_tables_equals_oracle():
    """Tables of any size travel as HBM arrays behind Params pointers (CudaModel tables=)."""
    pomdp = _random_pomdp(40, 6, 7, 3)
    om = oracle.TabularModel(pomdp)
    pm = tabular_cuda_model(pomdp)
    g = np.random.default_rng(4)
    n = 8192
    states = om.states_from_indices(g.integers(0, 40, n))
    acts = g.integers(0, 6, n)
    rng = oracle.RowRng.from_seed(2).derive(5).bind(np.arange(n))
    want, got = om.step_batch(states, acts, rng), pm.step_batch(states, acts, rng)
    np.testing.assert_array_equal(got.next_states.idx, want.next_states.idx)
    np.testing.assert_array_equal(got.observations, want.observations)
    np.testing.assert_array_equal(got.rewards, want.rewards)
    belief = oracle.ParticleBelief.from_model(om, 2000, oracle.RowRng.from_seed(9).derive(3))
    cfg = oracle.SolverConfig(n_parallel=1024, iterations=6)
    rng = oracle.RowRng.from_seed(9).derive(1, 0)
    ref = oracle.plan(belief, om, cfg, rng)
    out = vp.plan(belief, pm, cfg, rng, precision="fp64", exact=True, keep_tree=True)
    assert out.tree_stats == ref.tree_stats and out.chosen_action == ref.chosen_action
    t, w = out.tree.tables(), ref.tree.tables()
    for k in INT_COLUMNS:
        np.testing.assert_array_equal(t[k], np.asarray(w[k]).astype(np.int64), err_msg=k)


@pytest.mark.parametrize("precision,exact", [("fp64", True), ("fp32", False)])
def test_cooperative_plugin_equals_single_lane_form(precision, exact):
    """A large-record plug-in (520 B) built warp-cooperative (VP_USER_COOP: one row per warp, the
    lanes splitting the record) plans exactly like its one-row-per-lane build."""
    from paper_2510_27191_b200.envs.plugin_examples import levels_cuda_model

    coop, lane = levels_cuda_model(coop=True), levels_cuda_model(coop=False)
    belief = vp.ParticleBelief.from_model(lane, 500, vp.RowRng.from_seed(2).derive(3))
    cfg = vp.SolverConfig(n_parallel=1024, iterations=6)
    rng = vp.RowRng.from_seed(2).derive(1, 0)
    a = vp.plan(belief, coop, cfg, rng, precision=precision, exact=exact, keep_tree=True)
    b = vp.plan(belief, lane, cfg, rng, precision=precision, exact=exact, keep_tree=True)
    assert a.tree_stats == b.tree_stats and a.chosen_action == b.chosen_action
    ta, tb = a.tree.tables(), b.tree.tables()
    for k in INT_COLUMNS:
        np.testing.assert_array_equal(ta[k], tb[k], err_msg=k)
    # values: the backup's L2 reductions sum in arrival order (1 ulp apart between runs)
    tol = 1e-12 if precision == "fp64" else 1e-5
    np.testing.assert_allclose(ta["prefs"], tb["prefs"], rtol=tol, atol=tol * np.abs(tb["prefs"]).max())
    assert a.tree_stats["belief_rows"] > 100


def test_cooperative_plugin_sir_and_episode():
    from paper_2510_27191_b200.envs.plugin_examples import levels_cuda_model

    coop, lane = levels_cuda_model(coop=True), levels_cuda_model(coop=False)
    belief = vp.ParticleBelief.from_model(lane, 2000, vp.RowRng.from_seed(4).derive(3))
    env = lane.sample_initial_states(1, vp.RowRng.from_seed(4).derive(0, 0))
    res = lane.step_batch(env, np.array([2]), vp.RowRng.from_seed(4).derive(0, 1).bind([0]))
    o = int(res.observations[0])
    rng = vp.RowRng.from_seed(4).derive(2, 1)
    x = vp.sir_update(vp.DeviceBelief.from_host(belief, coop), coop, 2, o, rng, max_retries=3)
    y = vp.sir_update(vp.DeviceBelief.from_host(belief, lane), lane, 2, o, rng, max_retries=3)
    assert (x.retries, x.degenerate) == (y.retries, y.degenerate)
    np.testing.assert_array_equal(x.belief.records.cpu().numpy(), y.belief.records.cpu().numpy())
    cfg = vp.SolverConfig(n_parallel=512, iterations=4, particles=500)
    ea = vp.run_episode(coop, cfg, seed=1, precision="fp64")
    eb = vp.run_episode(lane, cfg, seed=1, precision="fp64")
    assert (ea.steps, ea.terminal_reason) == (eb.steps, eb.terminal_reason)
    assert ea.discounted_return == pytest.approx(eb.discounted_return, abs=1e-12)
