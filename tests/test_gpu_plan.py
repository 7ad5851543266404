"""Whole-planning-step parity of the device path (L1-L3 of SURVEY.md section 4).

* fp64 parity mode (numpy operation order): full ``plan()`` trees equal the
  REFERENCE's golden trees in every integer column; floats within 1e-9.
* fp32 fast mode with the oracle's sampled actions injected ("identical
  injected sample streams"): tree structure bit-exact, PSI / values within
  1e-5 relative (scale-aware).
* structural invariants and visit conservation at the C1 configuration.
"""

import numpy as np
import pytest
import torch

import oracle
import paper_2510_27191_b200 as vp
from golden_cases import INT_COLUMNS, load, manifest, plan_inputs

pytestmark = pytest.mark.gpu


def product_model(kind, seed):
    if kind.startswith("mars"):
        n, m = map(int, kind[4:].split("_"))
        return vp.MarsModel(n, m, layout_seed=seed)
    return {"tiger": vp.tiger_model, "synthetic": lambda: vp.SyntheticModel(seed=seed),
            "lightdark": vp.LightDarkModel}[kind]()


def scale_close(got, want, rel):
    """|x - y| <= rel * max(|y|, max |row|) (hard part 2)."""
    got, want = np.asarray(got), np.asarray(want)
    if want.ndim == 2:
        scale = np.maximum(np.abs(want), np.abs(want).max(axis=1, keepdims=True))
    else:
        scale = np.abs(want)
    return np.all(np.abs(got - want) <= rel * np.maximum(scale, 1.0))


@pytest.mark.parametrize("name", sorted(manifest()["plans"]))
def test_fp64_exact_plan_equals_reference_tree(name):
    case = manifest()["plans"][name]
    g = load(name)
    for run in case["runs"]:
        s = run["seed"]
        om, belief, cfg, rng = plan_inputs(case, s)
        out = vp.plan(belief, om, cfg, rng, precision="fp64", exact=True, keep_tree=True)
        assert out.tree_stats == run["tree_stats"], (name, s)
        t = out.tree.tables()
        for k in INT_COLUMNS:
            np.testing.assert_array_equal(t[k], g[f"s{s}_{k}"].astype(np.int64), err_msg=f"{name} s{s} {k}")
        np.testing.assert_allclose(t["action_reward_sum"], g[f"s{s}_action_reward_sum"], rtol=1e-12, atol=1e-9)
        np.testing.assert_allclose(t["prefs"][0], g[f"s{s}_prefs_root"], rtol=1e-9, atol=1e-9)
        np.testing.assert_allclose(t["prefs"].sum(axis=1), g[f"s{s}_prefs_row_sum"], rtol=1e-9, atol=1e-8)
        if f"s{s}_prefs" in g:
            assert scale_close(t["prefs"], g[f"s{s}_prefs"], 1e-9)
        assert out.chosen_action == run["chosen_action"]
        out.tree.validate()


@pytest.mark.parametrize("name", ["plan_mars7_8_small", "plan_navigation"])
def test_general_belief_key_plan_equals_reference_tree(name, monkeypatch):
    """The (action row, obs) belief key -- the fallback for |A| > 4096 or observation codes >= 2^20 --
    still reproduces the reference's trees (the planner defaults to (belief, action, obs) keys)."""
    monkeypatch.setenv("VP_BKEY_MODE", "0")
    case = manifest()["plans"][name]
    g = load(name)
    run = case["runs"][0]
    s = run["seed"]
    om, belief, cfg, rng = plan_inputs(case, s)
    planner = vp.Planner("fp64", exact=True)
    out = planner.plan(belief, om, cfg, rng, keep_tree=True)
    assert planner.tree is None or out.tree.struct.bkey_mode == 0
    t = out.tree.tables()
    for k in INT_COLUMNS:
        np.testing.assert_array_equal(t[k], g[f"s{s}_{k}"].astype(np.int64), err_msg=k)
    assert out.chosen_action == run["chosen_action"]


def _oracle_traces(case, seed):
    om, belief, cfg, rng = plan_inputs(case, seed)
    traces = []
    ref = oracle.plan(belief, om, cfg, rng, traces=traces)
    inject = [np.stack([lv["actions"] for lv in it["levels"]]) for it in traces]
    return om, belief, cfg, rng, ref, traces, inject


@pytest.mark.parametrize("name", ["plan_mars4_3", "plan_mars7_8_small", "plan_tiger", "plan_synthetic",
                                  "plan_lightdark", "plan_navigation", "plan_crowdnav40"])
@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_injected_streams_structure_exact_values_close(name, precision):
    case = manifest()["plans"][name]
    s = case["runs"][0]["seed"]
    om, belief, cfg, rng, ref, traces, inject = _oracle_traces(case, s)
    out = vp.plan(belief, om, cfg, rng, precision=precision, inject_actions=inject, keep_tree=True, trace=True)
    want = ref.tree.tables()
    got = out.tree.tables()
    for k in INT_COLUMNS:
        np.testing.assert_array_equal(got[k], want[k], err_msg=k)
    # per-level traces identical (observations / node ids)
    for it_d, it_o in zip(out.traces, traces):
        for lv_d, lv_o in zip(it_d["levels"], it_o["levels"]):
            np.testing.assert_array_equal(lv_d["observations"], lv_o["observations"])
            np.testing.assert_array_equal(lv_d["action_nodes"], lv_o["action_nodes"])
            np.testing.assert_array_equal(lv_d["next_beliefs"], lv_o["next_beliefs"])
    np.testing.assert_allclose(got["action_reward_sum"], want["action_reward_sum"], rtol=1e-12, atol=1e-9)
    rel = 1e-5 if precision == "fp32" else 1e-10
    assert scale_close(got["prefs"], want["prefs"], rel)


def test_c1_fp32_invariants_and_conservation():
    # RockSample(7,8) C1: n_parallel 1024, 8 iterations
    case = manifest()["plans"]["plan_mars7_8_c1"]
    for run in case["runs"]:
        s = run["seed"]
        om, belief, cfg, rng = plan_inputs(case, s)
        out = vp.plan(belief, om, cfg, rng, precision="fp32", keep_tree=True)
        t = out.tree
        t.validate()
        tab = t.tables()
        n = cfg.n_parallel
        assert tab["action_visits"].sum() == n * sum(range(1, cfg.iterations + 1))
        assert out.final_d_max == cfg.iterations and out.iterations_run == cfg.iterations
        # fp32 draws diverge from the fp64 reference after the first CDF-edge flip, so only
        # the scale is comparable (same-seed reference trees vary 13k-19k across plan keys)
        nb_ref = run["tree_stats"]["belief_rows"]
        assert 0.6 * nb_ref < out.tree_stats["belief_rows"] < 1.6 * nb_ref


@pytest.mark.parametrize("n_par", [30000, 40000])
def test_fp64_exact_large_batches_equal_oracle(n_par):
    """Large passes take the backup's 16- and 32-leaves-per-warp launch shapes (sized from
    the row count; small tests run 8): whole trees still equal the oracle's."""
    om = oracle.MarsModel(7, 8, layout_seed=5)
    belief = oracle.ParticleBelief.from_model(om, 2000, oracle.RowRng.from_seed(5).derive(3))
    cfg = oracle.SolverConfig(n_parallel=n_par, iterations=3, eta=2.0)
    rng = oracle.RowRng.from_seed(5).derive(1, 0)
    ref = oracle.plan(belief, om, cfg, rng)
    out = vp.plan(belief, om, cfg, rng, precision="fp64", exact=True, keep_tree=True)
    assert out.tree_stats == ref.tree_stats and out.chosen_action == ref.chosen_action
    got, want = out.tree.tables(), ref.tree.tables()
    for k in INT_COLUMNS:
        np.testing.assert_array_equal(got[k], want[k], err_msg=k)
    np.testing.assert_allclose(got["action_reward_sum"], want["action_reward_sum"], rtol=1e-12, atol=1e-9)
    assert scale_close(got["prefs"], want["prefs"], 1e-9)


@pytest.mark.parametrize("kind,n_par,iters", [("mars15_15", 65536, 10), ("synthetic", 65536, 20)])
def test_full_size_invariants(kind, n_par, iters):
    """BASELINE C3 / C5 at full size, fp32: properties that hold at any size -- every row adds
    one visit per level (visit conservation), the tree validates, PSI is finite, the
    chosen action is the root's first argmax, and depth-l beliefs never outnumber the rows."""
    om = oracle.MarsModel(15, 15, layout_seed=3) if kind.startswith("mars") else oracle.SyntheticModel(n_actions=16,
                                                                                                       n_obs=8, seed=3)
    belief = oracle.ParticleBelief.from_model(om, 10_000, oracle.RowRng.from_seed(3).derive(3))
    cfg = oracle.SolverConfig(n_parallel=n_par, iterations=iters)
    out = vp.plan(belief, om, cfg, oracle.RowRng.from_seed(3).derive(1, 0), keep_tree=True)
    t = out.tree.tables()
    assert t["action_visits"].sum() == n_par * sum(min(i + 1, cfg.d_max_cap) for i in range(iters))
    assert np.isfinite(t["prefs"]).all()
    assert out.chosen_action == int(np.argmax(t["prefs"][0]))
    depth_counts = np.bincount(t["depth"])
    assert depth_counts[0] == 1 and (depth_counts[1:] <= n_par * iters).all()
    assert out.tree_stats == {"belief_rows": len(t["depth"]), "action_rows": len(t["action_id"])}
    out.tree.validate()


def test_capacity_growth_matches_preallocated():
    case = manifest()["plans"]["plan_mars4_3"]
    s = case["runs"][0]["seed"]
    om, belief, cfg, rng = plan_inputs(case, s)
    base = vp.plan(belief, om, cfg, rng, precision="fp64", exact=True, keep_tree=True).tree.tables()
    planner = vp.Planner("fp64", exact=True)
    planner._capacity = lambda n, config, A: (64, config.iterations)  # force repeated growth + rehash
    out = planner.plan(belief, om, cfg, rng, keep_tree=True)
    got = out.tree.tables()
    for k in INT_COLUMNS:
        np.testing.assert_array_equal(got[k], base[k], err_msg=k)
    assert out.tree.cap_beliefs >= len(got["depth"])


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_fast_mode_growth_of_nodes_and_dense_pool_matches_graph_plan(precision):
    """Fast mode through the growing path (capacity forced small: node columns regrown and
    rehashed with static-id holes, the dense PSI pool grown on demand) equals the one-graph fixed
    plan of the same key: the same structure bit for bit, PSI up to the arrival order of the fp64
    L2 reductions (an ulp)."""
    case = manifest()["plans"]["plan_mars7_8_small"]
    s = case["runs"][0]["seed"]
    om, belief, cfg, rng = plan_inputs(case, s)
    base = vp.Planner(precision).plan(belief, om, cfg, rng, keep_tree=True)
    planner = vp.Planner(precision)
    planner._capacity = lambda n, config, A: (64, config.iterations)
    orig = vp.DeviceTree.dense_rows_for
    vp.DeviceTree.dense_rows_for = lambda self, cb, ca: 2  # a two-row pool: grown on demand
    try:
        out = planner.plan(belief, om, cfg, rng, keep_tree=True, trace=True)  # trace: the growing path
    finally:
        vp.DeviceTree.dense_rows_for = orig
    assert out.tree.cap_dense > 2 and out.tree.n_dense() > 2
    assert out.tree_stats == base.tree_stats and out.chosen_action == base.chosen_action
    got, want = out.tree.tables(), base.tree.tables()
    for k in INT_COLUMNS:
        np.testing.assert_array_equal(got[k], want[k], err_msg=k)
    np.testing.assert_allclose(got["prefs"], want["prefs"], rtol=1e-12, atol=1e-12)
    out.tree.validate()


def test_search_backup_api_from_interior_frontier():
    """Reference API: search from depth-1 beliefs, then backup to the root."""
    om = oracle.MarsModel(4, 3, layout_seed=0)
    belief = oracle.ParticleBelief.from_model(om, 500, oracle.RowRng.from_seed(0).derive(3))
    rng = oracle.RowRng.from_seed(0).derive(1, 0)
    # grow a small tree with the oracle plan then replay it onto the device tree
    cfg = oracle.SolverConfig(n_parallel=32, iterations=2)
    ref = oracle.plan(belief, om, cfg, rng)
    tree_o = ref.tree
    states = belief.sample_states(32, rng.derive(9))
    start = tree_o.nodes_at_depth(1)[0][:1].repeat(32)
    batch_o = oracle.SearchBatch(start, states, depth=1)
    # device tree with identical content via injected replay of the same plan
    traces = []
    oracle.plan(belief, om, cfg, rng, traces=traces)
    inject = [np.stack([lv["actions"] for lv in it["levels"]]) for it in traces]
    dev = vp.plan(belief, om, cfg, rng, precision="fp64", exact=True, keep_tree=True, inject_actions=inject).tree
    leaves_o = oracle.search(tree_o, om, batch_o, 3, 2.0, rng.derive(77))
    oracle.backup(tree_o, leaves_o, 3, 2.0, om.spec.discount)
    leaves_d = vp.search(dev, om, vp.SearchBatch(start, states, depth=1), 3, 2.0, vp.RowRng(rng.derive(77).key))
    np.testing.assert_array_equal(leaves_d.leaf_belief_indices, leaves_o.leaf_belief_indices)
    np.testing.assert_allclose(leaves_d.heuristic_values, leaves_o.heuristic_values, rtol=1e-13)
    vp.backup(dev, leaves_d, 3, 2.0, om.spec.discount)
    want, got = tree_o.tables(), dev.tables()
    for k in INT_COLUMNS:
        np.testing.assert_array_equal(got[k], want[k], err_msg=k)
    assert scale_close(got["prefs"], want["prefs"], 1e-10)


def test_tiger_decision_quality_vs_reference_solver():
    """Root decision of the fp32 device planner agrees with the reference
    planner on Tiger beliefs (SPEC.md:628 uses n_p = 1024)."""
    om = oracle.tiger_model()
    agree = 0
    cases = 0
    for p_left in (0.5, 0.2, 0.03, 0.97, 0.85):
        m = 2000
        k = int(round(p_left * m))
        states = oracle.TabularStates(np.array([0] * k + [1] * (m - k)), np.zeros(m, dtype=bool))
        belief = oracle.ParticleBelief(states, np.full(m, 1.0 / m))
        cfg = oracle.SolverConfig(n_parallel=1024, iterations=10)
        for s in range(3):
            rng = oracle.RowRng.from_seed(s).derive(1, 0)
            a_ref = oracle.plan(belief, om, cfg, rng).chosen_action
            a_dev = vp.plan(belief, om, cfg, rng, precision="fp32").chosen_action
            agree += a_ref == a_dev
            cases += 1
        if p_left >= 0.97:
            assert a_dev == 2  # confident tiger-left: open right
        if p_left <= 0.03:
            assert a_dev == 1
    assert agree >= cases - 2


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
@pytest.mark.parametrize("kind,n_par", [("mars7_8", 2048), ("mars11_11", 4096), ("tiger", 1024),
                                        ("synthetic", 2048), ("lightdark", 1024), ("navigation", 2048),
                                        ("crowdnav", 512)])
def test_fast_sampler_draws_follow_softmax_of_tree(kind, n_par, precision):
    """In-kernel fast draws (fresh rows via the shared initial CDF, other rows
    TMA-staged) equal the inverse CDF of softmax(eta * PSI) of the tree at the
    start of the iteration, for every row of every level."""
    seed = 3
    om = {"mars7_8": lambda: oracle.MarsModel(7, 8, layout_seed=seed),
          "mars11_11": lambda: oracle.MarsModel(11, 11, layout_seed=seed),
          "tiger": oracle.tiger_model, "synthetic": lambda: oracle.SyntheticModel(seed=seed),
          "lightdark": oracle.LightDarkModel, "navigation": oracle.NavigationModel,
          "crowdnav": lambda: oracle.CrowdNavModel(n_people=60)}[kind]()
    belief = oracle.ParticleBelief.from_model(om, 2000, oracle.RowRng.from_seed(seed).derive(3))
    rng = oracle.RowRng.from_seed(seed).derive(1, 0)
    k = 5
    before = vp.plan(belief, om, oracle.SolverConfig(n_parallel=n_par, iterations=k - 1), rng,
                     precision=precision, keep_tree=True).tree.tables()
    out = vp.plan(belief, om, oracle.SolverConfig(n_parallel=n_par, iterations=k), rng, precision=precision,
                  keep_tree=True, trace=True)
    prefs = before["prefs"]
    last = out.traces[-1]["levels"]
    search_rng = rng.derive(k - 1).derive(1)
    rows = np.arange(n_par)
    mism = total = 0
    belief_ids = np.zeros(n_par, dtype=np.int64)
    for lvl, tr in enumerate(last):
        u = search_rng.derive(lvl).derive(0).uniform(rows)
        known = belief_ids < len(prefs)  # beliefs created this iteration are fresh (init row)
        rowp = np.where(known[:, None], prefs[np.minimum(belief_ids, len(prefs) - 1)], 0.0)
        pol = oracle.softmax_rows(rowp, 2.0)
        cum = np.cumsum(pol, axis=1)
        want = np.minimum((cum <= u[:, None]).sum(axis=1), prefs.shape[1] - 1)
        got = tr["actions"]
        bad = np.flatnonzero(got != want)
        tol = 2e-5 if precision == "fp32" else 1e-12
        for i in bad:
            assert np.min(np.abs(cum[i] - u[i])) < tol, (lvl, i, got[i], want[i])
        mism += len(bad)
        total += n_par
        belief_ids = tr["next_beliefs"]
    assert mism <= max(3, 1e-3 * total)


@pytest.mark.parametrize("name", ["plan_mars7_8_c1", "plan_tiger", "plan_lightdark"])
@pytest.mark.parametrize("mode", [0, 1])
def test_vp_plan_modes_reproduce_reference(name, mode):
    """The CUDA-graph replay (mode 1) and direct launches (0) of vp_plan both
    reproduce the reference tree in fp64 parity mode; the second run of each
    planner replays with new keys/particles."""
    case = manifest()["plans"][name]
    g = load(name)
    planner = vp.Planner("fp64", exact=True)
    planner.mode = mode
    for run in case["runs"]:
        s = run["seed"]
        om, belief, cfg, rng = plan_inputs(case, s)
        out = planner.plan(belief, om, cfg, rng, keep_tree=True)
        assert out.tree_stats == run["tree_stats"]
        assert out.chosen_action == run["chosen_action"]
        t = out.tree.tables()
        for k in INT_COLUMNS:
            np.testing.assert_array_equal(t[k], g[f"s{s}_{k}"].astype(np.int64), err_msg=k)
        np.testing.assert_allclose(t["prefs"].sum(axis=1), g[f"s{s}_prefs_row_sum"], rtol=1e-9, atol=1e-8)


@pytest.mark.parametrize("mode", [0, 1])
def test_fp32_modes_agree(mode):
    """fp32 fast path: both vp_plan modes give the same tree structure
    (identical draws; only fp64 atomic summation order may differ)."""
    om = oracle.MarsModel(11, 11, layout_seed=5)
    belief = oracle.ParticleBelief.from_model(om, 4000, oracle.RowRng.from_seed(5).derive(3))
    cfg = oracle.SolverConfig(n_parallel=8192, iterations=6)
    rng = oracle.RowRng.from_seed(5).derive(1, 0)
    base = vp.Planner("fp32")
    base.mode = 0
    want = base.plan(belief, om, cfg, rng, keep_tree=True)
    p = vp.Planner("fp32")
    p.mode = mode
    got = p.plan(belief, om, cfg, rng, keep_tree=True)
    assert got.tree_stats == want.tree_stats
    a, b = got.tree.tables(), want.tree.tables()
    for k in INT_COLUMNS:
        np.testing.assert_array_equal(a[k], b[k], err_msg=k)
    assert scale_close(a["prefs"], b["prefs"], 1e-5)


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_search_backup_api_after_eta_change(precision):
    """The reference tree is eta-free: search / backup take eta per call (search.py:86,
    backup.py:75).  A device tree grown at eta = 2 and then searched and backed up at eta = 1
    must use LSEs / CDFs of eta = 1 everywhere (cached row LSEs and the initial row's CDF are
    recomputed on the eta change)."""
    om = oracle.MarsModel(4, 3, layout_seed=1)
    belief = oracle.ParticleBelief.from_model(om, 500, oracle.RowRng.from_seed(1).derive(3))
    rng = oracle.RowRng.from_seed(1).derive(1, 0)
    cfg = oracle.SolverConfig(n_parallel=64, iterations=3, eta=2.0)
    traces = []
    ref = oracle.plan(belief, om, cfg, rng, traces=traces)
    inject = [np.stack([lv["actions"] for lv in it["levels"]]) for it in traces]
    exact = precision == "fp64"
    dev = vp.plan(belief, om, cfg, rng, precision=precision, exact=exact, keep_tree=True,
                  inject_actions=inject).tree
    tree_o = ref.tree
    n = 64
    states = belief.sample_states(n, rng.derive(11))
    start = np.zeros(n, dtype=np.int64)
    # oracle draws at eta = 1, injected into the device search for fp32 (fp64 exact draws itself)
    tr_o = []
    leaves_o = oracle.search(tree_o, om, oracle.SearchBatch(start, states, depth=0), 3, 1.0, rng.derive(12),
                             trace=tr_o)
    kw = {} if exact else {"inject_actions": np.stack([lv["actions"] for lv in tr_o])}
    leaves_d = vp.search(dev, om, vp.SearchBatch(start, states, depth=0), 3, 1.0, vp.RowRng(rng.derive(12).key), **kw)
    np.testing.assert_array_equal(leaves_d.leaf_belief_indices, leaves_o.leaf_belief_indices)
    oracle.backup(tree_o, leaves_o, 3, 1.0, om.spec.discount)
    vp.backup(dev, leaves_d, 3, 1.0, om.spec.discount)
    want, got = tree_o.tables(), dev.tables()
    for k in INT_COLUMNS:
        np.testing.assert_array_equal(got[k], want[k], err_msg=k)
    assert scale_close(got["prefs"], want["prefs"], 1e-10 if exact else 1e-5)
