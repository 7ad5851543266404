"""The reference's acceptance criteria that have oracles (SPEC.md ACCEPTANCE 1, 4, 5;
/root/reference/pkg/src/vecpomdp/oracle.py), on the device.

1. Backup vs the serial per-node backup: 200 random trees (depth <= 4, <= 50
   beliefs, |A| <= 6, random rewards and heuristics, 1-3 passes), built by the
   device search from recorded trajectories (search_recorded, VP_SEARCH_INSERT)
   and backed up by the device kernel; every PSI entry within 1e-6 absolute of
   oracle/acceptance.serial_backup (pinned to the reference's serial_backup).
4. Tiger decisions against exact value iteration (the reference's alpha vectors
   at horizon 20, tests/golden/acceptance.npz): the device's decisions equal the
   reference planner's (fp64 parity mode) at every sampled belief, and its
   agreement with the optimum is reported and bounded; closed-loop return vs V*.
5. Device SIR vs exact_bayes_filter on random 2-state chains: m = 10^5
   particles, 50 sequences of 10 (a, o) steps, within 0.01 absolute.
"""

import numpy as np
import pytest

import oracle
import paper_2510_27191_b200 as vp
from golden_cases import load
from oracle import acceptance as acc

pytestmark = pytest.mark.gpu

G = load("acceptance")


def descriptor_model(A: int, O: int = 3):
    """Any device model with |A| actions: insert mode replays given samples, it never steps."""
    t = np.tile(np.eye(2), (A, 1, 1))
    z = np.full((A, 2, O), 1.0 / O)
    return vp.TabularModel(vp.TabularPOMDP(t, z, np.zeros((2, A)), np.array([1.0, 0.0]), 0.9,
                                           np.array([False, False]), "replay", 10))


def device_run(A, passes, eta, gamma, precision, exact):
    tree = vp.DeviceTree(A, precision=precision, exact=exact, eta=eta, cap_beliefs=64, cap_actions=64)
    model = descriptor_model(A)
    for p in passes:
        leaves = vp.search_recorded(tree, model, p["actions"], p["observations"], p["rewards"], p["leaf"])
        vp.backup(tree, leaves, p["d"], eta, gamma)
    return tree


@pytest.mark.parametrize("precision,exact,tol", [("fp64", True, 1e-6), ("fp64", False, 1e-6), ("fp32", False, None)])
def test_spec1_backup_matches_serial_on_200_random_trees(precision, exact, tol):
    worst = 0.0
    for k in range(200):
        A, passes = acc.random_tree_case(np.random.default_rng(k))
        serial = acc.serial_run(A, passes, 2.0, 0.9)
        tree = device_run(A, passes, 2.0, 0.9, precision, exact)
        t = tree.tables()
        paths = acc.belief_paths(t["parent_action"], t["parent_obs"], t["action_parent_belief"], t["action_id"])
        assert sorted(paths) == sorted(serial.prefs), k
        for i, p in enumerate(paths):
            want = np.array(serial.prefs[p])
            err = np.abs(t["prefs"][i] - want)
            if tol is None:  # fp32 storage: the scale-aware 1e-5 relative contract
                err = err / max(1.0, float(np.abs(want).max()))
            worst = max(worst, float(err.max()))
        # visits / rewards are the rows' own sums
        got_v = {paths[int(t["action_parent_belief"][x])] + (int(t["action_id"][x]),): int(t["action_visits"][x])
                 for x in range(len(t["action_id"]))}
        assert got_v == serial.visits, k
    assert worst <= (tol if tol is not None else 1e-5), worst


def tiger_belief(p_left: float, m: int = 2000):
    k = int(round(p_left * m))
    states = oracle.TabularStates(np.array([0] * k + [1] * (m - k)), np.zeros(m, dtype=bool))
    return oracle.ParticleBelief(states, np.full(m, 1.0 / m)), k / m


def test_spec4_tiger_decisions_vs_exact_value_iteration():
    """SPEC.md:628 protocol (n_p = 1024, eta = 2, fixed iterations; 100 beliefs sampled
    uniformly).  The shipped reference planner (heuristic 0, depth <= 10) opens early
    near p = 0.03 / 0.95 where the horizon-20 optimum still listens, so it agrees with the
    optimum on ~89 % of uniform beliefs; the device must make the reference's decisions
    (fp64 parity mode) and so inherits that rate (asserted >= 85 %, reported)."""
    om = oracle.tiger_model()
    vi = acc.AlphaSet(G["vi_h20_alphas"], G["vi_h20_actions"])
    g = np.random.default_rng(0)
    cfg = oracle.SolverConfig(n_parallel=1024, iterations=10)
    agree_dev = agree_ref = same = 0
    for i, p in enumerate(g.uniform(0.0, 1.0, size=100)):
        belief, p = tiger_belief(p)
        rng = oracle.RowRng.from_seed(i).derive(1, 0)
        a_dev = vp.plan(belief, om, cfg, rng, precision="fp64", exact=True).chosen_action
        a_ref = oracle.plan(belief, om, cfg, rng).chosen_action
        best = vi.action([p, 1.0 - p, 0.0])
        agree_dev += a_dev == best
        agree_ref += a_ref == best
        same += a_dev == a_ref
    print(f"tiger: device agrees with the horizon-20 optimum on {agree_dev}/100 beliefs, "
          f"the reference planner on {agree_ref}/100; device == reference on {same}/100")
    assert same == 100
    assert agree_dev >= 85
    # the fp32 fast path decides like the parity mode on the unambiguous beliefs
    for p_left, want in ((0.5, 0), (0.2, 0), (0.8, 0), (0.005, 1), (0.995, 2)):
        belief, p = tiger_belief(p_left)
        got = vp.plan(belief, om, cfg, oracle.RowRng.from_seed(7).derive(1, 0)).chosen_action
        assert got == want == vi.action([p, 1.0 - p, 0.0]), p_left


def test_spec4_tiger_return_vs_optimum():
    """200 closed-loop episodes (device planner, device SIR); the mean discounted return
    lies within 10 % of V*(b0) or within its own 95 % CI of it (one wrong door costs 110, so
    200 episodes resolve the mean only to a few units)."""
    om = vp.tiger_model()
    vi = acc.AlphaSet(G["vi_h20_alphas"], G["vi_h20_actions"])
    v_star = vi.value([0.5, 0.5, 0.0])
    cfg = vp.SolverConfig(n_parallel=1024, iterations=10, particles=2000)
    rets = np.array([vp.run_episode(om, cfg, seed=s).discounted_return for s in range(200)])
    mean, half = rets.mean(), 1.96 * rets.std(ddof=1) / np.sqrt(len(rets))
    print(f"tiger: mean discounted return {mean:.3f} +- {half:.3f} (95% CI) vs V*(b0) = {v_star:.3f}")
    assert abs(mean - v_star) <= max(0.1 * abs(v_star), half)


def chain_model(g):
    t = g.dirichlet([2.0, 2.0], size=(2, 2))
    z = g.dirichlet([2.0, 2.0], size=(2, 2))
    pomdp = vp.TabularPOMDP(t, z, np.zeros((2, 2)), np.array([0.5, 0.5]), 0.95, np.array([False, False]), "chain", 50)
    return vp.TabularModel(pomdp), pomdp


@pytest.mark.parametrize("exact", [True, False])
def test_spec5_device_sir_matches_exact_bayes_filter(exact):
    m = 100_000
    worst = 0.0
    for k in range(50):
        g = np.random.default_rng(3000 + k)
        model, pomdp = chain_model(g)
        host = vp.ParticleBelief(model.states_from_indices(np.repeat([0, 1], m // 2)), np.full(m, 1.0 / m))
        belief = vp.DeviceBelief.from_host(host, model)
        b = np.array([0.5, 0.5])
        rng = vp.RowRng.from_seed(k)
        for t in range(10):
            a = int(g.integers(0, 2))
            o = int(g.choice(2, p=pomdp.observations[a].T @ (pomdp.transitions[a].T @ b)))
            b = acc.exact_bayes_filter(pomdp, b, a, o)
            upd = vp.sir_update(belief, model, a, o, rng.derive(t), exact=exact)
            belief = upd.belief
            assert not upd.degenerate
            est = np.bincount(belief.states.idx, minlength=2) / m
            worst = max(worst, float(np.abs(est - b).max()))
    print(f"SIR vs exact filter: worst |posterior error| {worst:.4f} over 50 x 10 updates")
    assert worst <= 0.01


@pytest.mark.parametrize("case", __import__("golden_cases").SERIAL_CASES)
@pytest.mark.parametrize("precision,exact", [("fp64", True), ("fp64", False), ("fp32", False)])
def test_width1_device_search_equals_reference_serial_search(case, precision, exact):
    """SPEC ACCEPTANCE 2: with n_p = 1, fixed seeds, d_max <= 4, on 4x4 MARS toys, the device
    search + backup (one width-1 pass per episode) rebuild the reference's serial_search_backup
    tree: integer fields bit-identical, floats within 1e-9 (fp64; fp32 storage: 1e-5 relative)."""
    from golden_cases import parse_tree_text, serial_search_build

    n, m, seed = case[:3]
    want_i, want_f = parse_tree_text(str(load("serial_search")[f"mars{n}_{m}_s{seed}"]))
    tree = serial_search_build(vp, case, lambda model: vp.init_tree(model.spec, eta=case[5], precision=precision,
                                                                     exact=exact))
    got_i, got_f = parse_tree_text(tree.serialize())
    assert got_i == want_i
    if precision == "fp64":
        np.testing.assert_allclose(got_f, want_f, rtol=0, atol=1e-9)
    else:
        np.testing.assert_allclose(got_f, want_f, rtol=1e-5, atol=1e-5 * np.abs(want_f).max())


@pytest.mark.parametrize("precision,exact", [("fp64", True), ("fp64", False), ("fp32", False)])
def test_formula_checks_spec3(precision, exact):
    """SPEC ACCEPTANCE 3 (Eq. 3 / Eq. 6 properties) on the device LSE: max <= LSE <= max + log|A|/eta
    on 10^5 random rows; constant-row LSE = c + log|A|/eta within 1e-12 (fp64); the softmax built
    from it sums to 1 within 1e-9 and is shift-invariant."""
    g = np.random.default_rng(11)
    eta = 2.0
    for A in (2, 9, 64, 256):
        rows = g.normal(size=(100_000 // A * 4 if A > 16 else 100_000, A)) * 5.0
        if precision == "fp32":
            rows = rows.astype(np.float32).astype(np.float64)
        lse = vp.log_sum_exp_rows(rows, eta, precision=precision, exact=exact)
        mx = rows.max(axis=1)
        slack = 1e-12 if precision == "fp64" else 1e-5 * np.maximum(np.abs(mx), 1.0)
        assert np.all(lse >= mx - slack) and np.all(lse <= mx + np.log(A) / eta + slack)
        p = np.exp(eta * (rows - lse[:, None]))
        tol = 1e-9 if precision == "fp64" else 1e-5
        assert np.all(np.abs(p.sum(axis=1) - 1.0) <= tol)
        shift = g.normal(size=(len(rows), 1)) * 3.0
        if precision == "fp32":
            shift = np.round(shift * 8) / 8  # exactly representable shifts keep fp32 rows exact
        lse2 = vp.log_sum_exp_rows(rows + shift, eta, precision=precision, exact=exact)
        p2 = np.exp(eta * (rows + shift - lse2[:, None]))
        np.testing.assert_allclose(p2, p, rtol=0, atol=tol)
        c = g.normal(size=(1000, 1)) * 10.0
        const = np.repeat(c, A, axis=1)
        lc = vp.log_sum_exp_rows(const, eta, precision=precision, exact=exact)
        want = c[:, 0] + np.log(A) / eta
        if precision == "fp64":
            np.testing.assert_allclose(lc, want, rtol=0, atol=1e-12)
        else:
            np.testing.assert_allclose(lc, want, rtol=1e-6, atol=1e-5)


def test_batch_scaling_sanity_spec10():
    """SPEC ACCEPTANCE 10: episodes simulated per second at n_p = 32 768 are >= 8x those at
    n_p = 1 024 (RockSample(7,8), 8 iterations, belief resident, median of 5 planning steps)."""
    import torch
    from paper_2510_27191_b200.rng import key_of

    model = vp.MarsModel(7, 8, layout_seed=1)
    belief = vp.ParticleBelief.from_model(model, 2000, vp.RowRng.from_seed(1).derive(3))
    rate = {}
    for n in (1024, 32768):
        cfg = vp.SolverConfig(n_parallel=n, iterations=8)
        planner = vp.Planner("fp32")
        dm = vp.device_model(model)
        _, _, m = planner.upload_belief(dm, belief)
        ms = []
        for t in range(8):
            d, tree, work = planner.prepare(model, cfg, device_init=False)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            planner.run_fixed(d, tree, work, m, model.spec, cfg, key_of(vp.RowRng.from_seed(1).derive(1, t)),
                              from_host=False)
            e1.record()
            torch.cuda.synchronize()
            if t >= 3:
                ms.append(e0.elapsed_time(e1))
        rate[n] = n * sum(range(1, 9)) / sorted(ms)[len(ms) // 2]
    assert rate[32768] >= 8.0 * rate[1024], rate


@pytest.mark.parametrize("model_name", ["mars", "crowdnav"])
def test_structural_invariants_through_a_campaign_spec9(model_name):
    """SPEC ACCEPTANCE 9: through a closed loop (device belief, device SIR), every planning step's
    tree has unique A-pairs and B-pairs and conserves visits (sum of visits = rows x levels
    expanded), and every belief update leaves normalised weights."""
    import torch

    model = vp.MarsModel(7, 8, layout_seed=3) if model_name == "mars" else vp.CrowdNavModel(n_people=40)
    cfg = vp.SolverConfig(n_parallel=1024, iterations=6, particles=1000)
    root = vp.RowRng.from_seed(11)
    env = model.sample_initial_states(1, root.derive(0, 0))
    belief = vp.DeviceBelief.from_host(vp.ParticleBelief.from_model(model, cfg.particles, root.derive(3)), model)
    for t in range(8):
        out = vp.plan(belief, model, cfg, root.derive(1, t), keep_tree=True)
        out.tree.validate()  # unique (belief, action) and (action, observation) edges, depth chain
        visits = out.tree.tables()["action_visits"].sum()
        assert visits == cfg.n_parallel * sum(min(i + 1, cfg.d_max_cap) for i in range(cfg.iterations))
        res = model.step_batch(env, np.array([out.chosen_action]), root.derive(2, t).bind([0]))
        if bool(res.next_states.terminal[0]):
            break
        upd = vp.sir_update(belief, model, out.chosen_action, int(res.observations[0]), root.derive(4, t),
                            exact=False)
        w = upd.belief.weights_dev.double()
        assert torch.isfinite(w).all() and abs(float(w.sum()) - 1.0) < 1e-9
        env, belief = res.next_states, upd.belief
