"""Generate golden vectors from the REAL reference (run in the build container).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py            # everything
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py crowdnav   # only the CrowdNav cases
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py large      # only the C2 / C3 digests

Imports ``vecpomdp`` from /root/reference/pkg/src (read-only, never copied)
and writes small ``.npz`` fixtures next to this script.  The GPU box has no
/root/reference, so tests only ever read the committed fixtures.

Cases (see SURVEY.md section 4 "parity ladder" and Appendix C):
* rng_*       -- RowRng / BoundRng draws (rng.py:26-120)
* formulas    -- softmax / LSE / sample_actions / match_or_append_pairs /
                 aggregate_leaves / action_q_values examples
* plan_*      -- full ``plan()`` trees on MARS, Tiger and (reference solver
                 driving the oracle's new models) Synthetic and Light-Dark
* large_*     -- digests of full-size C2 / C3 ``plan()`` trees (MARS(11,11) 16384 x 10,
                 MARS(15,15) 65536 x 10)
* episode_*   -- closed-loop ``run_episode`` records
* acceptance  -- the reference's acceptance oracles (oracle.py; SPEC.md ACCEPTANCE 1, 4, 5):
                 serial_backup on random trees, exact_value_iteration on Tiger,
                 exact_bayes_filter on random 2-state chains
* serial_search -- SPEC.md ACCEPTANCE 2: the reference's serial_search_backup trees
                 (width-1 episodes, 4x4 MARS toys, d_max <= 4) as to_text() dumps
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

import vecpomdp as ref  # noqa: E402
from vecpomdp.envs import MarsModel, tiger_model  # noqa: E402
from vecpomdp.envs.navigation import NavigationModel  # noqa: E402
from vecpomdp.envs.crowdnav import CrowdNavModel  # noqa: E402

import oracle  # noqa: E402  (only for the two NEW models the reference lacks)


def tree_arrays(tree, full_prefs: bool) -> dict:
    out = {
        "parent_action": tree.parent_action.astype(np.int32),
        "parent_obs": tree.parent_obs.astype(np.int64),
        "depth": tree.depth.astype(np.int16),
        "action_parent_belief": tree.action_parent_belief.astype(np.int32),
        "action_id": tree.action_id.astype(np.int16),
        "action_reward_sum": tree.action_reward_sum.copy(),
        "action_visits": tree.action_visits.astype(np.int32),
        "prefs_row_sum": tree.prefs.sum(axis=1),
        "prefs_root": tree.prefs[0].copy(),
    }
    if full_prefs:
        out["prefs"] = tree.prefs.copy()
    return out


def gen_rng():
    out = {}
    rows = np.concatenate([np.arange(64), np.array([1000, 123456, 2**31 - 1, 2**40 + 7])]).astype(np.int64)
    seeds = [0, 1, 42, 2**63 + 5, 123456789]
    keys, uni, uni3, nor = [], [], [], []
    for s in seeds:
        r = ref.RowRng.from_seed(s)
        for path in [(), (0,), (1, 0), (3, 5, 7), (2, 11)]:
            d = r.derive(*path)
            keys.append(int(d.key))
            uni.append(d.uniform(rows))
            uni3.append(d.uniform(rows, 3))
            nor.append(d.normal(rows, 2))
    out["rows"] = rows
    out["keys"] = np.array(keys, dtype=np.uint64)
    out["uniform"] = np.stack(uni)
    out["uniform_k3"] = np.stack(uni3)
    out["normal_k2"] = np.stack(nor)
    out["uniform1"] = np.array([ref.RowRng.from_seed(12).derive(4).uniform1()])
    np.savez_compressed(os.path.join(HERE, "rng.npz"), **out)


def gen_formulas():
    g = np.random.default_rng(7)
    out = {}
    rows = g.normal(size=(40, 13)) * 3.0
    out["lse_in"] = rows
    out["lse_eta2"] = ref.log_sum_exp_rows(rows, 2.0)
    out["softmax_eta2"] = ref.softmax_rows(rows, 2.0)
    # sample_actions with groups (multi-group path) and single group path
    pol = ref.softmax_rows(g.normal(size=(5, 7)), 1.5)
    groups = g.integers(0, 5, size=300)
    rng = ref.RowRng.from_seed(3).derive(9)
    out["sa_pol"] = pol
    out["sa_groups"] = groups
    out["sa_multi"] = ref.sample_actions(pol, rng.bind(np.arange(300)), groups=groups)
    out["sa_single"] = ref.sample_actions(pol[:1], rng.bind(np.arange(300)), groups=np.zeros(300, dtype=np.int64))
    # match_or_append_pairs on 10^4 random pairs
    ex = np.unique(g.integers(0, 50, size=(300, 2)), axis=0)
    g.shuffle(ex)
    q = g.integers(0, 60, size=(10_000, 2))
    rows_out, n_new = ref.match_or_append_pairs(ex, q)
    out["moa_existing"], out["moa_query"], out["moa_rows"], out["moa_new"] = ex, q, rows_out, np.array([n_new])
    np.savez_compressed(os.path.join(HERE, "formulas.npz"), **out)


def make_model(kind: str, seed: int):
    if kind.startswith("mars"):
        n, m = map(int, kind[4:].split("_"))
        return MarsModel(n=n, m=m, layout_seed=seed)
    if kind == "tiger":
        return tiger_model()
    if kind == "synthetic":
        return oracle.SyntheticModel(n_actions=16, n_obs=8, seed=seed)
    if kind == "lightdark":
        return oracle.LightDarkModel()
    if kind == "navigation":
        return NavigationModel()
    if kind.startswith("crowdnav"):
        return CrowdNavModel(n_people=int(kind[8:] or 300))
    raise ValueError(kind)


# (name, model kind, n_parallel, iterations, seeds, full_prefs)
PLAN_CASES = [
    ("plan_mars4_3", "mars4_3", 64, 6, [0, 1, 2], True),
    ("plan_mars7_8_c1", "mars7_8", 1024, 8, [0, 1], False),
    ("plan_mars7_8_small", "mars7_8", 96, 5, [3], True),
    ("plan_tiger", "tiger", 256, 8, [0, 1], True),
    ("plan_synthetic", "synthetic", 256, 6, [0, 1], True),
    ("plan_lightdark", "lightdark", 128, 5, [0, 1], True),
    ("plan_navigation", "navigation", 256, 6, [0, 1], True),
]
CROWD_PLAN_CASES = [
    ("plan_crowdnav40", "crowdnav40", 128, 5, [0, 1], True),
    ("plan_crowdnav", "crowdnav", 64, 3, [0], True),
]


def gen_plans(cases=PLAN_CASES + CROWD_PLAN_CASES, particles=2000):
    manifest = {}
    for name, kind, n_par, iters, seeds, full in cases:
        arrays = {}
        meta = []
        for s in seeds:
            model = make_model(kind, s)
            belief = ref.ParticleBelief.from_model(model, particles, ref.RowRng.from_seed(s).derive(3))
            cfg = ref.SolverConfig(n_parallel=n_par, iterations=iters, eta=2.0)
            out = ref.plan(belief, model, cfg, ref.RowRng.from_seed(s).derive(1, 0))
            for k, v in tree_arrays(out.tree, full).items():
                arrays[f"s{s}_{k}"] = v
            meta.append({"seed": s, "chosen_action": out.chosen_action, "iterations_run": out.iterations_run,
                         "final_d_max": out.final_d_max, "tree_stats": out.tree_stats})
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **arrays)
        manifest[name] = {"kind": kind, "n_parallel": n_par, "iterations": iters, "particles": particles,
                          "eta": 2.0, "runs": meta}
    return manifest


def gen_episodes():
    out = {}
    cfg = ref.SolverConfig(n_parallel=64, iterations=4, particles=500)
    recs = []
    for s in range(3):
        rec = ref.run_episode(MarsModel(n=4, m=3, layout_seed=s), cfg, seed=s)
        recs.append({"seed": s, "return": rec.discounted_return, "steps": rec.steps,
                     "reason": rec.terminal_reason, "degenerate": rec.degenerate_updates})
    out["episode_mars4_3"] = recs
    # a larger sample for the statistical closed-loop check (fp32 device planner)
    cfg = ref.SolverConfig(n_parallel=256, iterations=5, particles=1000)
    recs = []
    for s in range(100, 130):
        rec = ref.run_episode(MarsModel(n=5, m=4, layout_seed=7), cfg, seed=s)
        recs.append({"seed": s, "return": rec.discounted_return, "steps": rec.steps})
    out["episode_mars5_4_campaign"] = recs
    return out


def gen_navigation_steps():
    """Navigation model vectors (navigation.py:172-251): steps from random states / actions,
    likelihoods of the realised observations, heuristics."""
    model = NavigationModel()
    n = 400
    st = model.sample_initial_states(n, ref.RowRng.from_seed(21))
    out = {"pos0": st.pos, "occ0": st.occ, "gate0": st.open_gate}
    for t in range(8):
        a = (ref.RowRng.from_seed(22 + t).uniform(np.arange(n)) * 9).astype(np.int64)
        res = model.step_batch(st, a, ref.RowRng.from_seed(40 + t).bind(np.arange(n)))
        out[f"a{t}"] = a
        out[f"pos{t + 1}"] = res.next_states.pos
        out[f"term{t + 1}"] = res.next_states.terminal
        out[f"obs{t + 1}"] = res.observations
        out[f"rew{t + 1}"] = res.rewards
        o = int(res.observations[0])
        out[f"ll{t + 1}"] = model.observation_log_likelihood(res.next_states, int(a[0]), o)
        out[f"llobs{t + 1}"] = np.array([int(a[0]), o])
        out[f"h{t + 1}"] = model.value_heuristic(res.next_states)
        st = res.next_states
    np.savez_compressed(os.path.join(HERE, "nav_steps.npz"), **out)


def gen_crowd_episodes():
    """Closed-loop CrowdNav episodes (reference run_episode with its refresh / reconcile hooks)."""
    cfg = ref.SolverConfig(n_parallel=128, iterations=4, particles=300)
    recs = []
    for s in range(2):
        rec = ref.run_episode(CrowdNavModel(n_people=40, hall_depth=8.0, max_steps=15), cfg, seed=s)
        recs.append({"seed": s, "return": rec.discounted_return, "steps": rec.steps, "reason": rec.terminal_reason,
                     "degenerate": rec.degenerate_updates, "counters": rec.counters})
    return recs


CROWD_FIELDS = ("robot", "persons", "curious", "tracked", "prev_dist", "last_code", "terminal")


def gen_crowd_steps():
    """CrowdNav vectors (crowdnav.py:98-224): 6 steps of 96 rows with 40 people (every
    field after every step except the people, kept at the start and the end) and 3
    steps of 8 rows at the default 300 people; likelihoods, heuristics, refresh."""
    out = {}
    for tag, people, n, steps in (("p40", 40, 96, 6), ("p300", 300, 8, 3)):
        model = CrowdNavModel(n_people=people)
        st = model.sample_initial_states(n, ref.RowRng.from_seed(31))
        for f in CROWD_FIELDS:
            out[f"{tag}_{f}0"] = getattr(st, f)
        for t in range(steps):
            a = (ref.RowRng.from_seed(32 + t).uniform(np.arange(n)) * 5).astype(np.int64)
            a[: n // 4] = 0  # a quarter of the rows walk north
            res = model.step_batch(st, a, ref.RowRng.from_seed(50 + t).bind(np.arange(n)))
            out[f"{tag}_a{t}"] = a
            for f in ("robot", "prev_dist", "last_code", "terminal"):
                out[f"{tag}_{f}{t + 1}"] = getattr(res.next_states, f)
            out[f"{tag}_obs{t + 1}"], out[f"{tag}_rew{t + 1}"] = res.observations, res.rewards
            o = int(res.observations[1])
            out[f"{tag}_ll{t + 1}"] = model.observation_log_likelihood(res.next_states, int(a[1]), o)
            out[f"{tag}_llobs{t + 1}"] = np.array([int(a[1]), o])
            out[f"{tag}_h{t + 1}"] = model.value_heuristic(res.next_states)
            st = res.next_states
        out[f"{tag}_persons_end"] = st.persons
        ref_st = model.refresh_executed(st.take([2]))
        out[f"{tag}_refresh_tracked"], out[f"{tag}_refresh_prev"] = ref_st.tracked, ref_st.prev_dist
    np.savez_compressed(os.path.join(HERE, "crowd_steps.npz"), **out)


# Full-size BASELINE configs: the trees are too large to commit,
# so each run stores SHA-256 digests of every integer column in reference order (and of the
# reward sums, which are exact integers for MARS), the per-depth belief counts, the root PSI row
# the PSI row sums of the first LARGE_HEAD rows, and per-depth totals of the row sums and of |PSI|.
# (name, (n, m), n_parallel, iterations, [(seed, plan step t)])  -- plan key RowRng(seed).derive(1, t)
LARGE_CASES = [
    ("large_c2", (11, 11), 16384, 10, [(1000, 5), (1000, 24)]),
    ("large_c3", (15, 15), 65536, 10, [(1000, 0)]),
]
LARGE_PARTICLES = 10_000
LARGE_HEAD = 1 << 15


def column_digests(tree) -> dict:
    import hashlib

    cols = {"parent_action": tree.parent_action, "parent_obs": tree.parent_obs, "depth": tree.depth,
            "action_parent_belief": tree.action_parent_belief, "action_id": tree.action_id,
            "action_visits": tree.action_visits}
    out = {k: hashlib.sha256(np.ascontiguousarray(v, dtype="<i8").tobytes()).hexdigest() for k, v in cols.items()}
    out["action_reward_sum"] = hashlib.sha256(
        np.ascontiguousarray(tree.action_reward_sum, dtype="<f8").tobytes()).hexdigest()
    return out


def gen_large(cases=LARGE_CASES):
    manifest = {}
    for name, (n, m), n_par, iters, runs in cases:
        arrays, meta = {}, []
        for seed, t in runs:
            model = MarsModel(n=n, m=m, layout_seed=seed)
            belief = ref.ParticleBelief.from_model(model, LARGE_PARTICLES, ref.RowRng.from_seed(seed).derive(3))
            cfg = ref.SolverConfig(n_parallel=n_par, iterations=iters, eta=2.0)
            out = ref.plan(belief, model, cfg, ref.RowRng.from_seed(seed).derive(1, t))
            tree = out.tree
            tag = f"s{seed}_t{t}"
            arrays[f"{tag}_prefs_root"] = tree.prefs[0].copy()
            rs = tree.prefs.sum(axis=1)
            arrays[f"{tag}_prefs_row_sum_head"] = rs[:LARGE_HEAD].copy()
            arrays[f"{tag}_prefs_row_sum_by_depth"] = np.bincount(tree.depth, weights=rs)
            arrays[f"{tag}_prefs_abs_sum_by_depth"] = np.bincount(tree.depth, weights=np.abs(tree.prefs).sum(axis=1))
            arrays[f"{tag}_depth_counts"] = np.bincount(tree.depth).astype(np.int64)
            meta.append({"seed": seed, "t": t, "chosen_action": out.chosen_action, "tree_stats": out.tree_stats,
                         "iterations_run": out.iterations_run, "digests": column_digests(tree)})
            print(name, tag, out.tree_stats, out.chosen_action, flush=True)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **arrays)
        manifest[name] = {"mars": [n, m], "n_parallel": n_par, "iterations": iters, "particles": LARGE_PARTICLES,
                          "eta": 2.0, "runs": meta}
    return manifest


ACCEPT_TREES = 24        # random serial_backup cases (SPEC #1 family)
ACCEPT_HORIZONS = (1, 2, 3, 5, 8)  # Tiger exact value iteration
ACCEPT_FILTERS = 10      # random 2-state chains x 10 (a, o) steps


# SPEC #2 (oracle equivalence -- search): width-1 episodes on a 4x4 MARS toy, the reference's
# serial_search_backup (oracle.py:176-206) building the tree episode by episode
SERIAL_CASES = [(4, 3, 5, 2, 30, 0.05), (4, 3, 6, 3, 30, 0.1), (4, 4, 7, 4, 40, 0.05)]  # n, m, seed, d cap, episodes, eta


def gen_serial_search():
    from vecpomdp import oracle as ro

    out = {}
    for n, m, seed, dcap, episodes, eta in SERIAL_CASES:
        model = MarsModel(n=n, m=m, layout_seed=seed)
        belief = ref.ParticleBelief.from_model(model, 200, ref.RowRng.from_seed(seed).derive(3))
        tree = ro.SerialTree(model.spec.action_count)
        for e in range(episodes):
            it = ref.RowRng.from_seed(seed).derive(1, e)
            state = belief.sample_states(1, it.derive(0))
            ro.serial_search_backup(model, state, it.derive(1), min(e + 1, dcap), eta, model.spec.discount,
                                    tree=tree)
        out[f"mars{n}_{m}_s{seed}"] = np.array(tree.to_text())
    np.savez_compressed(os.path.join(HERE, "serial_search.npz"), **out)
    print("serial_search:", list(out))


def two_state_chain(g):
    """A random 2-state, 2-action, 2-observation tabular chain (SPEC #5)."""
    t = g.dirichlet([2.0, 2.0], size=(2, 2))
    z = g.dirichlet([2.0, 2.0], size=(2, 2))
    r = g.normal(size=(2, 2))
    return ref.envs.tabular.TabularPOMDP(t, z, r, np.array([0.5, 0.5]), 0.95, np.array([False, False]), "chain", 50)


def gen_acceptance():
    """Outputs of the reference's own acceptance oracles (oracle.py:124-173, 259-323)."""
    from vecpomdp import oracle as ro
    from oracle.acceptance import random_tree_case

    out = {}
    for k in range(ACCEPT_TREES):
        A, passes = random_tree_case(np.random.default_rng(1000 + k))
        tree = ro.SerialTree(A)
        for p in passes:
            leaves = []
            for r in range(p["actions"].shape[1]):
                node = tree.root
                for lvl in range(p["d"]):
                    x = tree.get_or_add_action(node, int(p["actions"][lvl, r]))
                    x.visits += 1
                    x.reward_sum += float(p["rewards"][lvl, r])
                    node = tree.get_or_add_child(x, int(p["observations"][lvl, r]))
                leaves.append((node, float(p["leaf"][r])))
            ro.serial_backup(tree, leaves, p["d"], 2.0, 0.9)
        paths = []
        for b in tree.beliefs:
            path, cur = [], b
            while cur.parent_action is not None:
                path = [cur.parent_action.action, cur.parent_obs] + path
                cur = cur.parent_action.parent
            paths.append(tuple(path))
        order = sorted(range(len(paths)), key=lambda i: paths[i])
        out[f"tree{k}_prefs"] = np.array([tree.beliefs[i].prefs for i in order], dtype=np.float64)
        out[f"tree{k}_paths"] = np.array([list(paths[i]) + [-1] * (8 - len(paths[i])) for i in order], dtype=np.int64)
    tiger = ref.envs.tabular.tiger_model()
    grid = np.linspace(0.0, 1.0, 41)
    beliefs = np.stack([grid, 1.0 - grid, np.zeros_like(grid)], axis=1)
    out["vi_beliefs"] = beliefs
    for h in ACCEPT_HORIZONS:
        v = ro.exact_value_iteration(tiger.pomdp, h)
        out[f"vi_h{h}_values"] = np.array([v.value(b) for b in beliefs])
        out[f"vi_h{h}_actions"] = np.array([v.action(b) for b in beliefs], dtype=np.int64)
    v = ro.exact_value_iteration(tiger.pomdp, 20)  # the decision-quality ground truth (SPEC #4)
    out["vi_h20_alphas"], out["vi_h20_actions"] = v.alphas, v.actions.astype(np.int64)
    for k in range(ACCEPT_FILTERS):
        g = np.random.default_rng(2000 + k)
        pomdp = two_state_chain(g)
        b = np.array([0.5, 0.5])
        seq, post = [], []
        for _ in range(10):
            a = int(g.integers(0, 2))
            pred = pomdp.transitions[a].T @ b
            o = int(g.choice(2, p=pomdp.observations[a].T @ pred))
            b = ro.exact_bayes_filter(pomdp, b, a, o)
            seq.append((a, o))
            post.append(b)
        out[f"chain{k}_T"], out[f"chain{k}_Z"], out[f"chain{k}_R"] = pomdp.transitions, pomdp.observations, pomdp.rewards
        out[f"chain{k}_seq"] = np.array(seq, dtype=np.int64)
        out[f"chain{k}_post"] = np.array(post)
    np.savez_compressed(os.path.join(HERE, "acceptance.npz"), **out)
    print("acceptance: trees", ACCEPT_TREES, "horizons", ACCEPT_HORIZONS, "chains", ACCEPT_FILTERS)


if __name__ == "__main__":
    if sys.argv[1:] == ["acceptance"]:
        gen_acceptance()
        sys.exit(0)
    if sys.argv[1:] == ["serial"]:
        gen_serial_search()
        sys.exit(0)
    if sys.argv[1:] == ["large"]:
        with open(os.path.join(HERE, "manifest.json")) as f:
            manifest = json.load(f)
        manifest["large_plans"] = gen_large()
        with open(os.path.join(HERE, "manifest.json"), "w") as f:
            json.dump(manifest, f, indent=1, sort_keys=True)
        sys.exit(0)
    if sys.argv[1:] == ["crowdnav"]:
        gen_crowd_steps()
        with open(os.path.join(HERE, "manifest.json")) as f:
            manifest = json.load(f)
        manifest["plans"].update(gen_plans(CROWD_PLAN_CASES))
        manifest["episodes"]["episode_crowdnav40"] = gen_crowd_episodes()
        with open(os.path.join(HERE, "manifest.json"), "w") as f:
            json.dump(manifest, f, indent=1, sort_keys=True)
        sys.exit(0)
    gen_crowd_steps()
    gen_navigation_steps()
    gen_rng()
    gen_formulas()
    gen_acceptance()
    gen_serial_search()
    manifest = {"plans": gen_plans(), "large_plans": gen_large(), "episodes": dict(gen_episodes(), episode_crowdnav40=gen_crowd_episodes()),
                "numpy": np.__version__, "reference": "/root/reference/pkg/src/vecpomdp @ 0.1.0"}
    with open(os.path.join(HERE, "manifest.json"), "w") as f:
        json.dump(manifest, f, indent=1, sort_keys=True)
    print("wrote golden fixtures to", HERE)
