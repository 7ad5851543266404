"""Parity at the configurations the performance claims rest on (BASELINE.json configs[1..2],
SURVEY.md section 8d C2 / C3), against digests of the REAL reference's trees
(tests/golden/make_golden.py ``large``: MARS(11,11) 16 384 x 10 at two plan keys of the bench's
seed, MARS(15,15) 65 536 x 10).

* fp64 parity mode: SHA-256 of every integer column in reference order, the tree size, the
  chosen action, the root PSI row, the first 32 768 PSI row sums and per-depth PSI totals equal
  the reference's (floats within 1e-9).
* fp32 fast mode with identical injected sample streams: structure digests equal, every PSI cell
  within 1e-5 (scale-aware) of the fp64 values.  C2 injects the oracle's streams; C3 injects the
  streams of the fp64 parity plan, whose tree digests equal the reference's.
* the fp32 sampler at a pass that samples more than 65 536 distinct non-fresh beliefs, so the
  dense rows' CDF rows rebuilt by the backups: every draw equals the inverse CDF of
  softmax(eta PSI) of the tree at the start of the pass, up to fp32 CDF-edge flips.
"""

import hashlib

import numpy as np
import pytest

import oracle
import paper_2510_27191_b200 as vp
from golden_cases import load, manifest

pytestmark = pytest.mark.gpu

LARGE = manifest()["large_plans"]
CASES = [(name, i) for name in sorted(LARGE) for i in range(len(LARGE[name]["runs"]))]
INT_COLS = ("parent_action", "parent_obs", "depth", "action_parent_belief", "action_id", "action_visits")


def _inputs(case, run):
    n, m = case["mars"]
    seed, t = run["seed"], run["t"]
    model = vp.MarsModel(n=n, m=m, layout_seed=seed)
    belief = vp.ParticleBelief.from_model(model, case["particles"], vp.RowRng.from_seed(seed).derive(3))
    cfg = vp.SolverConfig(n_parallel=case["n_parallel"], iterations=case["iterations"], eta=case["eta"])
    return model, belief, cfg, vp.RowRng.from_seed(seed).derive(1, t)


def _digests(tab) -> dict:
    out = {k: hashlib.sha256(np.ascontiguousarray(tab[k], dtype="<i8").tobytes()).hexdigest() for k in INT_COLS}
    out["action_reward_sum"] = hashlib.sha256(
        np.ascontiguousarray(tab["action_reward_sum"], dtype="<f8").tobytes()).hexdigest()
    return out


def _check_against_golden(tab, golden, tag, run, rel):
    assert _digests(tab) == run["digests"], tag
    prefs = tab["prefs"]
    root = golden[f"{tag}_prefs_root"]
    assert np.all(np.abs(prefs[0] - root) <= rel * np.maximum(np.abs(root).max(), 1.0))
    rs = prefs.sum(axis=1)
    head = golden[f"{tag}_prefs_row_sum_head"]
    scale = np.maximum(np.abs(prefs[: len(head)]).sum(axis=1), 1.0)
    assert np.all(np.abs(rs[: len(head)] - head) <= rel * scale)
    depth = tab["depth"]
    np.testing.assert_array_equal(np.bincount(depth), golden[f"{tag}_depth_counts"])
    by_depth = np.bincount(depth, weights=rs)
    abs_by_depth = np.bincount(depth, weights=np.abs(prefs).sum(axis=1))
    want_abs = golden[f"{tag}_prefs_abs_sum_by_depth"]
    assert np.all(np.abs(by_depth - golden[f"{tag}_prefs_row_sum_by_depth"]) <= rel * np.maximum(want_abs, 1.0))
    assert np.all(np.abs(abs_by_depth - want_abs) <= rel * np.maximum(want_abs, 1.0))


def _scale_close(got, want, rel):
    scale = np.maximum(np.abs(want), np.abs(want).max(axis=1, keepdims=True))
    return np.all(np.abs(got - want) <= rel * np.maximum(scale, 1.0))


@pytest.mark.parametrize("name,idx", CASES)
def test_fp64_exact_plan_equals_reference_digests(name, idx):
    case = LARGE[name]
    run = case["runs"][idx]
    model, belief, cfg, rng = _inputs(case, run)
    out = vp.plan(belief, model, cfg, rng, precision="fp64", exact=True, keep_tree=True)
    assert out.tree_stats == run["tree_stats"]
    assert out.chosen_action == run["chosen_action"]
    assert out.iterations_run == run["iterations_run"]
    _check_against_golden(out.tree.tables(), load(name), f"s{run['seed']}_t{run['t']}", run, 1e-9)


def test_fp32_injected_streams_c2_oracle():
    """C2, the oracle's own sample streams injected: structure = reference digests; PSI within
    1e-5 of the oracle's fp64 PSI."""
    case = LARGE["large_c2"]
    run = case["runs"][0]
    n, m = case["mars"]
    om = oracle.MarsModel(n=n, m=m, layout_seed=run["seed"])
    belief = oracle.ParticleBelief.from_model(om, case["particles"], oracle.RowRng.from_seed(run["seed"]).derive(3))
    cfg = oracle.SolverConfig(n_parallel=case["n_parallel"], iterations=case["iterations"], eta=case["eta"])
    rng = oracle.RowRng.from_seed(run["seed"]).derive(1, run["t"])
    traces = []
    ref = oracle.plan(belief, om, cfg, rng, traces=traces)
    assert ref.tree_stats == run["tree_stats"] and ref.chosen_action == run["chosen_action"]
    inject = [np.stack([lv["actions"] for lv in it["levels"]]) for it in traces]
    out = vp.plan(belief, om, cfg, rng, precision="fp32", inject_actions=inject, keep_tree=True)
    tab = out.tree.tables()
    _check_against_golden(tab, load("large_c2"), f"s{run['seed']}_t{run['t']}", run, 1e-5)
    assert _scale_close(tab["prefs"], ref.tree.prefs, 1e-5)


def test_fp32_injected_streams_c3_chain():
    """C3: the fp64 parity plan's streams (its tree digests equal the reference's) injected into
    the fp32 fast path: identical structure, PSI within 1e-5 of the fp64 PSI."""
    case = LARGE["large_c3"]
    run = case["runs"][0]
    model, belief, cfg, rng = _inputs(case, run)
    exact = vp.plan(belief, model, cfg, rng, precision="fp64", exact=True, keep_tree=True, trace=True)
    want = exact.tree.tables()
    assert _digests(want) == run["digests"]
    inject = [np.stack([lv["actions"] for lv in it["levels"]]) for it in exact.traces]
    del exact
    out = vp.plan(belief, model, cfg, rng, precision="fp32", inject_actions=inject, keep_tree=True)
    got = out.tree.tables()
    assert _digests(got) == run["digests"]
    assert _scale_close(got["prefs"], want["prefs"], 1e-5)


@pytest.mark.parametrize("kind,n,k", [("synthetic", 131072, 12), ("mars11_11", 16384, 10)])
def test_fp32_sampler_at_scale(kind, n, k):
    """fp32 draws at scale: Synthetic at 131 072 rows x 12 iterations samples ~95k distinct
    existing beliefs in its last pass (overlay records and dense rows, whose CDF rows the
    previous backup rebuilt); MARS(11,11) at the C2 workload.  Every draw is the inverse CDF of
    softmax(eta PSI) of the tree at the start of the pass, except fp32 CDF-edge flips."""
    model = vp.SyntheticModel(n_actions=16, n_obs=8, seed=3) if kind == "synthetic" else vp.MarsModel(11, 11,
                                                                                                      layout_seed=3)
    belief = vp.ParticleBelief.from_model(model, 10_000, vp.RowRng.from_seed(3).derive(3))
    rng = vp.RowRng.from_seed(3).derive(1, 0)
    before = vp.Planner("fp32").plan(belief, model, vp.SolverConfig(n_parallel=n, iterations=k - 1), rng,
                                     keep_tree=True).tree.tables()
    out = vp.Planner("fp32").plan(belief, model, vp.SolverConfig(n_parallel=n, iterations=k), rng,
                                  keep_tree=True, trace=True)
    prefs = before["prefs"]
    nb, A = prefs.shape
    search_rng = rng.derive(k - 1).derive(1)
    rows = np.arange(n)
    ids = np.zeros(n, dtype=np.int64)
    distinct_known = set()
    mism = total = 0
    for lvl, tr in enumerate(out.traces[-1]["levels"]):
        u = search_rng.derive(lvl).derive(0).uniform(rows)
        known = ids < nb
        distinct_known.update(np.unique(ids[known]).tolist())
        # rows at beliefs created in this pass draw from the initial row (all zeros for these models)
        rowp = np.where(known[:, None], prefs[np.minimum(ids, nb - 1)], 0.0)
        cum = np.cumsum(oracle.softmax_rows(rowp, 2.0), axis=1)
        want = np.minimum((cum <= u[:, None]).sum(axis=1), A - 1)
        bad = np.flatnonzero(tr["actions"] != want)
        if len(bad):
            edge = np.min(np.abs(cum[bad] - u[bad, None]), axis=1)
            assert np.all(edge < 2e-5), (lvl, bad[:5], edge.max())
        mism += len(bad)
        total += n
        ids = tr["next_beliefs"]
    if kind == "synthetic":
        assert len(distinct_known) > 65536, len(distinct_known)
    assert mism <= max(3, 1e-3 * total), (mism, total)
