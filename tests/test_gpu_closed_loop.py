"""Closed-loop parity: plan -> env step -> SIR.

* fp64 parity mode reproduces the reference's episodes exactly (same plans,
  hence the same executed actions, observations, SIR updates and returns);
  the environment and the SIR propagation step through the DEVICE model.
* fp32 fast mode: mean discounted return over a 30-episode campaign is
  statistically indistinguishable from the reference's (two-sample z test at
  the 99 % level, and the means' 95 % CIs overlap).
"""

import json

import numpy as np
import pytest

import paper_2510_27191_b200 as vp
from golden_cases import manifest

pytestmark = pytest.mark.gpu


def test_fp64_exact_episodes_equal_reference():
    recs = manifest()["episodes"]["episode_mars4_3"]
    cfg = vp.SolverConfig(n_parallel=64, iterations=4, particles=500)
    for r in recs:
        got = vp.run_episode(vp.MarsModel(n=4, m=3, layout_seed=r["seed"]), cfg, seed=r["seed"], precision="fp64",
                             exact=True)
        assert got.steps == r["steps"] and got.terminal_reason == r["reason"]
        assert got.degenerate_updates == r["degenerate"]
        assert abs(got.discounted_return - r["return"]) < 1e-9


def test_fp64_exact_crowdnav_episodes_equal_reference():
    """CrowdNav closed loop: device planner, device env step and host SIR behind the
    model's refresh / reconcile hooks reproduce the reference's episodes."""
    cfg = vp.SolverConfig(n_parallel=128, iterations=4, particles=300)
    for r in manifest()["episodes"]["episode_crowdnav40"]:
        model = vp.CrowdNavModel(n_people=40, hall_depth=8.0, max_steps=15)
        got = vp.run_episode(model, cfg, seed=r["seed"], precision="fp64", exact=True)
        assert (got.steps, got.terminal_reason, got.degenerate_updates) == (r["steps"], r["reason"], r["degenerate"])
        assert abs(got.discounted_return - r["return"]) < 1e-9
        assert got.counters == pytest.approx(r["counters"])


@pytest.mark.parametrize("seed", [0, 1])
def test_crowdnav_device_belief_equals_host_belief(seed):
    """Device-resident CrowdNav loop (device SIR + reconcile_device broadcast) equals the host
    belief loop (host SIR + numpy reconcile_belief) step for step."""
    model = vp.CrowdNavModel(n_people=40, hall_depth=8.0, max_steps=12)
    cfg = vp.SolverConfig(n_parallel=256, iterations=4, particles=300)
    a = vp.run_episode(model, cfg, seed=seed, precision="fp64", device_belief=True)
    b = vp.run_episode(model, cfg, seed=seed, precision="fp64", device_belief=False)
    assert (a.steps, a.terminal_reason, a.degenerate_updates) == (b.steps, b.terminal_reason, b.degenerate_updates)
    assert a.discounted_return == pytest.approx(b.discounted_return, abs=1e-12)
    assert a.counters == pytest.approx(b.counters)


def test_fp32_campaign_returns_match_reference():
    recs = manifest()["episodes"]["episode_mars5_4_campaign"]
    cfg = vp.SolverConfig(n_parallel=256, iterations=5, particles=1000)
    model = vp.MarsModel(n=5, m=4, layout_seed=7)
    ref = np.array([r["return"] for r in recs])
    dev = np.array([vp.run_episode(model, cfg, seed=r["seed"], precision="fp32").discounted_return for r in recs])
    se = np.sqrt(ref.var(ddof=1) / len(ref) + dev.var(ddof=1) / len(dev))
    z = abs(dev.mean() - ref.mean()) / se
    assert z < 2.58, (dev.mean(), ref.mean(), se)
    half_ref = 1.96 * ref.std(ddof=1) / np.sqrt(len(ref))
    half_dev = 1.96 * dev.std(ddof=1) / np.sqrt(len(dev))
    assert abs(dev.mean() - ref.mean()) <= half_ref + half_dev


def test_time_budget_mode_runs_at_least_one_iteration():
    """planning_seconds budget (solver.py:106-110): the first iteration always
    completes; d_max grows by one per completed iteration."""
    model = vp.MarsModel(n=7, m=8, layout_seed=0)
    belief = vp.ParticleBelief.from_model(model, 1000, vp.RowRng.from_seed(0).derive(3))
    out = vp.plan(belief, model, vp.SolverConfig(n_parallel=1024, planning_seconds=1e-6), vp.RowRng.from_seed(0))
    assert out.iterations_run == 1 and out.final_d_max == 1
    out = vp.plan(belief, model, vp.SolverConfig(n_parallel=1024, planning_seconds=0.05, d_max_cap=6),
                  vp.RowRng.from_seed(0))
    assert out.iterations_run >= 2
    assert out.final_d_max == min(out.iterations_run, 6)
    assert 0 <= out.chosen_action < model.spec.action_count


def test_campaign_jsonl_on_device(tmp_path):
    """paper_2510_27191_b200.campaign: config header, one record per run, summary (bench.py:128-146)."""
    from paper_2510_27191_b200.campaign import CampaignConfig, run_campaign

    out = tmp_path / "c.jsonl"
    cfg = CampaignConfig(problem="tiger", solver=vp.SolverConfig(n_parallel=1024, iterations=4, particles=500),
                         runs=3, out_path=str(out))
    records, summary = run_campaign(cfg)
    lines = [json.loads(x) for x in out.read_text().splitlines()]
    assert [x["type"] for x in lines] == ["config", "run", "run", "run", "summary"]
    assert [r["run_index"] for r in records] == [0, 1, 2]
    assert summary["n"] == 3 and "discounted_return" in summary["metrics"]
