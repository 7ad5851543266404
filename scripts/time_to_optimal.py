"""Time-to-near-optimal return (the second half of BASELINE.json's metric) on the GPU planner.

Closed-loop campaigns with a wall-clock budget per planning step, reported as mean +- 95% CI per
budget plus the smallest budget whose mean lies inside the CI of the best mean observed (SURVEY
section 8d, C2 sweep: RockSample(11,11) = MARS(11,11), n_parallel 16 384).

The paper's MARS(20,20) numbers are printed beside MARS(20,20) runs for
context only: the shipped reference scores far lower on MARS(20,20) at these budgets (its episodes
mostly truncate at 90 steps), and the device planner reproduces the reference, not the paper's
unshipped implementation (scripts/debug_mars20_oracle.py).

    python scripts/time_to_optimal.py [--n 11 --m 11 --n-parallel 16384] [--runs 30] [--budgets ...]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2510_27191_b200 import SolverConfig  # noqa: E402
from paper_2510_27191_b200.campaign import CampaignConfig, run_campaign  # noqa: E402

PAPER = {0.01: (31.1, 2.6), 0.05: (50.0, 1.9), 0.1: (53.3, 2.1), 1.0: (58.8, 2.1)}

ap = argparse.ArgumentParser()
ap.add_argument("--runs", type=int, default=30)
ap.add_argument("--budgets", default="0.001,0.003,0.01,0.03,0.1")
ap.add_argument("--n", type=int, default=11)
ap.add_argument("--m", type=int, default=11)
ap.add_argument("--n-parallel", type=int, default=16_384)
ap.add_argument("--problem", default="mars", choices=["mars", "navigation", "tiger", "lightdark"])
ap.add_argument("--out", default=None)
ap.add_argument("--cpu-runs", type=int, default=0,
                help="also run the CPU reference algorithm (oracle/ port) at its smallest budget")
a = ap.parse_args()
rows = []
for b in [float(x) for x in a.budgets.split(",")]:
    cfg = CampaignConfig(problem=a.problem, problem_params={"n": a.n, "m": a.m} if a.problem == "mars" else {},
                         solver=SolverConfig(n_parallel=a.n_parallel, planning_seconds=b), runs=a.runs)
    t0 = time.perf_counter()
    recs, summ = run_campaign(cfg)
    st = summ["metrics"]["discounted_return"]
    row = {"planning_seconds": b, "runs": a.runs, "mean_return": round(st["mean"], 3), "ci95": round(st["ci95"], 3),
           "mean_steps": round(summ["metrics"]["steps"]["mean"], 2),
           "mean_plan_seconds": round(summ["metrics"]["plan_seconds"]["mean"], 5),
           "campaign_wall_s": round(time.perf_counter() - t0, 1)}
    if b in PAPER and (a.n, a.m) == (20, 20) and a.problem == "mars":
        row["paper_laptop_gpu"] = {"mean_return": PAPER[b][0], "ci95": PAPER[b][1]}
    rows.append(row)
    print(json.dumps(row), flush=True)
best = max(rows, key=lambda r: r["mean_return"])
near = min((r for r in rows if r["mean_return"] >= best["mean_return"] - best["ci95"]),
           key=lambda r: r["planning_seconds"])
res = {"problem": f"MARS({a.n},{a.m})" if a.problem == "mars" else a.problem, "n_parallel": a.n_parallel, "eta": 2.0, "budgets": rows,
       "time_to_near_optimal_s": near["planning_seconds"],
       "definition": "smallest planning_seconds whose mean return lies within the 95% CI of the best mean (SURVEY 8d)",
       "runs_per_budget": a.runs}
if a.cpu_runs and a.problem == "mars":
    # the reference always completes its first iteration (solver.py:106-110), so on the CPU the
    # smallest achievable planning step is one iteration of n_parallel rows
    import oracle  # CPU baseline only

    t0 = time.perf_counter()
    recs = []
    for i in range(a.cpu_runs):
        model = oracle.MarsModel(n=a.n, m=a.m, layout_seed=i)
        recs.append(oracle.run_episode(model, oracle.SolverConfig(n_parallel=a.n_parallel, planning_seconds=1e-6),
                                       seed=i))
    rets = [r.discounted_return for r in recs]
    import numpy as np

    res["cpu_reference_min_budget"] = {
        "runs": a.cpu_runs, "mean_return": round(float(np.mean(rets)), 3),
        "ci95": round(float(1.96 * np.std(rets, ddof=1) / np.sqrt(len(rets))), 3) if len(rets) > 1 else 0.0,
        "mean_plan_seconds": round(float(np.mean([np.mean(r.plan_wall_times) for r in recs])), 4),
        "cores": 1, "kind": "port (oracle/, numpy restatement of vecpomdp.plan)",
        "wall_s": round(time.perf_counter() - t0, 1)}
print(json.dumps(res))
if a.out:
    json.dump(res, open(a.out, "w"), indent=1)
