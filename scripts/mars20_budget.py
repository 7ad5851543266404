"""MARS(20,20) at the paper's planning budgets on one B200 (60 000 rows, fp32): iterations
completed, tree size and whether deepening stopped on the memory bound, per planning step.

    python scripts/mars20_budget.py --budgets 0.1,1.0 --steps 3 > profiles/r02_mars20_budget.json
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2510_27191_b200 as vp  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--budgets", default="0.01,0.05,0.1,1.0")
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--n-parallel", type=int, default=60_000)
a = ap.parse_args()
model = vp.MarsModel(20, 20, layout_seed=1000)
belief = vp.ParticleBelief.from_model(model, 10_000, vp.RowRng.from_seed(1000).derive(3))
planner = vp.Planner("fp32")
out = {"problem": "MARS(20,20)", "actions": model.spec.action_count, "n_parallel": a.n_parallel, "budgets": []}
for b in (float(x) for x in a.budgets.split(",")):
    cfg = vp.SolverConfig(n_parallel=a.n_parallel, planning_seconds=b)
    rows = []
    for t in range(a.steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        o = planner.plan(belief, model, cfg, vp.RowRng.from_seed(1000).derive(1, t))
        torch.cuda.synchronize()
        rows.append({"wall_s": round(time.perf_counter() - t0, 4), "iterations": o.iterations_run,
                     "d_max": o.final_d_max,
                     "tree_stats": o.tree_stats, "chosen_action": o.chosen_action})
    free, total = torch.cuda.mem_get_info()
    out["budgets"].append({"planning_seconds": b, "steps": rows,
                           "stopped_on_memory": any(r["tree_stats"].get("stopped") == "memory" for r in rows),
                           "hbm_used_gb": round((total - free) / 1e9, 1)})
print(json.dumps(out))
