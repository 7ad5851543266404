"""Host overhead of the time-budgeted (planning_seconds) path: iterations reached within a wall
budget vs the device time of the same number of iterations run as one fixed-iteration graph.

    python scripts/budget_overhead.py
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2510_27191_b200 as vp  # noqa: E402

model = vp.MarsModel(11, 11, layout_seed=0)
belief = vp.ParticleBelief.from_model(model, 10_000, vp.RowRng.from_seed(0).derive(3))
rows = []
for n in (16384, 65536):
    for budget in (0.005, 0.01, 0.02):
        its, walls = [], []
        for t in range(6):
            cfg = vp.SolverConfig(n_parallel=n, planning_seconds=budget, d_max_cap=90)
            torch.cuda.synchronize()
            w0 = time.perf_counter()
            out = vp.plan(belief, model, cfg, vp.RowRng.from_seed(5).derive(1, t))
            walls.append(time.perf_counter() - w0)
            its.append(out.iterations_run)
        k = sorted(its)[len(its) // 2]
        cfg = vp.SolverConfig(n_parallel=n, iterations=k, d_max_cap=90)
        ms = []
        for t in range(5):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            vp.plan(belief, model, cfg, vp.RowRng.from_seed(5).derive(1, t))
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        rows.append({"n_parallel": n, "budget_s": budget, "iterations": its, "wall_s": [round(w, 5) for w in walls],
                     "fixed_graph_ms_same_iterations": round(sorted(ms)[2], 3)})
print(json.dumps({"workload": "RockSample(11,11) plan() with planning_seconds budgets", "rows": rows}))
