"""Time-budget planning (planning_seconds, the iterative host loop) against the fixed-iteration
CUDA-graph step: iterations completed within the budget vs the graph's time for as many."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2510_27191_b200 as vp  # noqa: E402

model = vp.MarsModel(11, 11, layout_seed=1000)
belief = vp.ParticleBelief.from_model(model, 10_000, vp.RowRng.from_seed(1000).derive(3))
for budget in (0.002, 0.005, 0.01, 0.02):
    its = []
    for t in range(6):
        out = vp.plan(belief, model, vp.SolverConfig(n_parallel=16384, planning_seconds=budget),
                      vp.RowRng.from_seed(1000).derive(1, t))
        its.append(out.iterations_run)
    k = int(sorted(its)[len(its) // 2])
    cfg = vp.SolverConfig(n_parallel=16384, iterations=k)
    for t in range(3):
        vp.plan(belief, model, cfg, vp.RowRng.from_seed(1000).derive(1, t))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for t in range(5):
        vp.plan(belief, model, cfg, vp.RowRng.from_seed(1000).derive(1, t))
    fixed_ms = (time.perf_counter() - t0) / 5 * 1e3
    print(f"budget {budget * 1e3:5.1f} ms: iterations {its} (median {k}); fixed-iteration graph for {k}: {fixed_ms:.2f} ms")
