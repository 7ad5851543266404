"""Host-side cost of one e2e plan() call (pack, keys, launch, sync) on the GPU box."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2510_27191_b200 as vp
model = vp.MarsModel(11, 11, layout_seed=1000)
belief = vp.ParticleBelief.from_model(model, 10_000, vp.RowRng.from_seed(1000).derive(3))
cfg = vp.SolverConfig(n_parallel=16384, iterations=10)
for t in range(5):
    vp.plan(belief, model, cfg, vp.RowRng.from_seed(1000).derive(1, t))
torch.cuda.synchronize()
t0 = time.perf_counter()
for t in range(20):
    vp.plan(belief, model, cfg, vp.RowRng.from_seed(1000).derive(1, t))
print("e2e ms per plan", (time.perf_counter() - t0) / 20 * 1e3)
pr = cProfile.Profile(); pr.enable()
for t in range(20):
    vp.plan(belief, model, cfg, vp.RowRng.from_seed(1000).derive(1, t))
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
