import cProfile, pstats, sys, time
sys.path.insert(0, "/root/repo")
import torch
import paper_2510_27191_b200 as vp
model = vp.MarsModel(11, 11, layout_seed=1000)
belief = vp.ParticleBelief.from_model(model, 10_000, vp.RowRng.from_seed(1000).derive(3))
cfg = vp.SolverConfig(n_parallel=16384, iterations=10)
rngs = [vp.RowRng.from_seed(1000).derive(1, t) for t in range(400)]
for t in range(20):
    vp.plan(belief, model, cfg, rngs[t])
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for t in range(20, 220):
    vp.plan(belief, model, cfg, rngs[t])
pr.disable()
st = pstats.Stats(pr); st.sort_stats("tottime").print_stats(18)
