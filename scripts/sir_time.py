import sys, time, torch, numpy as np
sys.path.insert(0, "/root/repo")
import paper_2510_27191_b200 as vp
from paper_2510_27191_b200 import _lib
model = vp.MarsModel(11, 11, layout_seed=3)
belief = vp.ParticleBelief.from_model(model, 10_000, vp.RowRng.from_seed(3).derive(3))
db = vp.DeviceBelief.from_host(belief, model)
env = model.sample_initial_states(1, vp.RowRng.from_seed(3).derive(0, 0))
res = model.step_batch(env, np.array([5]), vp.RowRng.from_seed(3).derive(0, 1).bind([0]))
o = int(res.observations[0])
for t in range(3): vp.sir_update(db, model, 5, o, vp.RowRng.from_seed(t))
torch.cuda.synchronize()
_lib.profile_enable(True)
t0 = time.perf_counter()
for t in range(50): vp.sir_update(db, model, 5, o, vp.RowRng.from_seed(t))
torch.cuda.synchronize()
print("sir_update wall ms", (time.perf_counter() - t0) / 50 * 1e3, "device", {k: round(v[0] / 50, 4) for k, v in _lib.profile_read().items() if v[1]})
