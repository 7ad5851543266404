"""Host-side cost of one e2e plan() call on the GPU box: wall time per call, the
device time of the same calls, and the host pieces timed one by one (no profiler)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2510_27191_b200 as vp  # noqa: E402
from paper_2510_27191_b200.rng import key_of  # noqa: E402
from paper_2510_27191_b200.solver import get_planner, initial_prefs  # noqa: E402

model = vp.MarsModel(11, 11, layout_seed=1000)
belief = vp.ParticleBelief.from_model(model, 10_000, vp.RowRng.from_seed(1000).derive(3))
cfg = vp.SolverConfig(n_parallel=16384, iterations=10)
N = 200
for t in range(10):
    vp.plan(belief, model, cfg, vp.RowRng.from_seed(1000).derive(1, t))
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
e0.record()
for t in range(N):
    vp.plan(belief, model, cfg, vp.RowRng.from_seed(1000).derive(1, t))
e1.record()
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / N * 1e3
print(f"e2e wall ms per plan {wall:.4f}   events {e0.elapsed_time(e1) / N:.4f}")

p = get_planner()
dm = vp.device_model(model)
rng = vp.RowRng.from_seed(1000).derive(1, 0)


def timeit(name, fn, reps=N):
    fn()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    print(f"{name:<28} {(time.perf_counter() - t0) / reps * 1e6:9.1f} us")


timeit("device_model", lambda: vp.device_model(model))
timeit("initial_prefs", lambda: initial_prefs(model, cfg.eta))
timeit("prepare(device_init=False)", lambda: p.prepare(model, cfg, device_init=False))
timeit("pack", lambda: dm.pack(belief.states))
timeit("cumsum", lambda: np.cumsum(np.asarray(belief.weights, dtype=np.float64)))
timeit("stage_belief", lambda: p.stage_belief(dm, belief))
timeit("key_of", lambda: key_of(rng))
timeit("torch.cuda.is_available", torch.cuda.is_available)
timeit("get_planner", get_planner)
