"""Time the CrowdNav planning step (reference bench.py default: 8192 rows, 300 people)
on the device -- belief resident (one vp_plan graph replay) and end to end through
vp.plan -- with the per-kernel-kind split, beside the oracle port of the reference
on the host for the same plan.  One JSON line (profiles/r01_crowdnav_step.json).

    python scripts/crowdnav_step.py --n-parallel 8192 --iterations 10 --cpu
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2510_27191_b200 as vp  # noqa: E402
from paper_2510_27191_b200 import _lib  # noqa: E402
from paper_2510_27191_b200.rng import key_of  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n-parallel", type=int, default=8192)
ap.add_argument("--iterations", type=int, default=10)
ap.add_argument("--people", type=int, default=300)
ap.add_argument("--particles", type=int, default=2000)
ap.add_argument("--steps", type=int, default=5)
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--precision", default="fp32")
ap.add_argument("--rng", default="splitmix64", choices=["splitmix64", "philox"])
ap.add_argument("--cpu", action="store_true", help="also time the oracle port on the host (one plan)")
a = ap.parse_args()

model = vp.CrowdNavModel(n_people=a.people)
belief = vp.ParticleBelief.from_model(model, a.particles, vp.RowRng.from_seed(1000).derive(3))
cfg = vp.SolverConfig(n_parallel=a.n_parallel, iterations=a.iterations)
planner = vp.Planner(a.precision)
dm = vp.device_model(model)
particles, cumw, m = planner.upload_belief(dm, belief)
rng_cls = vp.PhiloxRowRng if a.rng == "philox" else vp.RowRng
rngs = [rng_cls.from_seed(1000).derive(1, t) for t in range(a.warmup + a.steps)]


def step(t):
    d, tree, work = planner.prepare(model, cfg, device_init=False)
    d.desc.rng_kind = 1 if a.rng == "philox" else 0
    return planner.run_fixed(d, tree, work, m, model.spec, cfg, key_of(rngs[t]), from_host=False)


def timed(fn):
    for t in range(a.warmup):
        fn(t)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for t in range(a.steps):
        out = fn(a.warmup + t)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / a.steps, out


ms, out = timed(step)
e2e_ms, out_e2e = timed(lambda t: vp.plan(belief, model, cfg, rngs[t], precision=a.precision))
_lib.profile_enable(True)
for t in range(2):
    step(a.warmup + t)
torch.cuda.synchronize()
prof = _lib.profile_read()
_lib.profile_enable(False)
sims = a.n_parallel * a.iterations
res = {"workload": f"crowdnav {a.people} people, {a.n_parallel} rows x {a.iterations} iterations, "
                   f"{a.particles} particles, {a.precision}, {a.rng} streams",
       "state_bytes": dm.state_bytes, "ms_per_step": ms, "sims_per_s": sims / (ms / 1e3),
       "e2e_ms_per_step": e2e_ms, "e2e_sims_per_s": sims / (e2e_ms / 1e3),
       "kernel_ms_per_step": {k: v[0] / 2 for k, v in prof.items() if v[1]},
       "tree_stats": out_e2e.tree_stats, "chosen_action": out_e2e.chosen_action}
if a.cpu:
    import oracle

    om = oracle.CrowdNavModel(n_people=a.people)
    ob = oracle.ParticleBelief.from_model(om, a.particles, oracle.RowRng.from_seed(1000).derive(3))
    t0 = time.perf_counter()
    ref = oracle.plan(ob, om, oracle.SolverConfig(n_parallel=a.n_parallel, iterations=a.iterations),
                      oracle.RowRng.from_seed(1000).derive(1, 0))
    cpu_s = time.perf_counter() - t0
    res["cpu_port"] = {"seconds_per_step": cpu_s, "sims_per_s": sims / cpu_s, "cores": 1,
                       "tree_stats": ref.tree_stats}
print(json.dumps(res))
os.makedirs("gpurun_out", exist_ok=True)
with open("gpurun_out/crowdnav_step.json", "w") as f:
    f.write(json.dumps(res) + "\n")
