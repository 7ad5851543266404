"""Run a few planning steps of the bench workload (for ncu / nsight captures)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2510_27191_b200 as vp  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--n", type=int, default=11)
ap.add_argument("--m", type=int, default=11)
ap.add_argument("--n-parallel", type=int, default=16384)
ap.add_argument("--iterations", type=int, default=10)
ap.add_argument("--precision", default="fp32")
ap.add_argument("--problem", default="mars", choices=["mars", "synthetic", "lightdark", "crowdnav"])
a = ap.parse_args()
model = {"mars": lambda: vp.MarsModel(a.n, a.m, layout_seed=1000),
         "synthetic": lambda: vp.SyntheticModel(n_actions=16, n_obs=8, seed=1000),
         "lightdark": vp.LightDarkModel, "crowdnav": vp.CrowdNavModel}[a.problem]()
belief = vp.ParticleBelief.from_model(model, 10_000, vp.RowRng.from_seed(1000).derive(3))
cfg = vp.SolverConfig(n_parallel=a.n_parallel, iterations=a.iterations)
for t in range(a.steps):
    out = vp.plan(belief, model, cfg, vp.RowRng.from_seed(1000).derive(1, t), precision=a.precision)
torch.cuda.synchronize()
print(out.chosen_action, out.tree_stats)
