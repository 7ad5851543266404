"""Plug-in models plan at built-in speed: the tabular CudaModel plug-in (a user's CUDA
source compiled into a plug-in build) against the built-in Tabular model on Tiger, and
Philox against SplitMix64 streams, same workload, belief resident (one vp_plan graph
replay per planning step, CUDA events on the launching stream).  One JSON line
(profiles/r02_plugin_speed.json).

    python scripts/plugin_speed.py --n-parallel 16384 --iterations 10
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2510_27191_b200 as vp  # noqa: E402
from paper_2510_27191_b200.envs.plugin_examples import corridor_cuda_model, tabular_cuda_model  # noqa: E402
from paper_2510_27191_b200.rng import key_of, kind_of  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n-parallel", type=int, default=16384)
ap.add_argument("--iterations", type=int, default=10)
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--warmup", type=int, default=3)
a = ap.parse_args()


def time_plan(model, rng_cls, label):
    belief = vp.ParticleBelief.from_model(model, 2000, vp.RowRng.from_seed(7).derive(3))
    cfg = vp.SolverConfig(n_parallel=a.n_parallel, iterations=a.iterations)
    planner = vp.Planner("fp32")
    dm = vp.device_model(model)
    particles, cumw, m = planner.upload_belief(dm, belief)
    rngs = [rng_cls.from_seed(7).derive(1, t) for t in range(a.warmup + a.steps)]
    st = torch.cuda.current_stream()
    ms = []
    for t, r in enumerate(rngs):
        d, tree, work = planner.prepare(model, cfg, device_init=False)
        d.desc.rng_kind = kind_of(r)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(st)
        out = planner.run_fixed(d, tree, work, m, model.spec, cfg, key_of(r), from_host=False)
        e1.record(st)
        torch.cuda.synchronize()
        if t >= a.warmup:
            ms.append(e0.elapsed_time(e1))
    ms.sort()
    return {"model": label, "rng": rng_cls.__name__, "ms_per_step_median": round(ms[len(ms) // 2], 4),
            "ms_per_step_min": round(ms[0], 4), "tree_stats": out.tree_stats,
            "sims_per_s": round(a.n_parallel * a.iterations / (ms[len(ms) // 2] * 1e-3), 1)}


rows = [time_plan(vp.tiger_model(), vp.RowRng, "Tiger (built-in TabularModel)"),
        time_plan(tabular_cuda_model(vp.tiger_model().pomdp), vp.RowRng, "Tiger (CudaModel plug-in)"),
        time_plan(vp.tiger_model(), vp.PhiloxRowRng, "Tiger (built-in TabularModel)"),
        time_plan(vp.MarsModel(11, 11, layout_seed=0), vp.RowRng, "RockSample(11,11)"),
        time_plan(vp.MarsModel(11, 11, layout_seed=0), vp.PhiloxRowRng, "RockSample(11,11)"),
        time_plan(corridor_cuda_model(), vp.RowRng, "corridor (plug-in only)"),
        time_plan(corridor_cuda_model(), vp.PhiloxRowRng, "corridor (plug-in only)")]
print(json.dumps({"workload": f"plan(), n_parallel={a.n_parallel}, iterations={a.iterations}, fp32, belief resident",
                  "device": torch.cuda.get_device_name(0), "rows": rows}))
