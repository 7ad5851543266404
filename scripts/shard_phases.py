"""Per-phase device time of the sharded planning step, run as virtual ranks on one GPU.

    python scripts/shard_phases.py [--world 8] [--rows-per-gpu 16384] [--iterations 10] [--problem mars|crowdnav]

On G GPUs the trajectory phase runs concurrently (each GPU its own block of rows), so
the projected per-GPU step time is trajectory / G + exchange + insert + backup, with
the exchange an NCCL all-gather of (2 d + 1) x 8 B per row (measured here as the
in-process concatenation only).
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2510_27191_b200 as vp  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--world", type=int, default=8)
ap.add_argument("--rows-per-gpu", type=int, default=16384)
ap.add_argument("--iterations", type=int, default=10)
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--problem", default="mars", choices=["mars", "crowdnav"])
ap.add_argument("--particles", type=int, default=10_000)
ap.add_argument("--board", type=int, default=11, help="MARS board size (11: C2, 15: C3)")
a = ap.parse_args()
model = vp.MarsModel(a.board, a.board, layout_seed=1000) if a.problem == "mars" else vp.CrowdNavModel()
belief = vp.ParticleBelief.from_model(model, a.particles, vp.RowRng.from_seed(1000).derive(3))


def fused_ms(rows):
    """Device time of the single-GPU fused step (belief resident, one graph replay per step)."""
    from paper_2510_27191_b200.rng import key_of

    cfg = vp.SolverConfig(n_parallel=rows, iterations=a.iterations)
    pl = vp.Planner("fp32")
    particles, cumw, m = pl.upload_belief(vp.device_model(model), belief)
    keys = [key_of(vp.RowRng.from_seed(1000).derive(1, t)) for t in range(a.steps + 1)]

    def step(t):
        d, tree, work = pl.prepare(model, cfg, device_init=False)
        pl.run_fixed(d, tree, work, m, model.spec, cfg, keys[t], from_host=False)

    step(0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for t in range(a.steps):
        step(t + 1)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / a.steps

out = {}
for world in sorted({1, a.world}):
    cfg = vp.SolverConfig(n_parallel=a.rows_per_gpu * a.world, iterations=a.iterations)
    p = vp.ShardedPlanner(world=world, precision="fp32")
    p.plan(belief, model, cfg, vp.RowRng.from_seed(1000).derive(1, 0))
    p.phase_ms = {}
    for t in range(a.steps):
        p.plan(belief, model, cfg, vp.RowRng.from_seed(1000).derive(1, t + 1))
    torch.cuda.synchronize()
    out[world] = {k: v / a.steps for k, v in p.phase_ms.items()}
ph = out[a.world]
proj = ph["trajectory"] / a.world + ph["insert"] + ph["backup"]
one = fused_ms(a.rows_per_gpu)
res = {"problem": a.problem, "rows_total": a.rows_per_gpu * a.world, "world": a.world, "ms_per_step_by_phase": out,
       "projected_ms_per_step_per_gpu_excl_nccl": proj, "fused_1gpu_ms_per_step": one,
       "projected_weak_scaling_speedup_excl_nccl": a.world * one / proj,
       "bytes_all_gathered_per_step": sum((2 * min(i + 1, 90) + 1) * 8 * a.rows_per_gpu * a.world
                                          for i in range(a.iterations))}
print(json.dumps(res))
