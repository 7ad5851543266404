"""Determinism check: the same fp64 / fp32 fast-mode plan twice must give identical trees."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2510_27191_b200 as vp

for prec in ("fp64", "fp32"):
    model = vp.CrowdNavModel(n_people=40, hall_depth=8.0, max_steps=12)
    belief = vp.ParticleBelief.from_model(model, 300, vp.RowRng.from_seed(1).derive(3))
    cfg = vp.SolverConfig(n_parallel=256, iterations=4, particles=300)
    outs = []
    for rep in range(4):
        o = vp.plan(belief, model, cfg, vp.RowRng.from_seed(1).derive(1, 0), precision=prec, keep_tree=True)
        outs.append((o.chosen_action, o.tree_stats, o.tree.tables()))
    for rep in range(1, 4):
        a, b = outs[0], outs[rep]
        same_int = all(np.array_equal(a[2][k], b[2][k]) for k in ("parent_action", "parent_obs", "action_id", "action_visits"))
        dp = np.abs(a[2]["prefs"] - b[2]["prefs"]).max() if a[2]["prefs"].shape == b[2]["prefs"].shape else -1
        print(prec, "rep", rep, "action", a[0], b[0], a[1], b[1], "ints equal", same_int, "max dprefs", dp)
    for seed in (0, 1):
        r1 = vp.run_episode(model, cfg, seed=seed, precision=prec, device_belief=True)
        r2 = vp.run_episode(model, cfg, seed=seed, precision=prec, device_belief=True)
        r3 = vp.run_episode(model, cfg, seed=seed, precision=prec, device_belief=False)
        print(prec, "episode seed", seed, r1.discounted_return, r2.discounted_return, r3.discounted_return, r1.steps, r2.steps, r3.steps)
