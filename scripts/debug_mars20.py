import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
import paper_2510_27191_b200 as vp
om = oracle.MarsModel(20, 20, layout_seed=0)
pm = vp.MarsModel(20, 20, layout_seed=0)
belief = oracle.ParticleBelief.from_model(om, 10000, oracle.RowRng.from_seed(0).derive(3))
rng = oracle.RowRng.from_seed(0).derive(1, 0)
for it in (2, 4):
    cfg = oracle.SolverConfig(n_parallel=2048, iterations=it)
    ref = oracle.plan(belief, om, cfg, rng)
    dev = vp.plan(belief, om, cfg, rng, precision="fp64", exact=True, keep_tree=True)
    print("it", it, "ref", ref.chosen_action, ref.tree.stats(), "dev", dev.chosen_action, dev.tree_stats, flush=True)
    t = dev.tree.tables()
    print("  root psi max/min", t["prefs"][0].max(), t["prefs"][0].min(), "ref", ref.tree.prefs[0].max(), ref.tree.prefs[0].min())
for budget in (0.01, 0.05):
    cfg = vp.SolverConfig(n_parallel=60000, planning_seconds=budget)
    t0 = time.time()
    out = vp.plan(belief, pm, cfg, rng)
    print("budget", budget, "iters", out.iterations_run, "dmax", out.final_d_max, out.tree_stats, "act", out.chosen_action, round(time.time()-t0, 3), flush=True)
    db = vp.DeviceBelief.from_host(belief, pm)
    out = vp.plan(db, pm, cfg, rng)
    print("  device belief: iters", out.iterations_run, out.tree_stats, "act", out.chosen_action, flush=True)
cfg = vp.SolverConfig(n_parallel=60000, iterations=8)
for s in range(2):
    r = vp.run_episode(pm, cfg, seed=s)
    print("episode fixed-8", s, r.discounted_return, r.steps, r.terminal_reason, r.counters, flush=True)
cfg = vp.SolverConfig(n_parallel=60000, planning_seconds=0.05)
for s in range(2):
    r = vp.run_episode(pm, cfg, seed=s)
    print("episode 0.05s", s, r.discounted_return, r.steps, r.terminal_reason, r.counters, np.mean(r.plan_wall_times), flush=True)
