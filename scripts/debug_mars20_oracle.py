import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
import paper_2510_27191_b200 as vp
for n_par, its in ((4096, 6),):
    for s in range(3):
        om = oracle.MarsModel(20, 20, layout_seed=s)
        t0 = time.time()
        r = oracle.run_episode(om, oracle.SolverConfig(n_parallel=n_par, iterations=its), seed=s)
        t1 = time.time()
        d = vp.run_episode(om, vp.SolverConfig(n_parallel=n_par, iterations=its), seed=s, precision="fp64", exact=True)
        print(n_par, its, "seed", s, "oracle", round(r.discounted_return, 3), r.steps, r.counters, round(t1 - t0, 1), "s |",
              "device exact", round(d.discounted_return, 3), d.steps, d.counters, flush=True)
