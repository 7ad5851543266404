"""Closed-loop Navigation episodes: CPU oracle (pinned to the reference) vs the device planner in
fp64 parity mode, same seeds -- shows the returns are the reference algorithm's own."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
import paper_2510_27191_b200 as vp
for s in range(3):
    om = oracle.NavigationModel()
    t0 = time.time()
    r = oracle.run_episode(om, oracle.SolverConfig(n_parallel=2048, iterations=5), seed=s)
    d = vp.run_episode(om, vp.SolverConfig(n_parallel=2048, iterations=5), seed=s, precision="fp64", exact=True)
    print("seed", s, "oracle", round(r.discounted_return, 4), r.steps, r.terminal_reason, round(time.time() - t0, 1),
          "s | device", round(d.discounted_return, 4), d.steps, d.terminal_reason, flush=True)
