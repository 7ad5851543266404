"""Closed-loop CrowdNav on the device planner: wall time per environment step, split into the
planning step and the rest (env step + SIR + hooks)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_27191_b200 as vp  # noqa: E402

model = vp.CrowdNavModel(max_steps=int(sys.argv[1]) if len(sys.argv) > 1 else 20)
cfg = vp.SolverConfig(n_parallel=8192, iterations=10, particles=2000)
vp.run_episode(vp.CrowdNavModel(max_steps=2), cfg, seed=1)  # warm-up (graphs, tables)
t0 = time.perf_counter()
rec = vp.run_episode(model, cfg, seed=0)
wall = time.perf_counter() - t0
plan = sum(rec.plan_wall_times)
print(f"steps {rec.steps}  reason {rec.terminal_reason}  return {rec.discounted_return:.2f}  "
      f"wall/step {wall / rec.steps * 1e3:.2f} ms  plan/step {plan / rec.steps * 1e3:.2f} ms  "
      f"other/step {(wall - plan) / rec.steps * 1e3:.2f} ms  counters {rec.counters}")
