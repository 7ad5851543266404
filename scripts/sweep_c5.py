"""BASELINE config 5: synthetic scaling sweep (simulations per iteration x tree depth) on one B200,
one bench.py line per point; the CPU reference rate is measured once per depth on a bounded sample.

    python scripts/sweep_c5.py [--out profiles/r01_c5_sweep.json]
"""
import argparse
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ap = argparse.ArgumentParser()
ap.add_argument("--rows", default="1024,4096,16384,65536,262144,1048576")
ap.add_argument("--depths", default="10,20,50")
ap.add_argument("--max-nodes", type=float, default=6e8, help="skip points whose worst-case tree exceeds this")
ap.add_argument("--out", default=None)
a = ap.parse_args()
points = []
for d in [int(x) for x in a.depths.split(",")]:
    cpu_done = False
    for n in [int(x) for x in a.rows.split(",")]:
        nodes = n * d * (d + 1) / 2
        if nodes > a.max_nodes:
            points.append({"n_parallel": n, "iterations": d, "skipped": f"worst-case tree {nodes:.2e} nodes"})
            continue
        cmd = [sys.executable, os.path.join(REPO, "bench.py"), "--config", "c5", "--n-parallel", str(n),
               "--iterations", str(d), "--steps", "3", "--warmup", "2", "--episodes", "0", "--cpu-budget-s", "5"]
        if cpu_done:
            cmd.append("--no-cpu-baseline")
        out = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
        try:
            line = json.loads(out.stdout.strip().splitlines()[-1])
        except (IndexError, json.JSONDecodeError):
            points.append({"n_parallel": n, "iterations": d, "error": out.stderr[-400:]})
            continue
        cpu_done = cpu_done or "cpu_baseline" in line
        pt = {"n_parallel": n, "iterations": d, "sims_per_s": line["value"], "e2e_sims_per_s": line["e2e"]["value"],
              "ms_per_step": line["ms_per_step"], "episode_steps_per_s": line["episode_steps_per_s"],
              "tree_stats": line["tree_stats"],
              "roofline": {k: (v["achieved"], v["frac"]) for k, v in line["roofline_other"].items() if v}}
        if "cpu_baseline" in line:
            pt["cpu_baseline"] = line["cpu_baseline"]
        points.append(pt)
        print(json.dumps(pt), flush=True)
res = {"config": "c5 synthetic sweep (|A|=16, |O|=8), 1 B200", "points": points}
if a.out:
    json.dump(res, open(a.out, "w"), indent=1)
