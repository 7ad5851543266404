"""Small repro of one golden plan case through vp_plan (for compute-sanitizer)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import paper_2510_27191_b200 as vp
from golden_cases import manifest, plan_inputs

name = sys.argv[1] if len(sys.argv) > 1 else "plan_mars4_3"
mode = int(sys.argv[2]) if len(sys.argv) > 2 else 2
prec = sys.argv[3] if len(sys.argv) > 3 else "fp64"
case = manifest()["plans"][name]
p = vp.Planner(prec, exact=(prec == "fp64"))
p.mode = mode
for run in case["runs"]:
    om, belief, cfg, rng = plan_inputs(case, run["seed"])
    out = p.plan(belief, om, cfg, rng, keep_tree=True)
    print(name, mode, out.chosen_action, run["chosen_action"], out.tree_stats, run["tree_stats"])
