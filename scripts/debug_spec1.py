"""Find and print the first SPEC #1 random tree where the fp32 device backup departs from the serial oracle."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from oracle import acceptance as acc
import test_gpu_acceptance as T

for prec in ("fp32", "fp64"):
    for k in range(200):
        A, passes = acc.random_tree_case(np.random.default_rng(k))
        serial = acc.serial_run(A, passes, 2.0, 0.9)
        tree = T.device_run(A, passes, 2.0, 0.9, prec, False)
        t = tree.tables()
        paths = acc.belief_paths(t["parent_action"], t["parent_obs"], t["action_parent_belief"], t["action_id"])
        bad = []
        for i, p in enumerate(paths):
            want = np.array(serial.prefs[p])
            err = np.abs(t["prefs"][i] - want).max() / max(1.0, np.abs(want).max())
            if err > 1e-5:
                bad.append((i, p, t["prefs"][i], want))
        if bad:
            print(prec, "case", k, "A", A, "passes", [(p["d"], p["actions"].shape[1]) for p in passes])
            for p in passes:
                print(" d", p["d"], "actions", p["actions"].tolist(), "obs", p["observations"].tolist(),
                      "rew", p["rewards"].tolist(), "leaf", p["leaf"].tolist())
            for b in bad[:6]:
                print("  belief", b[0], "path", b[1], "dev", b[2], "want", b[3])
            print("  lse", tree.b_lse[: len(paths)].cpu().numpy(), "flags", tree.b_flags[: len(paths)].cpu().numpy())
            break
    else:
        print(prec, "all ok")
