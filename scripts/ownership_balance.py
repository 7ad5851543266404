"""How evenly would subtree ownership split a planning step over G GPUs?

Runs one traced planning step and, for every pass and cut depth k, routes each row that reaches
depth k to the owner of its depth-k belief (hash of the belief id mod G).  Reports, per k:
  * rows_top:    row-levels above the cut (replicated on every rank),
  * imbalance:   max over ranks / mean of the row-levels below the cut,
  * subtrees:    distinct depth-k beliefs reached per pass (mean).
    python scripts/ownership_balance.py --config c2 --gpus 8 > profiles/r02_ownership_c2.json
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2510_27191_b200 as vp  # noqa: E402

CONFIGS = {
    "c2": (lambda: vp.MarsModel(11, 11, layout_seed=1000), 16384, 10),
    "c3": (lambda: vp.MarsModel(15, 15, layout_seed=1000), 65536, 10),
    "c5": (lambda: vp.SyntheticModel(n_actions=16, n_obs=8, seed=1000), 65536, 20),
}


def mix(x):
    x = (x ^ (x >> 30)) * np.uint64(0xBF58476D1CE4E5B9)
    x = (x ^ (x >> 27)) * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> 31)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--gpus", type=int, default=8)
    ap.add_argument("--rows-per-gpu", type=int, default=None)
    a = ap.parse_args()
    make, n1, iters = CONFIGS[a.config]
    n = (a.rows_per_gpu or n1) * a.gpus  # weak scaling: the whole job's rows in one tree
    model = make()
    belief = vp.ParticleBelief.from_model(model, 10_000, vp.RowRng.from_seed(1000).derive(3))
    out = vp.plan(belief, model, vp.SolverConfig(n_parallel=n, iterations=iters), vp.RowRng.from_seed(1000).derive(1, 0),
                  trace=True)
    res = {"config": a.config, "gpus": a.gpus, "rows": n, "iterations": iters, "cuts": {}}
    G = np.uint64(a.gpus)
    with np.errstate(over="ignore"):
        for k in (1, 2, 3, 4):
            top = below = 0
            imb, subtrees, pass_max, pass_mean = [], [], 0.0, 0.0
            per_rank_total = np.zeros(a.gpus)
            for it in out.traces:
                levels = it["levels"]
                d = len(levels)
                if d <= k:
                    top += n * d
                    per_rank_total += n * d / a.gpus  # rows stay home: even
                    continue
                owner_b = levels[k - 1]["next_beliefs"]  # belief at depth k per row
                reach = np.ones(n, dtype=bool)  # (terminal rows keep their belief: still routed)
                top += n * k
                load = np.zeros(a.gpus)
                owners = (mix(owner_b.astype(np.uint64) + np.uint64(0x9E3779B97F4A7C15)) % G).astype(np.int64)
                np.add.at(load, owners[reach], d - k)
                below += load.sum()
                per_rank_total += load + n * k / a.gpus
                imb.append(float(load.max() / max(load.mean(), 1e-9)))
                pass_max += load.max()
                pass_mean += load.mean()
                subtrees.append(int(len(np.unique(owner_b))))
            res["cuts"][k] = {"row_levels_top": int(top), "row_levels_below": int(below),
                              "top_fraction": round(top / max(top + below, 1), 4),
                              "imbalance_per_pass": [round(x, 3) for x in imb],
                              "imbalance_mean": round(float(np.mean(imb)) if imb else 1.0, 3),
                              "imbalance_weighted": round(pass_max / max(pass_mean, 1e-9), 3),
                              "subtrees_per_pass": subtrees,
                              "step_imbalance": round(float(per_rank_total.max() / per_rank_total.mean()), 3)}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
