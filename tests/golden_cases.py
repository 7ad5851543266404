"""Shared helpers: rebuild the golden plan cases with the oracle or the device.

The case list mirrors tests/golden/make_golden.py (which ran the REAL
reference).  Nothing here reads /root/reference.
"""

from __future__ import annotations

import json
import os

import numpy as np

import oracle

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden")

INT_COLUMNS = ("parent_action", "parent_obs", "depth", "action_parent_belief", "action_id", "action_visits")


def manifest() -> dict:
    with open(os.path.join(GOLDEN, "manifest.json")) as f:
        return json.load(f)


def load(name: str) -> dict:
    with np.load(os.path.join(GOLDEN, name + ".npz")) as z:
        return {k: z[k] for k in z.files}


def oracle_model(kind: str, seed: int):
    if kind.startswith("mars"):
        n, m = map(int, kind[4:].split("_"))
        return oracle.MarsModel(n=n, m=m, layout_seed=seed)
    if kind == "tiger":
        return oracle.tiger_model()
    if kind == "synthetic":
        return oracle.SyntheticModel(n_actions=16, n_obs=8, seed=seed)
    if kind == "lightdark":
        return oracle.LightDarkModel()
    if kind == "navigation":
        return oracle.NavigationModel()
    if kind.startswith("crowdnav"):
        return oracle.CrowdNavModel(n_people=int(kind[8:] or 300))
    raise ValueError(kind)


CROWD_CASES = (("p40", 40, 96, 6), ("p300", 300, 8, 3))  # tag, people, rows, steps (make_golden.py)
CROWD_FIELDS = ("robot", "persons", "curious", "tracked", "prev_dist", "last_code", "terminal")


def plan_inputs(case: dict, seed: int, model=None):
    """(model, belief, config, rng) exactly as make_golden.py built them."""
    model = model or oracle_model(case["kind"], seed)
    belief = oracle.ParticleBelief.from_model(model, case["particles"], oracle.RowRng.from_seed(seed).derive(3))
    cfg = oracle.SolverConfig(n_parallel=case["n_parallel"], iterations=case["iterations"], eta=case["eta"])
    rng = oracle.RowRng.from_seed(seed).derive(1, 0)
    return model, belief, cfg, rng


def tree_columns(tables: dict) -> dict:
    """Golden-comparable columns from a dict of full tables."""
    out = {k: np.asarray(tables[k]) for k in INT_COLUMNS}
    out["action_reward_sum"] = np.asarray(tables["action_reward_sum"], dtype=np.float64)
    prefs = np.asarray(tables["prefs"], dtype=np.float64)
    out["prefs"] = prefs
    out["prefs_row_sum"] = prefs.sum(axis=1)
    out["prefs_root"] = prefs[0]
    return out


# SPEC.md ACCEPTANCE 2 (make_golden.gen_serial_search): n, m, seed, d_max cap, episodes, eta
SERIAL_CASES = [(4, 3, 5, 2, 30, 0.05), (4, 3, 6, 3, 30, 0.1), (4, 4, 7, 4, 40, 0.05)]


def serial_search_build(vpmod, case, make_tree, **plan_kw):
    """Width-1 episodes through ``vpmod``'s search + backup (the vectorized path at n_p = 1),
    episode e from rng.derive(1, e) exactly as the reference's serial_search_backup builds it."""
    n, m, seed, dcap, episodes, eta = case
    model = vpmod.MarsModel(n=n, m=m, layout_seed=seed)
    belief = vpmod.ParticleBelief.from_model(model, 200, oracle.RowRng.from_seed(seed).derive(3))
    tree = make_tree(model)
    for e in range(episodes):
        it = oracle.RowRng.from_seed(seed).derive(1, e)
        state = belief.sample_states(1, it.derive(0))
        d = min(e + 1, dcap)
        leaves = vpmod.search(tree, model, vpmod.SearchBatch(np.zeros(1, dtype=np.int64), state), d, eta, it.derive(1))
        vpmod.backup(tree, leaves, d, eta, model.spec.discount)
    return tree


def parse_tree_text(text):
    """to_text() / serialize() dump -> (integer rows, float rows) for tolerance comparisons."""
    ints, floats = [], []
    for line in text.splitlines():
        f = line.split("\t")
        if f[0] == "B":
            ints.append(tuple(int(x) for x in f[1:]))
        elif f[0] == "A":
            ints.append((int(f[1]), int(f[2]), int(f[3]), int(f[5])))
            floats.append(float(f[4]))
        elif f[0] == "P":
            ints.append((int(f[1]), int(f[2])))
            floats.extend(float(x) for x in f[3:])
    return ints, np.array(floats)
