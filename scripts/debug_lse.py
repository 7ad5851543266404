"""Compare every belief's cached LSE with the LSE of its exported PSI row after an injected plan."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import torch
import paper_2510_27191_b200 as vp
from golden_cases import manifest
import test_gpu_plan as TP

for name, prec in (("plan_mars4_3", "fp64"), ("plan_crowdnav40", "fp32"), ("plan_mars4_3", "fp32")):
    case = manifest()["plans"][name]
    s = case["runs"][0]["seed"]
    om, belief, cfg, rng, ref, traces, inject = TP._oracle_traces(case, s)
    for it in (1, 2, 3, cfg.iterations):
        c2 = vp.SolverConfig(n_parallel=cfg.n_parallel, iterations=it)
        ref_it = __import__("oracle").plan(belief, om, __import__("oracle").SolverConfig(n_parallel=cfg.n_parallel, iterations=it), rng)
        out = vp.plan(belief, om, c2, rng, precision=prec, inject_actions=inject[:it], keep_tree=True, trace=True)
        t = out.tree
        tab = t.tables()
        want = ref_it.tree.tables()["prefs"]
        got = tab["prefs"]
        eta = 2.0
        border, brank, _, _ = t.canonical()
        lse_dev = t.b_lse[: len(got)][border].cpu().numpy()
        z = eta * got
        m = z.max(axis=1)
        lse_row = m / eta + np.log(np.exp(z - m[:, None]).sum(axis=1)) / eta
        err_lse = np.abs(lse_dev - lse_row)
        err_p = np.abs(got - want).max(axis=1)
        rec = t.b_rec[: len(got)][border].cpu().numpy()
        nact = t.b_nact[: len(got)][border].cpu().numpy()
        bad = np.argsort(-err_p)[:5]
        print(name, prec, "iters", it, "max |lse_dev - lse(row)|", err_lse.max(), "max prefs err", err_p.max())
        for b in bad:
            print("   belief", b, "depth", tab["depth"][b], "prefs err", err_p[b], "lse err", err_lse[b], "nact", nact[b],
                  "rec", rec[b][:4], "got", got[b][:6], "want", want[b][:6])
        worst_l = np.argsort(-err_lse)[:3]
        for b in worst_l:
            print("   lse-worst belief", b, "depth", tab["depth"][b], "lse err", err_lse[b], "nact", nact[b], "rec", rec[b][:4])
