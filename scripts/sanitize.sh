# compute-sanitizer on small planning steps (memcheck, racecheck, synccheck); bounded by timeouts
cat > /tmp/san_plan.py <<'PY'
import sys
sys.path.insert(0, ".")
import numpy as np
import oracle
import paper_2510_27191_b200 as vp
for om, n, it in ((oracle.MarsModel(7, 8, layout_seed=1), 96, 4), (oracle.SyntheticModel(seed=2), 64, 5),
                  (oracle.CrowdNavModel(n_people=40), 32, 3)):
    b = oracle.ParticleBelief.from_model(om, 200, oracle.RowRng.from_seed(1).derive(3))
    for prec, exact in (("fp32", False), ("fp64", True)):
        out = vp.plan(b, om, oracle.SolverConfig(n_parallel=n, iterations=it), oracle.RowRng.from_seed(1),
                      precision=prec, exact=exact, keep_tree=True)
        out.tree.validate()
    db = vp.DeviceBelief.from_host(b, om)
    vp.sir_update(db, om, 0, 0, oracle.RowRng.from_seed(5))
    # Philox streams (fast mode) on the same plan
    vp.plan(b, om, oracle.SolverConfig(n_parallel=n, iterations=it), vp.PhiloxRowRng.from_seed(1)).tree_stats
# a user-model plug-in (CudaModel): plan + SIR through its plug-in build
from paper_2510_27191_b200.envs.plugin_examples import corridor_cuda_model
pm = corridor_cuda_model()
pb = vp.ParticleBelief.from_model(pm, 200, vp.RowRng.from_seed(1).derive(3))
for prec, exact in (("fp32", False), ("fp64", True)):
    vp.plan(pb, pm, vp.SolverConfig(n_parallel=64, iterations=4), vp.RowRng.from_seed(1), precision=prec,
            exact=exact, keep_tree=True).tree.validate()
vp.sir_update(vp.DeviceBelief.from_host(pb, pm), pm, 1, 3, vp.RowRng.from_seed(5))
print("plans ok")
PY
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python /tmp/san_plan.py > gpurun_out/san_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|plans ok|Error" gpurun_out/san_$tool.log | head -5
done
