"""Phase timeline of the persistent planning kernel (globaltimer per barrier)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2510_27191_b200 as vp  # noqa: E402
from paper_2510_27191_b200 import _lib  # noqa: E402
from paper_2510_27191_b200.rng import fold, key_of  # noqa: E402

iters = int(os.environ.get("ITERS", "10"))
npar = int(os.environ.get("NPAR", "16384"))
model = vp.MarsModel(11, 11, layout_seed=1000)
belief = vp.ParticleBelief.from_model(model, 10_000, vp.RowRng.from_seed(1000).derive(3))
cfg = vp.SolverConfig(n_parallel=npar, iterations=iters)
p = vp.Planner("fp32")
for t in range(3):
    p.plan(belief, model, cfg, vp.RowRng.from_seed(1000).derive(1, t))
dm, tree, work = p.prepare(model, cfg, device_init=False)
m = p.stage_belief(dm, belief)
tl = torch.zeros(4096, dtype=torch.int64, device="cuda")
# reuse run_fixed's buffers, then call vp_plan directly with a timeline
p.run_fixed(dm, tree, work, m, model.spec, cfg, key_of(vp.RowRng.from_seed(1000).derive(1, 5)))
dm, tree, work = p.prepare(model, cfg, device_init=False)
a = _lib.VpPlanArgs()
a.iterations, a.d_max_cap, a.m, a.mode = iters, cfg.d_max_cap, m, 2
a.gamma = model.spec.discount
a.particles_host, a.particles_dev = p._bufs["particles_host"].data_ptr(), p._bufs["particles_dev"].data_ptr()
a.cumw_host, a.cumw_dev = p._bufs["cumw_host"].data_ptr(), p._bufs["cumw_dev"].data_ptr()
a.keys_host, a.keys_dev = p._bufs["keys_host"].data_ptr(), p._bufs["keys_dev"].data_ptr()
a.out_host, a.out_dev = p._bufs["out_host"].data_ptr(), p._bufs["out_dev"].data_ptr()
a.timeline_dev, a.timeline_cap = tl.data_ptr(), 4096
_lib.call("vp_plan", C.byref(tree.struct), C.byref(dm.desc), C.byref(work.struct), C.byref(a),
          torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
t = tl.cpu().numpy()
t = t[: np.flatnonzero(t)[-1] + 1]
dt = np.diff(t) / 1e3
print("total_us", (t[-1] - t[0]) / 1e3, "phases", len(dt))
# label phases
labels = ["init+draw"]
for it in range(iters):
    d = min(it + 1, cfg.d_max_cap)
    if it:
        labels.append("draw")
    for l in range(d):
        labels += [f"sample{l}", f"assignA+accum{l}"]
    labels[-1] = labels[-1]
    labels += ["assignB_last+leaf", "backup_leaves"]
    for lv in range(d - 1, -1, -1):
        labels += [f"q{lv}", f"v{lv}"]
import collections
agg = collections.defaultdict(float)
cnt = collections.Counter()
for lab, x in zip(labels, dt):
    key = ''.join(ch for ch in lab if not ch.isdigit())
    agg[key] += x
    cnt[key] += 1
for k, v in sorted(agg.items(), key=lambda kv: -kv[1]):
    print(f"{k:24s} n={cnt[k]:4d} total_us={v:9.1f} avg_us={v / cnt[k]:7.2f}")
print("last iteration:", [f"{lab}:{x:.1f}" for lab, x in zip(labels[-60:], dt[-60:])])
