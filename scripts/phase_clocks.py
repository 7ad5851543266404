"""Per-phase cycles of the search kernel (measurement build, see phase_clocks.sh)."""
import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2510_27191_b200 as vp  # noqa: E402
from paper_2510_27191_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=11)
ap.add_argument("--n-parallel", type=int, default=16384)
ap.add_argument("--iterations", type=int, default=10)
a = ap.parse_args()
model = vp.MarsModel(a.n, a.n, layout_seed=1000)
belief = vp.ParticleBelief.from_model(model, 10_000, vp.RowRng.from_seed(1000).derive(3))
cfg = vp.SolverConfig(n_parallel=a.n_parallel, iterations=a.iterations)
lib = _lib.load()
buf = (C.c_ulonglong * 24)()
for t in range(3):
    vp.plan(belief, model, cfg, vp.RowRng.from_seed(1000).derive(1, t))
torch.cuda.synchronize()
lib.vp_debug_phases(buf)
names = ["rec wait", "draw", "model", "claims", "post-action", "belief-post", "arrive+tail", "leaf"]
tot = sum(buf[:8])
warps = (a.n_parallel + 31) // 32
levels = sum(min(i + 1, 50) for i in range(a.iterations)) * 3
for k in range(8):
    print(f"{names[k]:16s} {100.0 * buf[k] / tot:5.1f}%  {buf[k] / warps / levels:8.0f} cycles per warp-level")
dr = ["-", "init/overlay draw", "-", "stage issue", "TMA wait", "-", "bsearch"]
for k in (1, 3, 4, 6):
    print(f"  draw.{dr[k]:18s} {buf[8 + k] / warps / levels:8.0f} cycles per warp-level")
bk = ["belief completion (prev) + loop test", "climb step (loads, deliveries, Q)", "final completion"]
for k in range(3):
    print(f"  backup.{bk[k]:34s} {buf[16 + k] / 1e6:8.2f} Mcycles (warp sum)")
# the backup completion wave of one planning step: per pass and depth, when completions happened
import numpy as np  # noqa: E402
buf_t = (C.c_ulonglong * (1 << 21))()
lib.vp_debug_trace(None, 0)
vp.plan(belief, model, cfg, vp.RowRng.from_seed(1000).derive(1, 99))
torch.cuda.synchronize()
cnt = lib.vp_debug_trace(buf_t, 1 << 21)
tr = np.frombuffer(buf_t, dtype=np.uint64, count=cnt)
t = (tr >> np.uint64(24)).astype(np.int64)
ps = ((tr >> np.uint64(18)) & np.uint64(63)).astype(np.int64)
dp = ((tr >> np.uint64(12)) & np.uint64(63)).astype(np.int64)
wp = (tr & np.uint64(4095)).astype(np.int64)
for p in sorted(set(ps.tolist())):
    m = ps == p
    t0 = t[m & (dp == 63)].min()
    parts = []
    for d in sorted(set(dp[m].tolist()) - {63}):
        x = (t[m & (dp == d)] - t0) / 1e3
        parts.append(f"d{d}:{np.percentile(x, 50):.1f}/{np.percentile(x, 90):.1f}/{x.max():.1f}(n={len(x)})")
    print(f"  backup pass {p} completion us p50/p90/max after the first warp:", " ".join(parts))
    if p == max(ps.tolist()):  # the last pass: the critical path's warps
        sel = np.flatnonzero(m & (dp != 63))
        late = sel[np.argsort(t[sel])[-40:]]
        print("   last completions (us, depth, warp):", [(round((t[i] - t0) / 1e3, 1), int(dp[i]), int(wp[i])) for i in late])
        starts = {int(wp[i]): round((t[i] - t0) / 1e3, 1) for i in np.flatnonzero(m & (dp == 63))}
        print("   those warps started at:", {w: starts.get(w) for w in sorted(set(int(wp[i]) for i in late))})
print(f"  backup multi-delivery belief deliveries: {buf[20]}, distinct (warp, iteration, belief) groups: {buf[21]}")
