"""Benchmark of the PORPP planning step on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Workload (BASELINE.json configs[1]): one planning
step ``plan()`` on RockSample(11,11) = MarsModel(n=11, m=11), |A| = 256,
n_parallel = 16 384 simulations per iteration, 10 iterations (d_max 1..10),
eta = 2.0, a 10 000-particle belief.  A "step" is one whole planning step.

* ``value``  -- simulations/s with the belief already resident in HBM: each
  step is tree reset + 10 x (root draw, search, backup) + root argmax, timed
  with CUDA events on the planner's stream around each step; L2 is flushed
  (256 MB write) between steps, outside the events.
* ``e2e``    -- the same metric through the public ``plan()`` call with the
  particle StateBatch on the host (pack + pinned H2D + D2H of the action).
* ``roofline`` -- the dominant kernel's algorithmic bytes per launch over its
  CUDA-event duration (profiled pass of the same steps) vs MEASURED_PEAKS, and
  beside it a latency floor: dependent L2 round trips per level x the L2 load /
  atomic latency measured on this GPU (vp_probe_latency).
* ``secondary`` -- (N = 1) the same measurements for C3 (RockSample(15,15),
  65 536 x 10), C5 (Synthetic, 65 536 x 20) and the headline in fp64.
* ``cpu_baseline`` -- the CPU oracle (numpy port of the reference) timed on
  this host, one core, on one planning step of the same workload.
* ``--impl reference`` -- the reference algorithm on the host CPU (the oracle
  port; /root/reference is not on the GPU box): one concurrent plan() per core.

Multi-GPU (torchrun, N > 1): every rank plans its own replica of the
workload (different seeds); the value is the sum over ranks, timed as the
max over ranks ("replicas", scaling "weak").
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

WORKLOAD = {"problem": "mars", "n": 11, "m": 11, "n_parallel": 16384, "iterations": 10, "eta": 2.0,
            "particles": 10_000}
# BASELINE.json configs: c2 is the headline workload;
# the others are measured on request (--config) for the scaling evidence.
CONFIGS = {
    "c1": {"problem": "mars", "n": 7, "m": 8, "n_parallel": 1024, "iterations": 8,
           "name": "RockSample(7,8)=MarsModel(7,8)"},
    "c2": {"problem": "mars", "n": 11, "m": 11, "n_parallel": 16384, "iterations": 10,
           "name": "RockSample(11,11)=MarsModel(11,11)"},
    "c3": {"problem": "mars", "n": 15, "m": 15, "n_parallel": 65536, "iterations": 10,
           "name": "RockSample(15,15)=MarsModel(15,15)"},
    "c4": {"problem": "lightdark", "n_parallel": 16384, "iterations": 20, "name": "LightDark(64x64 bins)"},
    "c5": {"problem": "synthetic", "n_parallel": 65536, "iterations": 20, "name": "Synthetic(|A|=16,|O|=8)"},
}
METRIC = "belief-tree simulations/sec per planning step"
UNIT = "simulations/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--n-parallel", type=int, default=None)
    ap.add_argument("--iterations", type=int, default=None)
    ap.add_argument("--precision", default="fp32", choices=["fp32", "fp64"])
    ap.add_argument("--rng", default="splitmix64", choices=["splitmix64", "philox"],
                    help="per-row streams: the reference's SplitMix64 hash or the Philox4x32-10 fast mode")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", dest="secondary", action="store_false",
                    help="skip the secondary workloads (C3, C5, fp64 C2) measured beside the headline at N = 1")
    ap.add_argument("--cpu-budget-s", type=float, default=20.0)
    ap.add_argument("--episodes", type=int, default=3, help="closed-loop episodes reported beside the step metric")
    ap.add_argument("--multi", default="sharded", choices=["sharded", "replicas"],
                    help="N > 1: one planning step sharded over the GPUs (n_parallel rows per GPU, "
                         "trajectories all-gathered over NCCL) or independent replicas")
    a = ap.parse_args()
    c = CONFIGS[a.config]
    a.n_parallel = a.n_parallel or c["n_parallel"]
    a.iterations = a.iterations or c["iterations"]
    return a


def make_model(lib, args, seed):
    """The config's problem model from `lib` (the product package or the oracle)."""
    c = CONFIGS[args.config]
    if c["problem"] == "mars":
        return lib.MarsModel(n=c["n"], m=c["m"], layout_seed=seed)
    if c["problem"] == "lightdark":
        return lib.LightDarkModel()
    return lib.SyntheticModel(n_actions=16, n_obs=8, seed=seed)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload_config(args, actions):
    """The workload, identical in the b200 and reference arms (how it is executed goes to the line's
    top-level "execution" key)."""
    c = CONFIGS[args.config]
    return {"workload": f"{c['name']} plan(), n_parallel={args.n_parallel}, iterations={args.iterations}",
            "config_id": args.config, "problem": c["name"], "actions": actions, "n_parallel": args.n_parallel,
            "iterations": args.iterations, "eta": WORKLOAD["eta"], "particles": WORKLOAD["particles"],
            "simulations_per_step": args.n_parallel * args.iterations,
            "episode_steps_per_step": args.n_parallel * sum(range(1, args.iterations + 1)),
            "parallelism": "one plan() per step",
            "l2": "flushed between timed steps (256 MB write, outside the per-step CUDA events)",
            **({"rng": "philox4x32-10"} if getattr(args, "rng", "splitmix64") == "philox" else {})}


# ---------------------------------------------------------------- clocks


class ClockSampler:
    """SM clock and clock-event reasons sampled DURING the timed region: NVML polled every
    2 ms from a thread (the region can be ~10 ms, shorter than nvidia-smi's first sample);
    nvidia-smi -lms 100 as the fallback when NVML is unavailable."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))

    def __init__(self, index: int, period_s: float = 0.002):
        self.sm, self.mx, self.reasons = [], [], set()
        self.proc = None
        try:
            import threading

            import pynvml

            pynvml.nvmlInit()
            visible = os.environ.get("CUDA_VISIBLE_DEVICES", "")
            nvml_index = int(visible.split(",")[index]) if visible and visible.split(",")[index].isdigit() else index
            h = pynvml.nvmlDeviceGetHandleByIndex(nvml_index)
            get_reasons = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons",
                                  getattr(pynvml, "nvmlDeviceGetCurrentClocksThrottleReasons", None))
            bits = [(nm, getattr(pynvml, attr, 0)) for nm, attr in self.REASONS]
            max_sm = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            self._stop = threading.Event()

            def poll():
                while True:
                    self.sm.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                    self.mx.append(max_sm)
                    r = get_reasons(h) if get_reasons else 0
                    self.reasons.update(nm for nm, bit in bits if r & bit)
                    if self._stop.wait(period_s):
                        return

            self.thread = threading.Thread(target=poll, daemon=True)
            self.thread.start()
            self.source = "nvml"
        except Exception:  # noqa: BLE001 -- no NVML: nvidia-smi
            self.thread = None
            self.source = "nvidia-smi"
            self.path = tempfile.mktemp(suffix=".csv")
            q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap")
            try:
                self.proc = subprocess.Popen(["nvidia-smi", f"--id={index}", f"--query-gpu={q}",
                                              "--format=csv,noheader,nounits", "-lms", "100"],
                                             stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            except OSError:
                self.proc = None

    def stop(self) -> dict:
        if self.thread is not None:
            self._stop.set()
            self.thread.join()
        elif self.proc is not None:
            self.proc.terminate()
            self.proc.wait()
            names = [nm for nm, _ in self.REASONS]
            for line in open(self.path):
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 7:
                    continue
                try:
                    self.sm.append(float(parts[0]))
                    self.mx.append(float(parts[1]))
                except ValueError:
                    continue
                for nm, v in zip(names, parts[3:7]):
                    if v.lower().startswith("active"):
                        self.reasons.add(nm)
            os.unlink(self.path)
        else:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no NVML, no nvidia-smi"], "samples": 0}
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None, "sm_max_mhz": max(self.mx) if self.mx else None,
                "reasons": sorted(self.reasons), "samples": len(self.sm), "source": self.source}


# ---------------------------------------------------------------- algorithmic bytes


def algorithmic_bytes(st, n, S, A, psi_b, passes):
    """Compulsory HBM bytes of the search, backup and CDF kernels summed over `passes` passes,
    from the device traffic counters (adapted to the fused design: states
    and frontier ids stay in registers across levels; node fields at element granularity, hash
    probes at 32-B sector granularity; fast-mode PSI: a belief is its overlay record -- one
    record + its cached LSE per distinct belief visited -- and only beliefs with more than 4
    action children own a dense row, whose CDF row the search reads once per pass when sampled).

    U   interior beliefs backed up (= distinct beliefs sampled from), P distinct action nodes
        visited, L distinct leaves, NA / NB new action / belief nodes, D dense rows changed by
        a backup (their CDF rows rebuilt; ~ the distinct dense rows the next pass samples),
        M dense rows materialised, F full-row LSE reads (fallback), R dense rows in use.
    """
    U, P, L, NA, NB = st[0], st[1], st[7], st[5], st[6]
    D, M, F = st[11], st[10], st[8]
    rec = 8 * psi_b + 8  # overlay record: 32 B (fp32) / 48 B (fp64)
    children = (U - passes) + L  # distinct (a, o) probes: every visited non-root belief
    search = (n * passes * S                   # root-state gather
              + (rec + 8) * (U + L)            # record + cached LSE of every distinct belief reached
              + psi_b * A * D                  # CDF row per distinct dense belief sampled
              + 32 * (P + children)            # one hash sector per distinct probe (claims)
              + 16 * P                         # reward / visit / row reductions per action
              + 24 * NA + 40 * NB              # new node columns (+ child count, overlay slot)
              + psi_b * A * M                  # dense rows materialised
              + 12 * L)                        # leaf heuristic sums + leaf list
    backup = (24 * L                           # leaf (rows, value) read + reset
              + (56 + rec + 2 * psi_b) * P     # action stats + slot, accumulator r/w, record + cell r/w
              + 76 * U                         # belief LSE / rows / parents, accumulator r/w
              + psi_b * A * F                  # full-row LSE (ill-conditioned incremental sums)
              + 16 * D)                        # CDF rebuild request (LSE, pass) per changed dense row
    cdf = 2 * psi_b * A * D                    # k_cdf_rows: the changed rows read, their CDFs written
    return search, backup, cdf


# dependent global round trips on a warp's critical path per level:
# search = the child's overlay record + a dense row's CDF (TMA) (loads), the (b,a) and (a,o)
# claims issued together, ids static (one atomic); backup = node fetch (load) + delivery to
# the parent (atomic)
ROUND_TRIPS = {"search": {"load": 2, "atomic": 1}, "backup": {"load": 1, "atomic": 1}}


def probe_latency(vp_lib, torch) -> dict:
    """Unloaded L2 load and L2 atomic round-trip latency on this GPU (vp_probe_latency: one thread
    chasing a random cycle of 128-B lines in a 64 MB, L2-resident buffer)."""
    lines = 1 << 19
    perm = torch.randperm(lines, device="cuda", dtype=torch.int64)
    nxt = torch.zeros(lines * 16, dtype=torch.int64, device="cuda")
    nxt[perm * 16] = torch.roll(perm, -1) * 16
    out = torch.zeros(3, dtype=torch.float64, device="cuda")
    stream = torch.cuda.current_stream().cuda_stream
    res = {}
    for name, atomic in (("l2_load", 0), ("l2_atomic", 1)):
        vals = []
        for rep in range(3):
            vp_lib.call("vp_probe_latency", nxt.data_ptr(), 20000, atomic, int(perm[0].item()) * 16, out.data_ptr(),
                        stream)
            torch.cuda.synchronize()
            vals.append(out[:2].cpu().numpy().copy())
        best = min(vals, key=lambda v: v[0])
        res[name] = {"ns": round(float(best[0]), 1), "cycles": round(float(best[1]), 1)}
    del nxt, perm
    return res


# ---------------------------------------------------------------- b200 arm


def _dist_setup(args):
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    local = local % max(1, torch.cuda.device_count())  # VP_DIST_BACKEND=gloo check on one GPU
    torch.cuda.set_device(local)
    if world > 1:
        # VP_DIST_BACKEND=gloo: several ranks on ONE GPU (NCCL refuses a shared device) -- a
        # functional check of the multi-rank path only, never a measurement
        backend = os.environ.get("VP_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return rank, world, local


def measure(args, rank, world, local, *, profile=True, clocks=True, latency=None) -> dict:
    """One workload: device-timed planning steps (belief resident), the same through the public
    plan() with host buffers (e2e), and a profiled pass (per-kernel times + traffic counters)."""
    import torch
    import torch.distributed as dist

    import paper_2510_27191_b200 as vp
    from paper_2510_27191_b200 import _lib
    from paper_2510_27191_b200.rng import key_of, kind_of

    sharded = world > 1 and args.multi == "sharded"
    # sharded: ONE planning step over world * n_parallel rows (same seed on every rank);
    # replicas: every rank plans its own problem
    seed = 1000 + (0 if sharded else rank)
    model = make_model(vp, args, seed)
    A = model.spec.action_count
    belief = vp.ParticleBelief.from_model(model, WORKLOAD["particles"], vp.RowRng.from_seed(seed).derive(3))
    n_rows = args.n_parallel * (world if sharded else 1)
    cfg = vp.SolverConfig(eta=WORKLOAD["eta"], n_parallel=n_rows, iterations=args.iterations)
    # single GPU: the planner the public vp.plan() uses, so the device-timed and the e2e steps
    # share one tree arena (large configs only fit once)
    planner = vp.ShardedPlanner(world, rank, group=dist.group.WORLD, precision=args.precision) if sharded \
        else vp.solver.get_planner(args.precision, False)
    dm = vp.device_model(model)
    particles, cumw, m = planner.upload_belief(dm, belief)
    rng_cls = vp.PhiloxRowRng if getattr(args, "rng", "splitmix64") == "philox" else vp.RowRng
    rngs = [rng_cls.from_seed(seed).derive(1, t) for t in range(args.warmup + args.steps)]

    def step(t):
        if sharded:  # trajectories of this rank's rows, one NCCL all-gather per pass, replicated insert + backup
            return planner.plan(belief, model, cfg, rngs[t], resident=(particles, cumw, m))
        # belief resident in HBM; one vp_plan call (CUDA graph replay) per planning step
        d, tree, work = planner.prepare(model, cfg, device_init=False)
        d.desc.rng_kind = kind_of(rngs[t])
        return planner.run_fixed(d, tree, work, m, model.spec, cfg, key_of(rngs[t]), from_host=False)

    def plan_e2e(t):
        if sharded:
            return planner.plan(belief, model, cfg, rngs[t])
        return vp.plan(belief, model, cfg, rngs[t], precision=args.precision)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # L2 flush between timed steps (outside the timed events): a 256 MB write, twice the L2
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def timed(fn, t0, count):
        """Per-step CUDA events on the planner's stream with an L2 flush between steps; returns
        (sum of step times in ms, outputs)."""
        evs, outs = [], []
        for t in range(count):
            flush_buf.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            outs.append(fn(t0 + t))
            b.record()
            evs.append((a, b))
        torch.cuda.synchronize()
        return sum(a.elapsed_time(b) for a, b in evs), outs

    for t in range(args.warmup):
        step(t)
    barrier()
    sampler = ClockSampler(local) if clocks else None
    launches0 = _lib.launch_count()
    elapsed, outs = timed(step, args.warmup, args.steps)
    barrier()
    launches = _lib.launch_count() - launches0  # the library's own launches (flushes are torch's)
    elapsed_ms = max_over_ranks(elapsed)
    clk = sampler.stop() if sampler else None
    sims = args.n_parallel * args.iterations * args.steps * world
    value = sims / (elapsed_ms / 1e3)

    # e2e through the public API with host buffers (own warm-up: first call captures its graph)
    for t in range(args.warmup):
        plan_e2e(t)
    barrier()
    e2e_elapsed, _ = timed(plan_e2e, args.warmup, args.steps)
    barrier()
    e2e_ms = max_over_ranks(e2e_elapsed)
    e2e = sims / (e2e_ms / 1e3)
    # bytes actually copied per e2e step: the particle records, plus the weight CDF unless the
    # weights are exactly uniform (then the planner uses its cached device CDF)
    w = np.asarray(belief.weights, dtype=np.float64)
    h2d = len(belief.states) * dm.state_bytes + (0 if not (w != 1.0 / len(w)).any() else 8 * len(w))

    res = {"value": round(value, 1), "ms_per_step": round(elapsed_ms / args.steps, 4),
           "e2e": {"value": round(e2e, 1), "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": 16,
                   "ms_per_step": round(e2e_ms / args.steps, 4)},
           "gpu_launches": int(launches), "clocks": clk, "actions": A,
           "tree_stats": outs[-1].tree_stats, "chosen_action": outs[-1].chosen_action}
    if not profile:
        return res

    # profiled pass of the same steps: per-kernel-kind device time (CUDA events around every
    # launch on the planner's stream) and the traffic counters the kernels keep
    _lib.profile_enable(True)
    prof_steps = min(args.steps, 3)
    planner.work.stats.zero_()
    planner.work.enable_stats(True)
    for t in range(prof_steps):
        step(args.warmup + t)
    torch.cuda.synchronize()
    prof = _lib.profile_read()
    _lib.profile_enable(False)
    planner.work.enable_stats(False)
    st = planner.work.stats.cpu().numpy().astype(np.float64)
    kinds = {k: v for k, v in prof.items() if v[1]}
    total_ms = sum(v[0] for v in kinds.values())
    top = max(kinds, key=lambda k: kinds[k][0])
    peaks = json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(REPO, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0}
    peak = float(peaks.get("hbm_gbs", 6650.0))
    psi_b = 4 if args.precision == "fp32" else 8
    S = dm.state_bytes
    passes = prof_steps * args.iterations
    b_search, b_backup, b_cdf = algorithmic_bytes(st, args.n_parallel, S, A, psi_b, passes)
    levels_per_pass = st[4] / max(1.0, args.n_parallel * passes)

    # measured DRAM bytes per launch of the same workload (ncu launch list, scripts/ncu_capture.sh +
    # scripts/launch_traffic.py), committed under profiles/
    tpath = os.path.join(REPO, "profiles", f"traffic_{args.config}.json")
    measured = {}
    if os.path.exists(tpath) and world == 1:
        tj = json.load(open(tpath))
        if tj.get("precision", "fp32") == args.precision and tj.get("n_parallel", args.n_parallel) == args.n_parallel:
            measured = tj["kernels"]

    def roof(kind, kname, total_bytes, formula):
        ms, cnt = kinds.get(kind, (0.0, 0))
        if not cnt:
            return None
        per_launch = total_bytes / cnt
        avg_ms = ms / cnt
        ach = per_launch / (avg_ms / 1e3) / 1e9
        traffic = measured.get(kname, {}).get("dram_bytes_per_launch")
        out = {"kernel": kname, "bound": "hbm", "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
               "frac": round(ach / peak, 4), "traffic": round(traffic) if traffic else None,
               "traffic_source": f"profiles/traffic_{args.config}.json (ncu dram__bytes_read+write, "
                                 f"avg per launch)" if traffic else None,
               "bytes_per_launch": round(per_launch),
               "avg_launch_us": round(avg_ms * 1e3, 2), "share_of_step": round(ms / total_ms, 3),
               "algorithmic_bytes": formula, "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured copy)"}
        if latency and kind in ROUND_TRIPS:
            rt = ROUND_TRIPS[kind]
            lvl_ns = rt["load"] * latency["l2_load"]["ns"] + rt["atomic"] * latency["l2_atomic"]["ns"]
            floor_us = levels_per_pass * lvl_ns / 1e3
            out["latency"] = {"bound": "l2_round_trips", "levels_per_launch": round(levels_per_pass, 2),
                              "round_trips_per_level": rt, "ns_per_level": round(lvl_ns, 1),
                              "floor_us": round(floor_us, 2), "frac": round(floor_us / (avg_ms * 1e3), 4),
                              "latency_source": "vp_probe_latency (unloaded, this GPU)"}
        return out

    roof_search = roof("search", "k_search", b_search,
                       "n S + (rec + 8)(U + L) + psi_b|A| (D + M) + 48 P + 32 children + 24 NA + 40 NB + 12 L "
                       "per pass (bench.algorithmic_bytes)")
    roof_backup = roof("backup", "k_backup", b_backup,
                       "24 L + (56 + rec + 2 psi_b) P + 76 U + psi_b|A| F + 16 D per pass (bench.algorithmic_bytes)")
    roof_cdf = roof("cdf_rows", "k_cdf_rows", b_cdf, "2 psi_b|A| D per pass (bench.algorithmic_bytes)")
    names = ["interior_beliefs", "actions_visited", "psi_rows_staged", "search_launches", "row_levels",
             "new_actions", "new_beliefs", "leaves", "full_row_lse_reads", "overlay_draws", "dense_rows_made",
             "dense_cdfs_built", "overlay_lse_fallbacks"]
    res.update({
        "roofline": {"search": roof_search, "backup": roof_backup}.get(top) or roof_search,
        "roofline_other": {"k_search": roof_search, "k_backup": roof_backup, "k_cdf_rows": roof_cdf},
        "kernels": {k: {"ms_per_step": round(v[0] / prof_steps, 4), "launches_per_step": v[1] // prof_steps}
                    for k, v in kinds.items()},
        "dominant_kernel": top,
        "traffic_per_step": {nm: st[i] / prof_steps for i, nm in enumerate(names)},
        "episode_steps_per_s": round(value * sum(range(1, args.iterations + 1)) / args.iterations, 1)})
    res["_model"] = model
    return res


# secondary workloads measured beside the headline at N = 1 (BASELINE configs[2] and [4] and the
# reference precision of the headline)
SECONDARY = [("c3", "fp32", "splitmix64"), ("c5", "fp32", "splitmix64"), ("c2", "fp64", "splitmix64"),
             ("c2", "fp32", "philox")]


def run_b200(args):
    import torch
    import torch.distributed as dist

    import paper_2510_27191_b200 as vp
    from paper_2510_27191_b200 import _lib

    rank, world, local = _dist_setup(args)
    sharded = world > 1 and args.multi == "sharded"
    latency = probe_latency(_lib, torch) if world == 1 else None
    main = measure(args, rank, world, local, latency=latency)
    model = main.pop("_model")
    line = {"metric": METRIC, "value": main["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": main["ms_per_step"], "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32" if args.precision == "fp32" else "f64",
            "data": "synthetic (MARS belief sampled from the model; no dataset)",
            "config": workload_config(args, main["actions"]),
            "execution": (f"sharded x{world}: {args.n_parallel} rows per GPU, one tree, NCCL all-gather of "
                          f"trajectories per pass" if sharded else f"replicas x{world}") if world > 1 else "1 GPU",
            **{k: main[k] for k in ("e2e", "gpu_launches", "clocks", "roofline", "roofline_other", "kernels",
                                    "dominant_kernel", "traffic_per_step", "episode_steps_per_s", "tree_stats",
                                    "chosen_action")}}
    if latency:
        line["latency_probe"] = latency
    if rank == 0 and world == 1 and args.secondary:
        sec = {}
        for cid, prec, rk in SECONDARY:
            if cid == args.config and prec == args.precision and rk == args.rng:
                continue
            a2 = argparse.Namespace(**vars(args))
            a2.config, a2.precision, a2.rng = cid, prec, rk
            a2.n_parallel, a2.iterations = CONFIGS[cid]["n_parallel"], CONFIGS[cid]["iterations"]
            r = measure(a2, rank, world, local, clocks=False, latency=latency)
            r.pop("_model")
            sec[f"{cid}_{prec}" + ("_philox" if rk == "philox" else "")] = {
                                    "config": workload_config(a2, r["actions"]), "value": r["value"],
                                    "ms_per_step": r["ms_per_step"], "e2e": r["e2e"], "dtype": prec, "rng": rk,
                                    "roofline_other": r["roofline_other"], "kernels": r["kernels"],
                                    "tree_stats": r["tree_stats"], "traffic_per_step": r["traffic_per_step"]}
            torch.cuda.empty_cache()
        line["secondary"] = sec
    if rank == 0 and world == 1 and args.episodes > 0:
        line["closed_loop"] = closed_loop(args, vp, model)
    if rank == 0 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args)
        line["speedup_vs_cpu_1core"] = round(line["e2e"]["value"] / line["cpu_baseline"]["value"], 1)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def closed_loop(args, vp, model) -> dict:
    """Closed-loop episodes (solver.py:130-194) with the belief resident in HBM: plan ->
    execute -> device SIR per step.  Reports the planning throughput inside the loop and
    the episode returns (BASELINE configs[1]: RockSample(11,11) closed-loop episodes)."""
    cfg = vp.SolverConfig(eta=WORKLOAD["eta"], n_parallel=args.n_parallel, iterations=args.iterations,
                          particles=WORKLOAD["particles"])
    vp.run_episode(model, cfg, seed=999, precision=args.precision)  # warm-up (graph capture)
    t0 = time.perf_counter()
    recs = [vp.run_episode(model, cfg, seed=s, precision=args.precision) for s in range(args.episodes)]
    wall = time.perf_counter() - t0
    steps = sum(r.steps for r in recs)
    plan_s = sum(sum(r.plan_wall_times) for r in recs)
    returns = [r.discounted_return for r in recs]
    return {"episodes": len(recs), "env_steps": steps, "belief": "device-resident (DeviceBelief, device SIR)",
            "plan_wall_ms_per_step": round(1e3 * plan_s / steps, 4),
            "simulations_per_s_in_loop": round(steps * args.n_parallel * args.iterations / plan_s, 1),
            "env_steps_per_s": round(steps / wall, 1), "mean_discounted_return": round(float(np.mean(returns)), 3),
            "returns": [round(x, 3) for x in returns]}


# ---------------------------------------------------------------- CPU (oracle port of the reference)


def _cpu_plan(seed, n_parallel, iterations, config="c2"):
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    import oracle

    model = make_model(oracle, argparse.Namespace(config=config), seed)
    belief = oracle.ParticleBelief.from_model(model, WORKLOAD["particles"], oracle.RowRng.from_seed(seed).derive(3))
    cfg = oracle.SolverConfig(eta=WORKLOAD["eta"], n_parallel=n_parallel, iterations=iterations)
    t0 = time.perf_counter()
    out = oracle.plan(belief, model, cfg, oracle.RowRng.from_seed(seed).derive(1, 0))
    return time.perf_counter() - t0, out.tree_stats


CPU_SAMPLE_ROWS = 16384  # larger workloads are timed on a bounded sample of their rows


def cpu_baseline(args) -> dict:
    """One core, whole planning steps of the same problem and iteration budget until the time
    budget is used.  Workloads above CPU_SAMPLE_ROWS rows per iteration run on that many rows to
    bound the time; the value is then the sample's rate, not a measurement at the full row count
    (the reference's per-simulation cost changes with the row count), and the
    sample string says so."""
    rows = min(args.n_parallel, CPU_SAMPLE_ROWS)
    times = []
    t_start = time.perf_counter()
    while not times or (time.perf_counter() - t_start < args.cpu_budget_s and len(times) < 3):
        dt, _ = _cpu_plan(1000 + len(times), rows, args.iterations, args.config)
        times.append(dt)
    sims = rows * args.iterations
    sample = f"{len(times)} full planning step(s) of the same workload on 1 core"
    if rows < args.n_parallel:
        sample = f"{len(times)} planning step(s) of the same problem and iterations with {rows} of the " \
                 f"{args.n_parallel} rows per iteration, 1 core"
    return {"value": round(sims * len(times) / sum(times), 1), "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"{sample} ({sum(times):.1f} s; oracle/ numpy port of vecpomdp.plan)"}


def _actions(args) -> int:
    import oracle

    return make_model(oracle, args, 1000).spec.action_count


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import multiprocessing as mp

    cores = os.cpu_count() or 1
    try:  # each process holds one reference tree (~1 GB at the default workload)
        import psutil

        cores = max(1, min(cores, int(psutil.virtual_memory().available // (2 << 30))))
    except ImportError:
        pass
    # keep each step bounded: every core runs one whole planning step of the workload
    ctx = mp.get_context("spawn")
    os.environ["OMP_NUM_THREADS"] = "1"  # inherited by the spawned workers
    with ctx.Pool(cores) as pool:
        for w in range(args.warmup):
            pool.starmap(_cpu_plan, [(2000 + w * cores + c, args.n_parallel, args.iterations, args.config)
                                     for c in range(cores)])
        t0 = time.perf_counter()
        for s in range(args.steps):
            pool.starmap(_cpu_plan, [(3000 + s * cores + c, args.n_parallel, args.iterations, args.config)
                                     for c in range(cores)])
        dt = time.perf_counter() - t0
    sims = args.n_parallel * args.iterations * cores * args.steps
    value = sims / dt
    line = {"metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": 0, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(dt / args.steps * 1e3, 2), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(args, _actions(args)),
            "execution": f"{cores} host processes, each one whole planning step of the workload per step",
            "impl": "reference",
            "cpu_baseline": {"value": round(value, 1), "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": f"each step: {cores} concurrent full planning steps (one per core) of "
                                       f"the workload, oracle/ numpy port of vecpomdp.plan"},
            "e2e": {"value": round(value, 1), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
