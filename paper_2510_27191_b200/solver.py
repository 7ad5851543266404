"""The planning step on the B200: ``plan(belief, model, config, rng) -> PlanOutcome``.

Drop-in for /root/reference/pkg/src/vecpomdp/solver.py:79-113 (same
arguments, same SolverConfig validation and budget semantics, same
PlanOutcome).  Per iteration the host only derives three 64-bit keys
(Appendix A of SURVEY.md) and issues three C-ABI calls; everything else --
root-state draw, D search levels, leaf aggregation, D backup levels -- is
queued on the current CUDA stream without synchronisation.  The host syncs
once at the end (root argmax, 4 bytes) or once per iteration in wall-time
budget mode (the reference checks perf_counter after every iteration).
"""

from __future__ import annotations

import ctypes as C
import os
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .backup import run_backup
from .belief import DeviceBelief, ParticleBelief, sir_update, uniform_cum
from .envs._device import device_model
from .rng import PhiloxRowRng, RowRng, fold, key_of, kind_of
from .search import Workspace, run_search
from .tree import DeviceTree, TreeHandle

NS_ENV, NS_PLAN, NS_SIR, NS_INIT_BELIEF = 0, 1, 2, 3
SITE_DRAW, SITE_SEARCH = 0, 1
_BKEY_MODE_MAX = int(os.environ.get("VP_BKEY_MODE", "1"))  # measurement only


def _torch():
    return _lib.torch_cuda()


@dataclass(frozen=True)
class SolverConfig:
    """Planner parameters (solver.py:33-60); exactly one budget must be set."""

    eta: float = 2.0
    n_parallel: int = 1024
    planning_seconds: float | None = None
    iterations: int | None = None
    d_max_cap: int = 90
    seed: int = 0
    particles: int = 10_000
    max_sir_retries: int = 3

    def __post_init__(self):
        if self.eta <= 0:
            raise ValueError("eta must be positive")
        if self.n_parallel < 1:
            raise ValueError("n_parallel must be >= 1")
        if self.d_max_cap < 1:
            raise ValueError("d_max_cap must be >= 1")
        if (self.planning_seconds is None) == (self.iterations is None):
            raise ValueError("set exactly one of planning_seconds / iterations")
        if self.planning_seconds is not None and self.planning_seconds <= 0:
            raise ValueError("planning_seconds must be positive")
        if self.iterations is not None and self.iterations < 1:
            raise ValueError("iterations must be >= 1")
        if self.particles < 1:
            raise ValueError("particles must be >= 1")


@dataclass
class PlanOutcome:
    chosen_action: int
    iterations_run: int
    final_d_max: int
    tree_stats: dict
    tree: object = field(repr=False, default=None)
    traces: list | None = field(repr=False, default=None)


def initial_prefs(model, eta: float):
    """Zero rows for a uniform reference, else log(pi0)/eta (solver.py:72-76)."""
    ref = np.asarray(model.reference_log_probs(), dtype=np.float64)
    if np.allclose(ref, ref[0]):
        return None
    return ref / eta


def _validate_config(config):
    # accept the reference's SolverConfig (or any duck-typed one) and re-check it
    SolverConfig(config.eta, config.n_parallel, config.planning_seconds, config.iterations, config.d_max_cap,
                 getattr(config, "seed", 0), getattr(config, "particles", 1), getattr(config, "max_sir_retries", 3))


class Planner:
    """Reusable device storage for repeated planning steps (one per stream).

    The reference rebuilds its tree every step (solver.py:91, SPEC tree
    freshness); so does this planner -- but into storage kept from the last
    step, so a closed-loop episode allocates once.
    """

    def __init__(self, precision: str = "fp32", exact: bool = False, mem_fraction: float = 0.6):
        self.precision, self.exact, self.mem_fraction = precision, exact, mem_fraction
        self.tree: DeviceTree | None = None
        self.work: Workspace | None = None
        self.uniform_weights = False  # the last staged belief had weights of exactly 1/m
        self._cap_cache = {}
        self._out = _torch().zeros(1, dtype=_torch().int32, device="cuda")
        self.mode = 1  # vp_plan: 1 CUDA graph of the step's launches (default), 0 direct launches
        self._bufs = {}

    def _capacity(self, n: int, config, A: int):
        """Worst-case node counts for the whole plan, bounded by a memory budget."""
        torch = _torch()
        cap_levels = config.d_max_cap
        if config.iterations is not None:
            total = sum(min(i + 1, cap_levels) for i in range(config.iterations))
            levels = min(config.iterations, cap_levels)
        else:
            total = sum(min(i + 1, cap_levels) for i in range(16))
            levels = cap_levels
        need = 1 + n * total
        # a fixed budget cannot grow inside its CUDA graph: give it up to 85 % of the free HBM
        frac = 0.85 if config.iterations is not None else None
        return min(need, max(self.node_budget(A, fraction=frac), 1 + n * levels)), levels

    def node_budget(self, A: int, fraction: float | None = None, dense: bool = True) -> int:
        """Nodes (belief + action pairs) that fit in mem_fraction of the free HBM: the B columns
        per belief (+ its overlay record), the A columns per action, a 2x-oversized 16-B hash
        slot each, and PSI rows -- one per belief in parity mode, one per 5 actions at most in
        fast mode (only beliefs with more than 4 action children own a dense row; ``dense=False``:
        the pool is grown on demand and budgeted separately, Planner.run)."""
        torch = _torch()
        elem = 4 if self.precision == "fp32" else 8
        per_row = (A + 4) * elem if self.exact else \
            (2 * (A + 4) * elem // (_lib.VP_OVERLAY_SLOTS + 1) if dense else 0) + 8 * elem + 8
        per_pair = per_row + 60 + 52 + 2 * 4 * 16  # hash: 2^k >= 2 cap slots, up to 4 per node
        free, _ = torch.cuda.mem_get_info()
        return int(free * (self.mem_fraction if fraction is None else fraction)) // per_pair

    def prepare(self, model, config, trace: bool = False, device_init: bool = True):
        dm = device_model(model)
        A = model.spec.action_count
        n = config.n_parallel
        ck = (n, config.iterations, config.d_max_cap, A)
        if ck not in self._cap_cache:
            self._cap_cache[ck] = self._capacity(n, config, A)
        cap, levels = self._cap_cache[ck]
        init = dm.init_prefs_cache.get(config.eta, False)
        if init is False:  # the model's reference policy is fixed: once per (model, eta)
            init = dm.init_prefs_cache[config.eta] = initial_prefs(model, config.eta)
        t = self.tree
        if t is None or t.action_count != A or t.precision != self.precision or t.exact != self.exact:
            t = self.tree = DeviceTree(A, init, eta=config.eta, precision=self.precision, exact=self.exact,
                                       cap_beliefs=cap, cap_actions=cap)
        else:
            if t.cap_beliefs < cap:
                t = self.tree = DeviceTree(A, init, eta=config.eta, precision=self.precision, exact=self.exact,
                                           cap_beliefs=cap, cap_actions=cap)
            else:
                t.reset(init, config.eta, device_init=device_init)
        # (belief, action, obs) belief keys when the action and observation codes fit
        mode = 1 if A <= 4096 and model.spec.observation_arity + 1 <= (1 << 20) else 0
        t.set_belief_key_mode(min(mode, _BKEY_MODE_MAX))
        w = self.work
        if w is None or not w.fits(n, levels, dm.state_bytes, trace):
            w = self.work = Workspace(n, levels, dm.state_bytes, trace)
        return dm, t, w

    def _buf(self, name: str, nbytes: int, pinned: bool):
        """Persistent (pinned host or device) byte buffers; stable pointers let
        the captured CUDA graph of a planning step be replayed."""
        torch = _torch()
        t = self._bufs.get(name)
        if t is None or t.numel() < nbytes:
            size = max(nbytes, 64)
            t = torch.empty(size, dtype=torch.uint8, pin_memory=True) if pinned else \
                torch.empty(size, dtype=torch.uint8, device="cuda")
            self._bufs[name] = t
        return t

    def stage_belief(self, dm, belief):
        """Pack the particle StateBatch and its weight CDF into pinned buffers."""
        weights = np.asarray(belief.weights, dtype=np.float64)
        m = len(weights)
        nbytes = m * dm.state_bytes
        hp = self._buf("particles_host", nbytes, True)
        if dm.pack_into(belief.states, hp.numpy()) != nbytes:
            raise ValueError("belief states and weights differ in length")
        # weights of exactly 1/m (every SIR update leaves them so, belief.py:101): their
        # sequential cumsum is the cached device array uniform_cum(m), bit for bit
        self.uniform_weights = bool(m) and not (weights != 1.0 / m).any()
        if not self.uniform_weights:
            hc = self._buf("cumw_host", 8 * m, True)
            np.cumsum(weights, out=hc.numpy()[: 8 * m].view(np.float64))  # sequential fp64 (belief.py:42)
        self._buf("particles_dev", nbytes, False)
        self._buf("cumw_dev", 8 * m, False)
        return m

    def upload_belief(self, dm, belief):
        """Copy the belief to HBM now (for callers that keep it resident).  A
        DeviceBelief is copied device to device into the planner's persistent
        buffers (stable pointers keep the captured CUDA graph valid)."""
        if isinstance(belief, DeviceBelief):
            m, nb = belief.m, belief.records.numel()
            pd, cd = self._buf("particles_dev", nb, False), self._buf("cumw_dev", 8 * m, False)
            pd[:nb].copy_(belief.records)
            cd[: 8 * m].view(_torch().float64).copy_(belief.cumw_dev)
            return pd, cd, m
        m = self.stage_belief(dm, belief)
        nb = m * dm.state_bytes
        pd, cd = self._bufs["particles_dev"], self._bufs["cumw_dev"]
        pd[:nb].copy_(self._bufs["particles_host"][:nb], non_blocking=True)
        if self.uniform_weights:
            cd[: 8 * m].view(_torch().float64).copy_(uniform_cum(m))
        else:
            cd[: 8 * m].copy_(self._bufs["cumw_host"][: 8 * m], non_blocking=True)
        return pd, cd, m

    def plan(self, belief, model, config, rng, *, keep_tree: bool = False, inject_actions=None,
             trace: bool = False) -> PlanOutcome:
        _validate_config(config)
        fixed = config.iterations is not None and inject_actions is None and not trace
        dm, tree, work = self.prepare(model, config, trace, device_init=not fixed)
        dm.desc.rng_kind = kind_of(rng)  # the stream kind of the caller's rng (PhiloxRowRng: fast mode)
        if fixed and not self.fits_fixed(tree, config):
            tree.reset(tree.init_prefs, config.eta)  # device reset for the iterative path
            fixed = False
        if fixed:
            if not tree.exact:  # the fixed graph cannot grow the dense pool: its worst case
                need = 1 + config.n_parallel * sum(min(i + 1, config.d_max_cap) for i in range(config.iterations))
                tree.ensure_dense(need // (_lib.VP_OVERLAY_SLOTS + 1) + 2)
            if isinstance(belief, DeviceBelief):
                _, _, m = self.upload_belief(dm, belief)
                return self.run_fixed(dm, tree, work, m, model.spec, config, key_of(rng), from_host=False,
                                      keep_tree=keep_tree)
            m = self.stage_belief(dm, belief)
            return self.run_fixed(dm, tree, work, m, model.spec, config, key_of(rng), from_host=True,
                                  keep_tree=keep_tree)
        particles, cumw, m = self.upload_belief(dm, belief)
        return self.run(dm, tree, work, particles, cumw, m, model.spec, config, key_of(rng),
                        keep_tree=keep_tree, inject_actions=inject_actions, trace=trace)

    @staticmethod
    def fits_fixed(tree, config) -> bool:
        """Whether the arena holds the worst case of a whole fixed-iteration plan."""
        need = 1 + config.n_parallel * sum(min(i + 1, config.d_max_cap) for i in range(config.iterations))
        return need <= tree.cap_beliefs and need <= tree.cap_actions

    def run_fixed(self, dm, tree, work, m: int, spec, config, key: int, *, from_host: bool = True,
                  keep_tree: bool = False) -> PlanOutcome:
        """A fixed-iteration planning step as ONE vp_plan call (CUDA graph replay).

        ``from_host``: copy the staged pinned belief inside the step (the e2e
        path); otherwise the particles already resident in HBM are used.
        """
        torch = _torch()
        iters = config.iterations
        kh = self._buf("keys_host", 16 * iters, True)
        # fold(fold(key, i), SITE_DRAW / SITE_SEARCH) for every iteration, straight into pinned memory
        _lib.call("vp_plan_keys", C.c_uint64(key), iters, kh.data_ptr())
        kd = self._buf("keys_dev", 16 * iters, False)
        oh = self._buf("out_host", 16, True)
        od = self._buf("out_dev", 16, False)
        if not self.fits_fixed(tree, config):
            raise _lib.CapacityError("tree arena smaller than the plan's worst case; use Planner.run")
        a = _lib.VpPlanArgs()
        a.iterations, a.d_max_cap, a.m, a.mode = iters, config.d_max_cap, m, int(self.mode)
        a.gamma = float(spec.discount)
        a.particles_host = self._bufs["particles_host"].data_ptr() if from_host else None
        a.particles_dev = self._bufs["particles_dev"].data_ptr()
        if from_host and self.uniform_weights:  # no weight bytes to copy: the cached uniform CDF
            a.cumw_host, a.cumw_dev = None, uniform_cum(m).data_ptr()
        else:
            a.cumw_host = self._bufs["cumw_host"].data_ptr() if from_host else None
            a.cumw_dev = self._bufs["cumw_dev"].data_ptr()
        a.keys_host, a.keys_dev = kh.data_ptr(), kd.data_ptr()
        a.out_host, a.out_dev = oh.data_ptr(), od.data_ptr()
        stream = torch.cuda.current_stream()
        dm.call("vp_plan", C.byref(tree.struct), C.byref(dm.desc), C.byref(work.struct), C.byref(a),
                stream.cuda_stream)
        stream.synchronize()
        tree.pass_cursor = iters  # vp_plan numbers its passes 1..iterations on the fresh tree
        work.last_pass = iters
        tree._canon_cache = None
        chosen, nb, na, overflow = (int(v) for v in oh.numpy()[:16].view(np.int32))
        if overflow:
            raise _lib.CapacityError("device tree overflowed its arena during plan()")
        held = tree if keep_tree else TreeHandle(tree)
        if keep_tree:
            self.tree = None
        d_final = min(iters, config.d_max_cap)
        return PlanOutcome(chosen, iters, d_final, {"belief_rows": nb, "action_rows": na}, held, None)

    def run(self, dm, tree, work, particles, cumw, m: int, spec, config, key: int, *, keep_tree: bool = False,
            inject_actions=None, trace: bool = False) -> PlanOutcome:
        """Iterations of one planning step from HBM-resident particles."""
        torch = _torch()
        n = config.n_parallel
        stream = torch.cuda.current_stream().cuda_stream
        ub_b, ub_a = 1, 0
        # fast mode: the dense PSI pool grows on demand (a pass makes at most one dense row per
        # new action), separately from the node columns
        tree.dense_on_demand = not tree.exact
        ub_d = tree.n_dense() if not tree.exact else 0
        d_max, done, last = 1, 0, 0
        # a fixed budget's whole id range (static per-row ids: exact); growth never goes past it
        total = (1 + n * sum(min(i + 1, config.d_max_cap) for i in range(config.iterations))
                 if config.iterations is not None else None)
        stopped = None
        traces = [] if trace else None
        t0 = time.perf_counter()
        while True:
            it_key = fold(key, done)
            if ub_b + n * d_max > tree.cap_beliefs or ub_a + n * d_max > tree.cap_actions:
                nb, na = tree.extent()
                ub_b, ub_a = nb, na
                need_b, need_a = nb + n * d_max, na + n * d_max
                if not done or not (need_b > tree.cap_beliefs or need_a > tree.cap_actions):
                    tree.ensure_capacity(need_b, need_a, limit=total)
                else:
                    # growth allocates the doubled arena beside the old one: stop deepening when
                    # it would not fit in HBM (a memory-bounded budget; the reference would
                    # exhaust host memory the same way, only later)
                    grown = max(tree.cap_beliefs, tree.cap_actions, 16)
                    while grown < max(need_b, need_a):
                        grown *= 2
                    if total is not None:
                        grown = max(min(grown, total), need_b, need_a)
                    budget = self.node_budget(tree.action_count, fraction=0.85, dense=tree.exact)
                    if grown > budget:
                        # near the memory bound: grow by what the next few iterations need
                        # rather than doubling (deeper trees before the bound)
                        grown = max(need_b, need_a) + 4 * n * min(d_max + 4, config.d_max_cap)
                        if total is not None:
                            grown = min(grown, total)
                    if grown > budget:
                        if config.iterations is not None:  # the reference always runs `iterations`
                            raise _lib.CapacityError(
                                f"a {config.iterations}-iteration plan does not fit in HBM after "
                                f"{done} iterations ({nb} beliefs, {na} actions)")
                        stopped = "memory"
                        break
                    tree.ensure_capacity(need_b, need_a, limit=grown)
            if not tree.exact and ub_d + n * d_max > tree.cap_dense:
                ub_d = tree.n_dense()
                need_d = ub_d + n * d_max
                if need_d > tree.cap_dense:
                    grown = max(tree.cap_dense, 16)
                    while grown < need_d:
                        grown *= 2
                    free, _ = torch.cuda.mem_get_info()
                    if done and (grown - tree.cap_dense) * tree.dense_bytes_per_row() > 0.85 * free:
                        if config.iterations is not None:
                            raise _lib.CapacityError(f"the dense PSI pool of a {config.iterations}-iteration plan "
                                                     f"does not fit in HBM after {done} iterations")
                        stopped = "memory"
                        break
                    tree.ensure_dense(need_d)
            inject = None
            if inject_actions is not None:
                arr = np.asarray(inject_actions[done], dtype=np.int32).reshape(d_max, n)
                inject = torch.from_numpy(arr.reshape(-1)).cuda()
            pass_ = tree.next_pass()
            run_search(tree, dm, work, fold(it_key, SITE_SEARCH), 0, d_max, pass_, inject,
                       particles=particles, cumw=cumw, m=m, draw_key=fold(it_key, SITE_DRAW))
            run_backup(tree, work, pass_, spec.discount)
            if trace:
                traces.append({"levels": work.traces(tree, 0, d_max),
                               "leaf_beliefs": tree.to_reference_beliefs(work.leaf_belief).cpu().numpy(),
                               "heuristic_values": work.leaf_value.cpu().numpy().copy()})
            ub_b += n * d_max
            ub_a += n * d_max
            ub_d += n * d_max
            done += 1
            last = d_max
            if config.iterations is not None:
                if done >= config.iterations:
                    break
            else:
                torch.cuda.current_stream().synchronize()
                if time.perf_counter() - t0 >= config.planning_seconds:
                    break
            d_max = min(d_max + 1, config.d_max_cap)
        _lib.call("vp_root_argmax", C.byref(tree.struct), self._out.data_ptr(), stream)
        _lib.call("vp_tree_counts", C.byref(tree.struct), tree._host_counts, stream)  # syncs once
        chosen = int(self._out.item())
        nb, na, overflow = (int(v) for v in tree._host_counts[:3])
        if overflow:
            raise _lib.CapacityError("device tree overflowed its arena during plan()")
        held = tree if keep_tree else TreeHandle(tree)
        if keep_tree:
            self.tree = None  # hand the storage to the caller
        stats = {"belief_rows": nb, "action_rows": na}
        if stopped:
            stats["stopped"] = stopped
        return PlanOutcome(chosen, done, last, stats, held, traces)


_PLANNERS: dict = {}


def get_planner(precision: str = "fp32", exact: bool = False) -> Planner:
    torch = _torch()
    key = (torch.cuda.current_device(), torch.cuda.current_stream().cuda_stream, precision, bool(exact))
    p = _PLANNERS.get(key)
    if p is None:
        p = _PLANNERS[key] = Planner(precision, exact)
    return p


def plan(belief, model, config, rng, *, precision: str = "fp32", exact: bool = False, keep_tree: bool = False,
         inject_actions=None, trace: bool = False) -> PlanOutcome:
    """One planning step on the device (solver.py:79-113).

    ``precision`` selects the PSI storage/compute type: "fp32" (default,
    the fast path) or "fp64"; ``exact=True`` (fp64 only) additionally follows
    numpy's operation order in softmax / LSE so whole-plan trees reproduce the
    reference bit for bit in every integer field.
    """
    return get_planner(precision, exact).plan(belief, model, config, rng, keep_tree=keep_tree,
                                              inject_actions=inject_actions, trace=trace)


@dataclass
class RunRecord:
    run_index: int
    seed: int
    discounted_return: float
    steps: int
    terminal_reason: str
    plan_wall_times: list
    counters: dict
    degenerate_updates: int


def _identity_hooks(model) -> bool:
    """The model keeps the base ProblemModel's reconcile_belief / refresh_executed
    (core.py:119-136), so beliefs never need the host between steps."""
    return all(getattr(type(model), name).__qualname__ == f"ProblemModel.{name}"
               for name in ("reconcile_belief", "refresh_executed"))


def run_episode(model, config, seed: int, run_index: int = 0, *, precision: str = "fp32",
                exact: bool = False, device_belief: bool | None = None, rng_kind: str = "splitmix64") -> RunRecord:
    """Plan / execute / filter loop (solver.py:130-194) around the device plan.

    ``device_belief`` (default: fast mode with identity belief hooks) keeps the
    particles in HBM and runs the SIR update on the device (belief.py:47-102);
    otherwise the update runs through the model's host step_batch, as the
    reference does (the fp64 parity mode reproduces the reference's episodes).
    ``rng_kind="philox"`` draws every stream of the episode from Philox4x32-10
    (the fast mode; statistically, not bitwise, the reference's episodes)."""
    spec = model.spec
    if rng_kind not in ("splitmix64", "philox"):
        raise ValueError(f"rng_kind must be 'splitmix64' or 'philox', got {rng_kind!r}")
    root = (PhiloxRowRng if rng_kind == "philox" else RowRng).from_seed(seed)
    env_rng = root.derive(NS_ENV)
    env_state = model.sample_initial_states(1, env_rng.derive(0))
    belief = ParticleBelief.from_model(model, config.particles, root.derive(NS_INIT_BELIEF))
    belief = ParticleBelief(model.reconcile_belief(belief.states, env_state), belief.weights)
    # a model with its own belief hooks can keep the belief resident when it reconciles on the
    # device (reconcile_device); refresh_executed runs on the single executed state
    device_hooks = hasattr(model, "reconcile_device")
    if device_belief is None:
        device_belief = not exact and (_identity_hooks(model) or device_hooks)
    if device_belief:
        if not (_identity_hooks(model) or device_hooks):
            raise ValueError("device-resident beliefs need identity reconcile_belief / refresh_executed hooks "
                             "or a model.reconcile_device")
        belief = DeviceBelief.from_host(belief, model)
    total, counters, times, degenerate, t, reason = 0.0, {}, [], 0, 0, "truncated"
    while t < spec.max_steps:
        t0 = time.perf_counter()
        outcome = plan(belief, model, config, root.derive(NS_PLAN, t), precision=precision, exact=exact)
        times.append(time.perf_counter() - t0)
        a = outcome.chosen_action
        res = model.step_batch(env_state, np.array([a], dtype=np.int64), env_rng.derive(1 + t).bind([0]))
        total += spec.discount ** t * float(res.rewards[0])
        for k, v in model.step_metrics(env_state, a, res).items():
            counters[k] = counters.get(k, 0.0) + float(v)
        env_state = res.next_states
        t += 1
        if bool(env_state.terminal[0]):
            reason = "terminal"
            break
        # fp32 fast mode also takes the parallel-scan SIR normaliser; fp64 keeps numpy's order
        upd = sir_update(belief, model, a, int(res.observations[0]), root.derive(NS_SIR, t),
                         max_retries=config.max_sir_retries, exact=precision != "fp32")
        degenerate += int(upd.degenerate)
        env_state = model.refresh_executed(env_state)
        if device_belief:
            belief = model.reconcile_device(upd.belief, env_state) if device_hooks else upd.belief
        else:
            belief = ParticleBelief(model.reconcile_belief(upd.belief.states, env_state), upd.belief.weights)
    return RunRecord(run_index, seed, total, t, reason, times, counters, degenerate)
