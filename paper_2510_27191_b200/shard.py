"""Planning step sharded over GPUs (north_star "simulations shard
naturally across the GPUs").

Within one pass of plan() (solver.py:96-111) a row's trajectory -- its actions,
observations, rewards and leaf value -- depends only on the tree as it stood when
the pass began: PSI changes only in the backup, and nodes created during the pass
are lazily initial, so every row that reaches one draws from the initial row.  A
pass therefore splits into

1. **trajectory** (VP_SEARCH_TRAJECTORY): each rank samples and steps its own
   contiguous block of rows, with global row ids so the counter-RNG streams are the
   single-GPU ones, against its replica of the tree, read-only;
2. **exchange**: one all-gather of the trajectories, (2 d + 1) x 8 bytes per row
   (NCCL over NVLink);
3. **insert** (VP_SEARCH_INSERT) + **backup** on every rank's replica: every rank
   replays the same trajectories, so the replicas stay structurally identical and
   the tree equals the single-GPU tree of the same plan (node ids are canonical at
   export, creation keys carry global row ids).

The expensive per-row work (PSI row staging, softmax draws, the generative model,
the RNG) is sharded; node insertion and the backup are replicated.

``world > 1`` with ``group=None`` runs the shards one after another in this process
("virtual ranks"): the exchange is then a concatenation, which is how the sharded
algorithm is tested on one GPU; torch.distributed (NCCL) does the same exchange
across processes.
"""

from __future__ import annotations

import ctypes as C

from . import _lib
from .backup import run_backup
from .rng import fold, key_of, kind_of
from .search import Workspace
from .solver import SITE_DRAW, SITE_SEARCH, Planner, PlanOutcome, _validate_config
from .tree import TreeHandle


def _torch():
    return _lib.torch_cuda()


def shard_rows(n: int, world: int, rank: int) -> tuple:
    """(first global row, row count) of `rank`'s contiguous block; n must divide evenly
    so every rank's trajectory block has the same shape for the all-gather."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world / rank")
    if n % world:
        raise ValueError(f"n_parallel={n} must be a multiple of the number of shards ({world})")
    per = n // world
    return rank * per, per


def pack_trajectories(actions, obs, rewards, leaf, torch):
    """[d, m] i32 actions / obs, [d, m] f64 rewards, [m] f64 leaf values -> one
    [2 d + 1, m] float64 buffer (integer pairs bit-cast), the all-gather payload."""
    d, m = actions.shape
    ao = (actions.to(torch.int64) & 0xFFFFFFFF) | ((obs.to(torch.int64) & 0xFFFFFFFF) << 32)
    return torch.cat([ao.view(torch.float64), rewards.reshape(d, m), leaf.reshape(1, m)], dim=0)


def unpack_trajectories(buf, d: int, torch):
    """Inverse of pack_trajectories on a [2 d + 1, n] buffer."""
    ao = buf[:d].contiguous().view(torch.int64)
    actions = (ao & 0xFFFFFFFF).to(torch.int32)
    obs = ((ao >> 32) & 0xFFFFFFFF).to(torch.int32)
    return actions, obs, buf[d:2 * d].contiguous(), buf[2 * d].contiguous()


def gather_blocks(blocks, torch):
    """Per-shard [2 d + 1, m] buffers (shard = rank order = row order) -> [2 d + 1, G m]."""
    return torch.cat(blocks, dim=1)


def all_gather_blocks(local, world: int, group, torch):
    """torch.distributed all-gather of equal-shape trajectory blocks, rank-major."""
    import torch.distributed as dist

    dev = local.device
    if dev.type == "cuda" and dist.get_backend(group) == "gloo":  # gloo moves host tensors (CPU tests)
        local = local.cpu()
    parts = [torch.empty_like(local) for _ in range(world)]
    dist.all_gather(parts, local.contiguous(), group=group)
    return gather_blocks(parts, torch).to(dev)


class ShardedPlanner(Planner):
    """plan() over `world` shards of the simulation rows; this process is `rank`.

    ``group`` -- a torch.distributed process group (NCCL on GPUs); None with world > 1
    runs every shard in this process (virtual ranks, single-GPU testing).
    """

    def __init__(self, world: int = 1, rank: int = 0, group=None, precision: str = "fp32", exact: bool = False,
                 mem_fraction: float = 0.6):
        super().__init__(precision, exact, mem_fraction)
        self.world, self.rank, self.group = int(world), int(rank), group
        self.distributed = group is not None or (world > 1 and self._dist_ready())
        self._traj_work = None
        self.phase_ms = None  # set to {} to accumulate per-phase device time (CUDA events)

    @staticmethod
    def _dist_ready() -> bool:
        try:
            import torch.distributed as dist

            return dist.is_available() and dist.is_initialized()
        except ImportError:
            return False

    def _shards(self):
        return [self.rank] if self.distributed else list(range(self.world))

    def plan(self, belief, model, config, rng, *, keep_tree: bool = False, resident=None, **_) -> PlanOutcome:
        """``resident`` = (particles, cum_weights, m) already in HBM (from upload_belief):
        skips the belief upload, for device-time measurements."""
        torch = _torch()
        _validate_config(config)
        if config.iterations is None:
            raise ValueError("the sharded planner runs a fixed iteration budget (SolverConfig.iterations)")
        n = config.n_parallel
        _, m_rows = shard_rows(n, self.world, 0)
        dm, tree, work = self.prepare(model, config, device_init=True)
        if not self.fits_fixed(tree, config):
            raise _lib.CapacityError("tree arena smaller than the plan's worst case (sharded plans do not grow)")
        levels = work.max_levels
        tw = self._traj_work
        if tw is None or not tw.fits(m_rows, levels, dm.state_bytes, True):
            tw = self._traj_work = Workspace(m_rows, levels, dm.state_bytes, trace=True)
        particles, cumw, m = resident if resident is not None else self.upload_belief(dm, belief)
        key = key_of(rng)
        dm.desc.rng_kind = kind_of(rng)
        stream = torch.cuda.current_stream().cuda_stream
        d_max = 1
        ev = []

        def mark(name):
            if self.phase_ms is not None:
                e = torch.cuda.Event(enable_timing=True)
                e.record()
                ev.append((name, e))

        for it in range(config.iterations):
            it_key = fold(key, it)
            pass_ = tree.next_pass()
            # 1. trajectories of this process's shard(s), read-only on the replica
            mark("start")
            blocks = []
            for s in self._shards():
                row0, cnt = shard_rows(n, self.world, s)
                args = _lib.VpSearchArgs()
                args.search_key, args.depth0, args.d_max, args.pass_ = fold(it_key, SITE_SEARCH), 0, d_max, pass_
                args.mode, args.row0 = _lib.VP_SEARCH_TRAJECTORY, row0
                args.particles, args.cum_weights, args.m = particles.data_ptr(), cumw.data_ptr(), m
                args.draw_key = fold(it_key, SITE_DRAW)
                dm.call("vp_search", C.byref(tree.struct), C.byref(dm.desc), C.byref(tw.struct), C.byref(args),
                        stream)
                a = tw.trace_action[: d_max * cnt].view(d_max, cnt)
                o = tw.trace_obs[: d_max * cnt].view(d_max, cnt)
                r = tw.trace_reward[: d_max * cnt].view(d_max, cnt)
                blocks.append(pack_trajectories(a, o, r, tw.leaf_value[:cnt], torch))
            mark("trajectory")
            # 2. exchange
            if self.distributed:
                full = all_gather_blocks(blocks[0], self.world, self.group, torch)
            else:
                full = gather_blocks(blocks, torch)
            actions, obs, rewards, leaf = unpack_trajectories(full, d_max, torch)
            mark("exchange")
            # 3. insert every trajectory into the replica, then back up
            args = _lib.VpSearchArgs()
            args.depth0, args.d_max, args.pass_ = 0, d_max, pass_
            args.mode = _lib.VP_SEARCH_INSERT
            args.inject_actions, args.inject_obs = actions.data_ptr(), obs.data_ptr()
            args.inject_reward, args.inject_leaf = rewards.data_ptr(), leaf.data_ptr()
            if pass_ != work.last_pass + 1:
                work.leaf_count.zero_()
            work.last_pass = pass_
            dm.call("vp_search", C.byref(tree.struct), C.byref(dm.desc), C.byref(work.struct), C.byref(args),
                    stream)
            tree._scratch_dirty = True
            mark("insert")
            run_backup(tree, work, pass_, model.spec.discount)
            mark("backup")
            d_max = min(d_max + 1, config.d_max_cap)
        _lib.call("vp_root_argmax", C.byref(tree.struct), self._out.data_ptr(), stream)
        _lib.call("vp_tree_counts", C.byref(tree.struct), tree._host_counts, stream)
        chosen = int(self._out.item())
        for (_, e0), (name, e1) in zip(ev, ev[1:]):
            if name != "start":
                self.phase_ms[name] = self.phase_ms.get(name, 0.0) + e0.elapsed_time(e1)
        nb, na, overflow = (int(v) for v in tree._host_counts[:3])
        if overflow:
            raise _lib.CapacityError("device tree overflowed its arena during plan()")
        held = tree if keep_tree else TreeHandle(tree)
        if keep_tree:
            self.tree = None
        return PlanOutcome(chosen, config.iterations, min(config.iterations, config.d_max_cap),
                           {"belief_rows": nb, "action_rows": na}, held, None)


__all__ = ["ShardedPlanner", "shard_rows", "pack_trajectories", "unpack_trajectories", "gather_blocks",
           "all_gather_blocks"]
