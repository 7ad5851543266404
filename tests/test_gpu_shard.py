"""Sharded planning (paper_2510_27191_b200/shard.py) on one GPU.

The trajectory phase of every shard runs against the replica read-only, the
trajectories are exchanged (here: virtual ranks, concatenated in rank order --
the same bytes NCCL's all-gather delivers across processes) and inserted.  The
result must be the single-GPU planning step: the reference's golden trees in fp64
parity mode, and the fused fp32 path's tree in fp32.
"""

import numpy as np
import pytest

import paper_2510_27191_b200 as vp
from golden_cases import INT_COLUMNS, load, manifest, plan_inputs
import oracle

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["plan_mars7_8_c1", "plan_tiger", "plan_lightdark", "plan_synthetic", "plan_navigation",
                                  "plan_crowdnav40"])
@pytest.mark.parametrize("world", [2, 4])
def test_sharded_fp64_plan_equals_reference_tree(name, world):
    case = manifest()["plans"][name]
    if case["n_parallel"] % world:
        pytest.skip("rows must divide into equal shards")
    g = load(name)
    planner = vp.ShardedPlanner(world=world, precision="fp64", exact=True)
    for run in case["runs"]:
        s = run["seed"]
        om, belief, cfg, rng = plan_inputs(case, s)
        out = planner.plan(belief, om, cfg, rng, keep_tree=True)
        assert out.tree_stats == run["tree_stats"], (name, s)
        t = out.tree.tables()
        for k in INT_COLUMNS:
            np.testing.assert_array_equal(t[k], g[f"s{s}_{k}"].astype(np.int64), err_msg=f"{name} s{s} {k}")
        np.testing.assert_allclose(t["prefs"].sum(axis=1), g[f"s{s}_prefs_row_sum"], rtol=1e-9, atol=1e-8)
        assert out.chosen_action == run["chosen_action"]


@pytest.mark.parametrize("world", [2, 8])
def test_sharded_fp32_equals_fused(world):
    om = oracle.MarsModel(11, 11, layout_seed=5)
    belief = oracle.ParticleBelief.from_model(om, 4000, oracle.RowRng.from_seed(5).derive(3))
    cfg = oracle.SolverConfig(n_parallel=8192, iterations=6)
    rng = oracle.RowRng.from_seed(5).derive(1, 0)
    want = vp.Planner("fp32").plan(belief, om, cfg, rng, keep_tree=True)
    got = vp.ShardedPlanner(world=world, precision="fp32").plan(belief, om, cfg, rng, keep_tree=True)
    assert got.tree_stats == want.tree_stats
    assert got.chosen_action == want.chosen_action
    a, b = got.tree.tables(), want.tree.tables()
    for k in INT_COLUMNS:
        np.testing.assert_array_equal(a[k], b[k], err_msg=k)
    np.testing.assert_allclose(a["prefs"], b["prefs"], rtol=1e-5, atol=1e-5)


def test_sharded_rejects_uneven_rows():
    om = oracle.MarsModel(4, 3, layout_seed=0)
    belief = oracle.ParticleBelief.from_model(om, 100, oracle.RowRng.from_seed(0).derive(3))
    with pytest.raises(ValueError):
        vp.ShardedPlanner(world=3).plan(belief, om, oracle.SolverConfig(n_parallel=100, iterations=2),
                                        oracle.RowRng.from_seed(0))


def _rank_worker(rank, world, port, name, q):
    """One process of a world-2 job on the same GPU: gloo carries the exchange (the code path
    NCCL drives on a multi-GPU box)."""
    import os

    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        case = manifest()["plans"][name]
        g = load(name)
        planner = vp.ShardedPlanner(world=world, rank=rank, group=dist.group.WORLD, precision="fp64", exact=True)
        ok = True
        for run in case["runs"]:
            s = run["seed"]
            om, belief, cfg, rng = plan_inputs(case, s)
            out = planner.plan(belief, om, cfg, rng, keep_tree=True)
            t = out.tree.tables()
            ok &= out.tree_stats == run["tree_stats"] and out.chosen_action == run["chosen_action"]
            ok &= all(np.array_equal(t[k], g[f"s{s}_{k}"].astype(np.int64)) for k in INT_COLUMNS)
            ok &= bool(np.allclose(t["prefs"].sum(axis=1), g[f"s{s}_prefs_row_sum"], rtol=1e-9, atol=1e-8))
        q.put((rank, bool(ok)))
    except Exception as e:  # noqa: BLE001 -- reported to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["plan_mars7_8_c1", "plan_synthetic"])
def test_sharded_planner_two_processes_gloo(name):
    """ShardedPlanner across two real processes (torch.distributed, gloo, 127.0.0.1) on one GPU:
    both replicas must equal the reference's golden trees in fp64 parity mode."""
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    procs = [ctx.Process(target=_rank_worker, args=(r, 2, port, name, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(600)
    res = sorted(q.get() for _ in range(2))
    assert res == [(0, True), (1, True)], res
