"""Campaign harness host logic (bench.py:93-146 mirror): summary statistics and the
JSON-lines layout, on synthetic run records (no GPU)."""

import json

import numpy as np
import pytest

from paper_2510_27191_b200.campaign import CampaignConfig, build_model, config_from_args, build_parser, \
    format_summary, summarize


def _records(returns):
    return [{"type": "run", "run_index": i, "seed": i, "discounted_return": r, "steps": 10 + i,
             "terminal_reason": "terminal" if i % 2 else "truncated", "plan_wall_times": [0.01, 0.03],
             "counters": {"rock_samples": float(i)}, "degenerate_updates": 0} for i, r in enumerate(returns)]


def test_summary_matches_reference_formulas():
    rets = [10.0, 12.5, 7.25, 30.0, -3.0]
    s = summarize(_records(rets))
    arr = np.asarray(rets)
    assert s["n"] == 5 and s["terminal_runs"] == 2
    m = s["metrics"]["discounted_return"]
    assert m["mean"] == pytest.approx(arr.mean())
    assert m["std"] == pytest.approx(arr.std(ddof=1))
    assert m["ci95"] == pytest.approx(1.96 * arr.std(ddof=1) / np.sqrt(5))
    assert s["metrics"]["plan_seconds"]["mean"] == pytest.approx(0.02)
    assert "rock_samples" in s["metrics"]
    assert "terminal runs: 2/5" in format_summary(s)
    with pytest.raises(ValueError):
        summarize([])


def test_single_run_has_zero_ci():
    s = summarize(_records([4.0]))
    assert s["metrics"]["discounted_return"] == {"mean": 4.0, "std": 0.0, "ci95": 0.0}


def test_config_header_and_cli_defaults():
    args = build_parser().parse_args(["--problem", "mars", "--runs", "3", "--planning-time", "0.05"])
    cfg = config_from_args(args)
    assert cfg.solver.n_parallel == 60_000 and cfg.solver.planning_seconds == 0.05  # bench.py:26-31 defaults
    head = cfg.to_dict()
    assert head["type"] == "config" and head["problem_params"] == {"n": 20, "m": 20}
    json.dumps(head)
    with pytest.raises(ValueError):
        CampaignConfig(problem="mars", runs=0)
    # MARS draws a fresh layout per run unless pinned (bench.py:64-72)
    from paper_2510_27191_b200 import MarsModel

    assert np.array_equal(build_model("mars", {"n": 6, "m": 4}, 7).rock_at, MarsModel(6, 4, layout_seed=7).rock_at)
    assert np.array_equal(build_model("mars", {"n": 6, "m": 4, "layout_seed": 1}, 7).rock_at,
                          MarsModel(6, 4, layout_seed=1).rock_at)


def _campaign_worker(rank, world, port, q):
    import os

    import torch.distributed as dist

    import paper_2510_27191_b200.campaign as camp

    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # stand-in episodes (no GPU): the record of run i depends only on i
        camp.play = lambda cfg, i: _records([float(i) * 1.5 - 2.0])[0] | {"run_index": i, "seed": i}
        cfg = CampaignConfig(problem="tiger", runs=7)
        recs, summ = camp.run_campaign(cfg, rank, world)
        q.put((rank, [r["run_index"] for r in recs], summ["metrics"]["discounted_return"]["mean"]))
    finally:
        dist.destroy_process_group()


def test_campaign_runs_split_over_ranks_gloo():
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    procs = [ctx.Process(target=_campaign_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    res = sorted(q.get() for _ in range(2))
    want_mean = np.mean([i * 1.5 - 2.0 for i in range(7)])
    for rank, idx, mean in res:
        assert idx == list(range(7)) and mean == pytest.approx(want_mean)


def test_cli_stream_kind():
    cfg = config_from_args(build_parser().parse_args(["--problem", "tiger", "--iterations", "2", "--rng", "philox"]))
    assert cfg.rng_kind == "philox" and cfg.to_dict()["rng_kind"] == "philox"
    cfg = config_from_args(build_parser().parse_args(["--problem", "tiger", "--iterations", "2"]))
    assert cfg.rng_kind == "splitmix64"
    with pytest.raises(SystemExit):
        build_parser().parse_args(["--problem", "tiger", "--rng", "xorshift"])


def test_cli_plugin_problems():
    """The example CudaModel plug-ins are campaign problems like the built-in ones."""
    for name in ("corridor", "levels"):
        cfg = config_from_args(build_parser().parse_args(["--problem", name, "--iterations", "3"]))
        model = cfg.model_for(0)
        assert type(model).__name__ == "CudaModel" and cfg.solver.n_parallel > 0
