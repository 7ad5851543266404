"""Host side of the sharded planning step on CPU: row partition, the trajectory
payload codec and the all-gather exchange over torch.distributed (gloo, world
size 2, 127.0.0.1) -- the same code paths NCCL drives on GPUs."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2510_27191_b200.shard import all_gather_blocks, gather_blocks, pack_trajectories, shard_rows, \
    unpack_trajectories


def _block(row0, cnt, d):
    """Deterministic stand-in trajectories of global rows row0..row0+cnt-1."""
    rows = torch.arange(row0, row0 + cnt, dtype=torch.int64)
    lv = torch.arange(d, dtype=torch.int64)[:, None]
    actions = ((rows[None, :] * 7 + lv * 3) % 256).to(torch.int32)
    obs = ((rows[None, :] * 5 + lv) % 9 + (lv == 0) * 0x7FFFFFF0).to(torch.int32)
    rewards = (rows[None, :] * 0.25 - lv * 1.5).to(torch.float64)
    leaf = torch.sin(rows.to(torch.float64))
    return actions, obs, rewards, leaf


def test_shard_rows_partition():
    n, world = 4096, 8
    blocks = [shard_rows(n, world, r) for r in range(world)]
    assert blocks[0] == (0, 512) and blocks[-1] == (3584, 512)
    assert sum(c for _, c in blocks) == n
    with pytest.raises(ValueError):
        shard_rows(100, 3, 0)
    with pytest.raises(ValueError):
        shard_rows(100, 2, 2)


def test_payload_roundtrip_and_concatenation():
    d, n, world = 5, 64, 4
    parts = []
    for r in range(world):
        row0, cnt = shard_rows(n, world, r)
        parts.append(pack_trajectories(*_block(row0, cnt, d), torch))
    full = unpack_trajectories(gather_blocks(parts, torch), d, torch)
    want = _block(0, n, d)
    for got, ref in zip(full, want):
        assert torch.equal(got, ref)


def _worker(rank, world, port, d, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        row0, cnt = shard_rows(n, world, rank)
        local = pack_trajectories(*_block(row0, cnt, d), torch)
        full = unpack_trajectories(all_gather_blocks(local, world, None, torch), d, torch)
        want = _block(0, n, d)
        q.put((rank, all(torch.equal(a, b) for a, b in zip(full, want))))
    finally:
        dist.destroy_process_group()


def test_all_gather_exchange_gloo_world2():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, 4, 96, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    res = sorted(q.get() for _ in range(2))
    assert res == [(0, True), (1, True)]
