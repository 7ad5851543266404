"""Philox fast-mode streams (north_star: "counter-based Philox RNG") on the CPU.

The oracle's Philox4x32-10 is pinned to the Random123 known-answer vectors
(Salmon et al., SC'11, kat_vectors: philox4x32 10 rounds); the product's host
draws (initial beliefs, episode environment steps) equal the oracle's bit for
bit; derivation keeps the stream kind.  Device parity: tests/test_gpu_philox.py.
"""

import numpy as np
import pytest

import oracle
import paper_2510_27191_b200 as vp
from oracle.rng import PhiloxRowRng, philox4x32_10
from paper_2510_27191_b200.rng import kind_of

# Random123 kat_vectors, philox4x32 with 10 rounds: counter, key -> output
KAT = [
    ((0x00000000, 0x00000000, 0x00000000, 0x00000000), (0x00000000, 0x00000000),
     (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
    ((0xFFFFFFFF, 0xFFFFFFFF, 0xFFFFFFFF, 0xFFFFFFFF), (0xFFFFFFFF, 0xFFFFFFFF),
     (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
    ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
     (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
]


@pytest.mark.parametrize("ctr,key,want", KAT)
def test_oracle_philox_known_answers(ctr, key, want):
    got = philox4x32_10(np.array(ctr), np.array(key))
    assert tuple(int(x) for x in got) == want


def test_product_host_draws_equal_oracle():
    rows = np.array([0, 1, 2, 7, 1 << 33, (1 << 40) + 5, 16383], dtype=np.int64)
    for seed in (0, 1, 12345):
        o = PhiloxRowRng.from_seed(seed).derive(4, 2)
        p = vp.PhiloxRowRng.from_seed(seed).derive(4, 2)
        assert int(o.key) == int(p.key) == int(oracle.RowRng.from_seed(seed).derive(4, 2).key)
        np.testing.assert_array_equal(p.uniform(rows), o.uniform(rows))
        np.testing.assert_array_equal(p.uniform(rows, 5), o.uniform(rows, 5))
        np.testing.assert_array_equal(p.normal(rows), o.normal(rows))
        np.testing.assert_array_equal(p.normal(rows, 3), o.normal(rows, 3))
        assert p.uniform1() == o.uniform1()


def test_stream_kind_survives_derive_and_bind():
    p = vp.PhiloxRowRng.from_seed(3)
    assert type(p.derive(1, 2)) is vp.PhiloxRowRng and type(PhiloxRowRng.from_seed(3).derive(9)) is PhiloxRowRng
    assert kind_of(p) == 1 and kind_of(p.derive(5).bind([0, 1])) == 1
    assert kind_of(vp.RowRng.from_seed(3)) == 0 and kind_of(oracle.RowRng.from_seed(3)) == 0
    assert kind_of(PhiloxRowRng.from_seed(3)) == 1
    b = p.derive(2).bind(np.arange(6))
    np.testing.assert_array_equal(b.uniform(2), p.derive(2).uniform(np.arange(6), 2))


def test_philox_streams_are_uniform_and_differ_from_splitmix():
    rows = np.arange(200_000, dtype=np.int64)
    u = vp.PhiloxRowRng.from_seed(11).derive(1).uniform(rows)
    assert abs(u.mean() - 0.5) < 5e-3 and abs(u.var() - 1.0 / 12.0) < 2e-3
    hist = np.bincount((u * 64).astype(np.int64), minlength=64)
    chi2 = ((hist - len(u) / 64) ** 2 / (len(u) / 64)).sum()
    assert chi2 < 120.0  # 63 dof: p < 1e-5 above ~120
    z = vp.PhiloxRowRng.from_seed(11).derive(2).normal(rows)
    assert abs(z.mean()) < 1e-2 and abs(z.std() - 1.0) < 1e-2
    s = vp.RowRng.from_seed(11).derive(1).uniform(rows)
    assert np.mean(u == s) < 1e-4


def test_oracle_plan_runs_on_philox_streams():
    model = oracle.MarsModel(n=5, m=4, layout_seed=1)
    belief = oracle.ParticleBelief.from_model(model, 500, oracle.RowRng.from_seed(1).derive(3))
    cfg = oracle.SolverConfig(n_parallel=128, iterations=4)
    a = oracle.plan(belief, model, cfg, PhiloxRowRng.from_seed(1).derive(1, 0))
    b = oracle.plan(belief, model, cfg, oracle.RowRng.from_seed(1).derive(1, 0))
    visits = cfg.n_parallel * sum(range(1, cfg.iterations + 1))
    assert a.tree.tables()["action_visits"].sum() == visits == b.tree.tables()["action_visits"].sum()
    ta, tb = a.tree.tables(), b.tree.tables()  # other streams: another tree
    assert a.tree_stats != b.tree_stats or not np.array_equal(ta["action_visits"], tb["action_visits"])


def test_run_episode_rejects_unknown_rng_kind():
    with pytest.raises(ValueError):
        vp.run_episode(vp.MarsModel(5, 4, layout_seed=1), vp.SolverConfig(n_parallel=8, iterations=1), 0,
                       rng_kind="mt19937")
