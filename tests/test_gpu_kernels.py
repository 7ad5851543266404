"""GPU parity of the individual device pieces against the oracle / golden
vectors: counter RNG (bit-exact), generative models (integer outputs
bit-exact), LSE and categorical draws."""

import ctypes as C

import numpy as np
import pytest
import torch

import oracle
import paper_2510_27191_b200 as vp
from paper_2510_27191_b200 import _lib
from golden_cases import load

pytestmark = pytest.mark.gpu


def dev_uniform(key, rows, k=0, normal=False):
    r = torch.from_numpy(np.asarray(rows, dtype=np.int64)).cuda()
    out = torch.empty(len(rows) * max(k, 1), dtype=torch.float64, device="cuda")
    _lib.call("vp_rng_normal" if normal else "vp_rng_uniform", int(key), r.data_ptr(), len(rows), k,
              out.data_ptr(), torch.cuda.current_stream().cuda_stream)
    res = out.cpu().numpy()
    return res.reshape(len(rows), k) if k else res


def test_device_rng_bit_exact_vs_reference_golden():
    g = load("rng")
    rows = g["rows"]
    for i, key in enumerate(g["keys"]):
        np.testing.assert_array_equal(dev_uniform(key, rows), g["uniform"][i])
        np.testing.assert_array_equal(dev_uniform(key, rows, 3), g["uniform_k3"][i])
        # Box-Muller goes through log/cos: CUDA and numpy may differ by an ulp
        np.testing.assert_allclose(dev_uniform(key, rows, 2, normal=True), g["normal_k2"][i], rtol=1e-14,
                                   atol=1e-14)


def _random_states(model, kind, n, rng):
    if kind == "mars":
        st = model.sample_initial_states(n, oracle.RowRng.from_seed(7))
        st.x = rng.integers(0, model.n + 1, size=(n, 2))
        st.y = rng.integers(0, model.n, size=(n, 2))
        st.terminal = (st.x[:, 0] == model.n) & (st.x[:, 1] == model.n) | (rng.random(n) < 0.05)
        return st
    if kind == "tiger":
        idx = rng.integers(0, 3, size=n)
        return oracle.TabularStates(idx, idx == 2)
    if kind == "synthetic":
        st = model.sample_initial_states(n, oracle.RowRng.from_seed(7))
        st.terminal = rng.random(n) < 0.05
        return st
    if kind == "navigation":
        st = model.sample_initial_states(n, oracle.RowRng.from_seed(7))
        free = np.flatnonzero(model.kind.reshape(-1) != 1)  # anywhere off the walls, incl. next to the goal
        st.pos = free[rng.integers(0, len(free), size=n)]
        st.terminal = rng.random(n) < 0.05
        return st
    if kind == "crowdnav":
        st = model.sample_initial_states(n, oracle.RowRng.from_seed(7))
        # robots anywhere in the hall (some a step from the exit), so reactions, bumps and exits all occur
        st.robot = rng.uniform(0.0, 1.0, size=(n, 2)) * model.hall
        st.robot[: n // 8, 1] = model.hall[1] - rng.uniform(0.0, 1.5, size=n // 8)
        st.terminal = rng.random(n) < 0.05
        return st
    st = model.sample_initial_states(n, oracle.RowRng.from_seed(7))
    st.x = st.x + rng.normal(size=n) * 4
    st.y = st.y + rng.normal(size=n) * 4
    st.terminal = rng.random(n) < 0.05
    return st


MODELS = [
    ("mars", lambda: (oracle.MarsModel(7, 8, layout_seed=1), vp.MarsModel(7, 8, layout_seed=1))),
    ("mars", lambda: (oracle.MarsModel(15, 15, layout_seed=2), vp.MarsModel(15, 15, layout_seed=2))),
    ("tiger", lambda: (oracle.tiger_model(), vp.tiger_model())),
    ("synthetic", lambda: (oracle.SyntheticModel(seed=3), vp.SyntheticModel(seed=3))),
    ("lightdark", lambda: (oracle.LightDarkModel(), vp.LightDarkModel())),
    ("navigation", lambda: (oracle.NavigationModel(), vp.NavigationModel())),
    ("crowdnav", lambda: (oracle.CrowdNavModel(), vp.CrowdNavModel())),
    ("crowdnav", lambda: (oracle.CrowdNavModel(n_people=17, n_tracked=8, p_curious=0.3),
                          vp.CrowdNavModel(n_people=17, n_tracked=8, p_curious=0.3))),
]
CROWD_FIELDS = ("robot", "persons", "curious", "tracked", "prev_dist", "last_code")


@pytest.mark.parametrize("kind,make", MODELS)
def test_device_model_step_matches_oracle(kind, make):
    om, dm = make()
    rng = np.random.default_rng(11)
    n = 1024 if kind == "crowdnav" else 4096
    st = _random_states(om, kind, n, rng)
    acts = rng.integers(0, om.spec.action_count, size=n)
    key = oracle.RowRng.from_seed(5).derive(2, 1)
    bound_rows = np.arange(1000, 1000 + n)
    want = om.step_batch(st, acts, key.bind(bound_rows))
    got = dm.step_batch(st, acts, vp.RowRng(key.key).bind(bound_rows))
    np.testing.assert_array_equal(got.observations, want.observations)
    np.testing.assert_array_equal(got.rewards, want.rewards)
    np.testing.assert_array_equal(got.next_states.terminal, want.next_states.terminal)
    for f in ("x", "y", "rocks", "idx", "word", "pos", "occ", "open_gate") + CROWD_FIELDS:
        if hasattr(want.next_states, f):
            np.testing.assert_array_equal(getattr(got.next_states, f), getattr(want.next_states, f), err_msg=f)
    h_want = om.value_heuristic(want.next_states)
    h_got = dm.value_heuristic(want.next_states)
    np.testing.assert_allclose(h_got, h_want, rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("tag,people,n,steps", [("p40", 40, 96, 6), ("p300", 300, 8, 3)])
def test_device_crowdnav_steps_equal_reference_golden(tag, people, n, steps):
    """The device CrowdNav step against vectors made by the REAL reference (crowdnav.py:116-197)."""
    g = load("crowd_steps")
    m = vp.CrowdNavModel(n_people=people)
    st = m.sample_initial_states(n, vp.RowRng.from_seed(31))
    for t in range(steps):
        res = m.step_batch(st, g[f"{tag}_a{t}"], vp.RowRng.from_seed(50 + t).bind(np.arange(n)))
        for f in ("robot", "prev_dist", "last_code", "terminal"):
            np.testing.assert_array_equal(getattr(res.next_states, f), g[f"{tag}_{f}{t + 1}"], err_msg=f)
        np.testing.assert_array_equal(res.observations, g[f"{tag}_obs{t + 1}"])
        np.testing.assert_array_equal(res.rewards, g[f"{tag}_rew{t + 1}"])
        np.testing.assert_array_equal(m.value_heuristic(res.next_states), g[f"{tag}_h{t + 1}"])
        st = res.next_states
    np.testing.assert_array_equal(st.persons, g[f"{tag}_persons_end"])


def test_device_lse_matches_oracle():
    g = np.random.default_rng(3)
    for width in (1, 3, 7, 9, 128, 169, 256, 400, 625):
        rows = g.normal(size=(64, width)) * 4.0
        want = oracle.log_sum_exp_rows(rows, 2.0)
        ex = vp.log_sum_exp_rows(rows, 2.0, precision="fp64", exact=True)
        np.testing.assert_allclose(ex, want, rtol=1e-14, atol=1e-14)
        fast64 = vp.log_sum_exp_rows(rows, 2.0, precision="fp64", exact=False)
        np.testing.assert_allclose(fast64, want, rtol=1e-13, atol=1e-13)
        f32 = vp.log_sum_exp_rows(rows.astype(np.float32).astype(np.float64), 2.0, precision="fp32")
        scale = np.maximum(np.abs(want), np.abs(rows).max(axis=1))
        assert np.all(np.abs(f32 - want) <= 1e-5 * scale + 1e-6)
    # SPEC.md:285-288 examples
    assert abs(vp.log_sum_exp_rows([[3.0] * 4], 2.0)[0] - (3.0 + np.log(4) / 2)) < 1e-12
    assert abs(vp.log_sum_exp_rows([[1.0, 2.0]], 1.0)[0] - 2.31326) < 1e-5


def test_device_sampling_exact_mode_matches_numpy_order():
    g = np.random.default_rng(5)
    for width in (2, 9, 16, 169, 256, 400):
        rows = g.normal(size=(40, width)) * 2.0
        groups = g.integers(0, 40, size=5000)
        u = g.random(5000)
        pol = oracle.softmax_rows(rows, 2.0)
        # numpy reference: per-row inverse CDF of the sequential cumsum (single-group form)
        cum = np.cumsum(pol, axis=1)
        want = np.array([min(np.searchsorted(cum[gg], uu, side="right"), width - 1) for gg, uu in zip(groups, u)])
        got = vp.sample_actions(rows, u, groups, eta=2.0, precision="fp64", exact=True)
        # exp may differ from numpy's SIMD exp by one ulp: allow only draws within 1e-12 of a CDF edge
        bad = np.flatnonzero(got != want)
        for i in bad:
            assert np.min(np.abs(cum[groups[i]] - u[i])) < 1e-12
        assert len(bad) <= 2


def test_device_sampling_fast_mode_distribution():
    g = np.random.default_rng(8)
    width = 169
    rows = g.normal(size=(3, width))
    groups = np.repeat(np.arange(3), 40000)
    u = g.random(len(groups))
    for prec in ("fp32", "fp64"):
        got = vp.sample_actions(rows, u, groups, eta=2.0, precision=prec, exact=False)
        pol = oracle.softmax_rows(rows, 2.0)
        cum = np.cumsum(pol, axis=1)
        want = np.array([min(np.searchsorted(cum[gg], uu, side="right"), width - 1) for gg, uu in zip(groups, u)])
        # identical except for draws within fp32 rounding of a CDF edge
        mism = np.flatnonzero(got != want)
        for i in mism:
            assert np.min(np.abs(cum[groups[i]] - u[i])) < 5e-5
        assert len(mism) < 0.002 * len(u)
    # degenerate row (1, 0, 0) -> action 0 always
    deg = np.array([[0.0, -1e4, -1e4]])
    assert set(vp.sample_actions(deg, g.random(1000), eta=1.0, precision="fp32", exact=False)) == {0}
