"""Device SIR update (belief.py:47-102 via vp_sir_weigh / vp_sir_resample) against the
oracle's host SIR: per-particle log-weights, the resampled particle set, retries and
the degenerate path; closed-loop episodes with device-resident beliefs equal the
host-belief episodes."""

import ctypes as C

import numpy as np
import pytest
import torch

import oracle
import paper_2510_27191_b200 as vp
from paper_2510_27191_b200 import _lib
from paper_2510_27191_b200.rng import key_of

pytestmark = pytest.mark.gpu

MODELS = {
    "mars7_8": lambda: (oracle.MarsModel(7, 8, layout_seed=2), vp.MarsModel(7, 8, layout_seed=2)),
    "tiger": lambda: (oracle.tiger_model(), vp.tiger_model()),
    "synthetic": lambda: (oracle.SyntheticModel(seed=4), vp.SyntheticModel(seed=4)),
    "lightdark": lambda: (oracle.LightDarkModel(), vp.LightDarkModel()),
    "navigation": lambda: (oracle.NavigationModel(), vp.NavigationModel()),
    "crowdnav": lambda: (oracle.CrowdNavModel(n_people=50), vp.CrowdNavModel(n_people=50)),
}


def _scenario(kind, seed, m=3000):
    om, pm = MODELS[kind]()
    belief = oracle.ParticleBelief.from_model(om, m, oracle.RowRng.from_seed(seed).derive(3))
    env = om.sample_initial_states(1, oracle.RowRng.from_seed(seed).derive(0, 0))
    rng = oracle.RowRng.from_seed(seed)
    a = int(rng.derive(5).uniform(np.arange(1))[0] * om.spec.action_count)
    res = om.step_batch(env, np.array([a]), oracle.RowRng.from_seed(seed).derive(0, 1).bind([0]))
    return om, pm, belief, a, int(res.observations[0])


def _states_equal(x, y):
    for f in ("x", "y", "rocks", "terminal", "idx", "word", "pos", "occ", "open_gate", "robot", "persons", "curious",
              "tracked", "prev_dist", "last_code"):
        if hasattr(x, f):
            np.testing.assert_array_equal(np.asarray(getattr(x, f)), np.asarray(getattr(y, f)), err_msg=f)


@pytest.mark.parametrize("kind", sorted(MODELS))
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_log_weights_match_oracle(kind, seed):
    om, pm, belief, a, o = _scenario(kind, seed)
    dbel = vp.DeviceBelief.from_host(belief, pm)
    m = dbel.m
    key = oracle.RowRng.from_seed(seed).derive(2, 1).derive(0)
    prop = torch.empty_like(dbel.records)
    logw = torch.empty(m, dtype=torch.float64, device="cuda")
    cum = torch.empty(m, dtype=torch.float64, device="cuda")
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    _lib.call("vp_sir_weigh", C.byref(dbel.dm.desc), dbel.records.data_ptr(), dbel.weights_dev.data_ptr(), m, a, o,
              key_of(key), prop.data_ptr(), logw.data_ptr(), cum.data_ptr(), flag.data_ptr(), 1,
              torch.cuda.current_stream().cuda_stream)
    res = om.step_batch(belief.states, np.full(m, a), key.bind(np.arange(m)))
    with np.errstate(divide="ignore"):
        want = np.log(belief.weights) + om.observation_log_likelihood(res.next_states, a, o)
    got = logw.cpu().numpy()
    np.testing.assert_array_equal(np.isfinite(got), np.isfinite(want))
    fin = np.isfinite(want)
    # compared as probabilities: Light-Dark's bin mass is a difference of two erf values, so a
    # far-tail mass of 1e-12 inherits the ~1e-16 absolute error of erf (math.erf vs CUDA erf)
    np.testing.assert_allclose(np.exp(got[fin]), np.exp(want[fin]), rtol=1e-12, atol=1e-15)
    assert int(flag.item()) == int(fin.any())


@pytest.mark.parametrize("kind", sorted(MODELS))
@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_device_sir_equals_oracle_sir(kind, seed):
    om, pm, belief, a, o = _scenario(kind, seed)
    rng = oracle.RowRng.from_seed(seed).derive(2, 1)
    want = oracle.sir_update(belief, om, a, o, rng, max_retries=3)
    got = vp.sir_update(vp.DeviceBelief.from_host(belief, pm), pm, a, o, rng, max_retries=3)
    assert (got.retries, got.degenerate) == (want.retries, want.degenerate)
    _states_equal(got.belief.states, want.belief.states)
    np.testing.assert_array_equal(got.belief.weights, want.belief.weights)


@pytest.mark.parametrize("kind", sorted(MODELS))
@pytest.mark.parametrize("seed", [0, 1])
def test_fast_sir_normaliser_matches_exact(kind, seed):
    """The fast mode's parallel-scan weight CDF (exact=False) resamples the same particles as
    numpy's serial order except where (j + u0) / m lies within a few ulps of a CDF edge."""
    om, pm, belief, a, o = _scenario(kind, seed)
    rng = oracle.RowRng.from_seed(seed).derive(2, 1)
    want = vp.sir_update(vp.DeviceBelief.from_host(belief, pm), pm, a, o, rng, max_retries=3, exact=True)
    got = vp.sir_update(vp.DeviceBelief.from_host(belief, pm), pm, a, o, rng, max_retries=3, exact=False)
    assert (got.retries, got.degenerate) == (want.retries, want.degenerate)
    rw, rg = want.belief.records.cpu().numpy(), got.belief.records.cpu().numpy()
    differ = np.any(rw.reshape(len(rw), -1) != rg.reshape(len(rg), -1), axis=1)
    assert differ.sum() <= 2, differ.sum()


def test_device_sir_degenerate_observation():
    om, pm = MODELS["mars7_8"]()
    belief = oracle.ParticleBelief.from_model(om, 500, oracle.RowRng.from_seed(9).derive(3))
    # no live particle can emit the terminal observation at the start
    rng = oracle.RowRng.from_seed(9).derive(2, 1)
    want = oracle.sir_update(belief, om, 0, om.spec.terminal_obs, rng, max_retries=2)
    got = vp.sir_update(vp.DeviceBelief.from_host(belief, pm), pm, 0, om.spec.terminal_obs, rng, max_retries=2)
    assert want.degenerate and got.degenerate and got.retries == want.retries == 3
    _states_equal(got.belief.states, want.belief.states)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_closed_loop_device_belief_equals_host_belief(seed):
    model = vp.MarsModel(n=5, m=4, layout_seed=7)
    cfg = vp.SolverConfig(n_parallel=2048, iterations=6, particles=2000)
    a = vp.run_episode(model, cfg, seed=seed, precision="fp64", device_belief=True)
    b = vp.run_episode(model, cfg, seed=seed, precision="fp64", device_belief=False)
    assert a.steps == b.steps and a.terminal_reason == b.terminal_reason
    assert a.discounted_return == pytest.approx(b.discounted_return, abs=1e-12)
