"""Edge cases of the planning step against the oracle (fp64 parity mode, tree structure bit-exact):
row counts that do not fill warps, a saturated depth cap, other eta, |A| large enough that a
warp stages its PSI rows in several batches, a non-uniform reference policy (init rows),
|A| = 1 or |O| = 1, heavy termination, and non-uniform or one-particle beliefs."""

import numpy as np
import pytest

import oracle
import paper_2510_27191_b200 as vp
from golden_cases import INT_COLUMNS

pytestmark = pytest.mark.gpu


def _compare(om, belief, cfg, rng, rel=1e-9):
    ref = oracle.plan(belief, om, cfg, rng)
    out = vp.plan(belief, om, cfg, rng, precision="fp64", exact=True, keep_tree=True)
    want, got = ref.tree.tables(), out.tree.tables()
    for k in INT_COLUMNS:
        np.testing.assert_array_equal(got[k], want[k], err_msg=k)
    np.testing.assert_allclose(got["prefs"], want["prefs"], rtol=rel, atol=rel)
    assert out.chosen_action == ref.chosen_action
    assert (out.iterations_run, out.final_d_max) == (ref.iterations_run, ref.final_d_max)
    return out


@pytest.mark.parametrize("n_par", [1, 5, 33, 1000])
def test_ragged_row_counts(n_par):
    om = oracle.MarsModel(5, 4, layout_seed=3)
    belief = oracle.ParticleBelief.from_model(om, 300, oracle.RowRng.from_seed(3).derive(3))
    _compare(om, belief, oracle.SolverConfig(n_parallel=n_par, iterations=4), oracle.RowRng.from_seed(3).derive(1, 0))


def test_depth_cap_saturates():
    om = oracle.tiger_model()
    belief = oracle.ParticleBelief.from_model(om, 200, oracle.RowRng.from_seed(4).derive(3))
    out = _compare(om, belief, oracle.SolverConfig(n_parallel=256, iterations=7, d_max_cap=3),
                   oracle.RowRng.from_seed(4).derive(1, 0))
    assert out.final_d_max == 3


@pytest.mark.parametrize("eta", [0.5, 5.0])
def test_other_eta(eta):
    om = oracle.MarsModel(4, 3, layout_seed=5)
    belief = oracle.ParticleBelief.from_model(om, 300, oracle.RowRng.from_seed(5).derive(3))
    _compare(om, belief, oracle.SolverConfig(n_parallel=512, iterations=4, eta=eta),
             oracle.RowRng.from_seed(5).derive(1, 0))


def test_large_action_space_multi_batch_staging():
    # |A| = (5 + 20)^2 = 625: a 32-KB warp stage holds 12 rows, so warps stage in batches
    om = oracle.MarsModel(6, 20, layout_seed=6)
    belief = oracle.ParticleBelief.from_model(om, 400, oracle.RowRng.from_seed(6).derive(3))
    cfg = oracle.SolverConfig(n_parallel=2048, iterations=3)
    rng = oracle.RowRng.from_seed(6).derive(1, 0)
    _compare(om, belief, cfg, rng)
    fast = vp.plan(belief, om, cfg, rng, precision="fp32", keep_tree=True)
    fast.tree.validate()
    assert fast.tree.tables()["action_visits"].sum() == 2048 * 6


class BiasedTiger(oracle.TabularModel):
    """Tiger with a non-uniform reference policy: initial PSI rows log(pi0)/eta (solver.py:72-76)."""

    def reference_log_probs(self):
        return np.log(np.array([0.6, 0.25, 0.15]))


def test_non_uniform_reference_policy():
    base = oracle.tiger_model()
    om = BiasedTiger(base.pomdp)
    belief = oracle.ParticleBelief.from_model(om, 300, oracle.RowRng.from_seed(7).derive(3))
    cfg = oracle.SolverConfig(n_parallel=512, iterations=5)
    rng = oracle.RowRng.from_seed(7).derive(1, 0)
    out = _compare(om, belief, cfg, rng)
    t = out.tree.tables()
    np.testing.assert_allclose(t["prefs"][-1], np.log([0.6, 0.25, 0.15]) / 2.0, rtol=1e-12)  # a lazy row
    fast = vp.plan(belief, om, cfg, rng, precision="fp32", keep_tree=True)
    fast.tree.validate()


@pytest.mark.parametrize("n_actions,n_obs", [(1, 3), (2, 1)])
def test_single_action_or_observation(n_actions, n_obs):
    """|A| = 1 (one-entry softmax rows and CDFs) and |O| = 1 (every action has one child)."""
    om = oracle.SyntheticModel(n_actions=n_actions, n_obs=n_obs, seed=2)
    belief = oracle.ParticleBelief.from_model(om, 200, oracle.RowRng.from_seed(2).derive(3))
    _compare(om, belief, oracle.SolverConfig(n_parallel=300, iterations=5), oracle.RowRng.from_seed(2))


def test_heavy_termination():
    """Half the transitions terminate: rows go absorbing mid-trajectory (terminal observation,
    zero reward) at every level."""
    om = oracle.SyntheticModel(term_per_mille=500, seed=4)
    belief = oracle.ParticleBelief.from_model(om, 500, oracle.RowRng.from_seed(4).derive(3))
    _compare(om, belief, oracle.SolverConfig(n_parallel=512, iterations=6), oracle.RowRng.from_seed(4))


@pytest.mark.parametrize("m", [1, 7])
def test_non_uniform_and_tiny_particle_sets(m):
    """Root draws through the weight CDF: non-uniform weights (the binary-search path, not the
    uniform guess) and a one-particle belief."""
    om = oracle.MarsModel(5, 4, layout_seed=6)
    base = oracle.ParticleBelief.from_model(om, m, oracle.RowRng.from_seed(6).derive(3))
    w = np.arange(1, m + 1, dtype=np.float64)
    belief = oracle.ParticleBelief(base.states, w / w.sum())
    _compare(om, belief, oracle.SolverConfig(n_parallel=256, iterations=5), oracle.RowRng.from_seed(6))
