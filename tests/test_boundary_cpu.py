"""CPU checks of the drop-in boundary: the C-ABI library loads and exports
every symbol include/vpb200.h declares, the ctypes mirrors match the C
layout, and the host-side pieces (key derivation, model layouts, packing,
config validation) agree with the oracle.  No CUDA call is made here."""

import os
import re

import numpy as np
import pytest

import oracle
import paper_2510_27191_b200 as vp
from paper_2510_27191_b200 import _lib
from paper_2510_27191_b200.envs import _device
from paper_2510_27191_b200.rng import fold, mix64_int

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_exports():
    txt = open(os.path.join(REPO, "include", "vpb200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int32_t|int64_t|const char\*)\s+(vp_\w+)\s*\(", txt, flags=re.M)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    declared = header_exports()
    assert len(declared) >= 15
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(_lib.EXPORTED_SYMBOLS) == declared
    assert lib.vp_abi_version() == _lib.ABI_VERSION


def test_ctypes_layout_matches_c():
    assert _lib.layout_mismatches() == []


def test_status_mapping():
    with pytest.raises(ValueError):
        _lib.check(_lib.VP_ERR_INVALID, "x")
    with pytest.raises(_lib.CapacityError):
        _lib.check(_lib.VP_ERR_CAPACITY, "x")
    with pytest.raises(TypeError):
        _lib.check(_lib.VP_ERR_MODEL, "x")
    _lib.check(_lib.VP_OK)


def test_host_key_derivation_matches_oracle():
    for seed in [0, 1, 12345, 2**63 + 11]:
        a = vp.RowRng.from_seed(seed)
        b = oracle.RowRng.from_seed(seed)
        assert int(a.key) == int(b.key)
        for path in [(1, 0), (3,), (2, 7, 9)]:
            assert int(a.derive(*path).key) == int(b.derive(*path).key)
        k = int(b.key)
        assert fold(k, 5) == int(oracle.rng.fold_word(b.key, 5))
        rows = np.arange(100)
        np.testing.assert_array_equal(a.uniform(rows, 3), b.uniform(rows, 3))
        np.testing.assert_array_equal(a.normal(rows), b.normal(rows))
    assert mix64_int(0) == 0


def test_product_models_match_oracle_host_parts():
    for n, m, s in [(4, 3, 0), (7, 8, 1), (11, 11, 2), (15, 15, 5)]:
        a, b = vp.MarsModel(n, m, layout_seed=s), oracle.MarsModel(n, m, layout_seed=s)
        np.testing.assert_array_equal(a.rock_x, b.rock_x)
        np.testing.assert_array_equal(a.rock_y, b.rock_y)
        assert a.spec.action_count == b.spec.action_count
        sa = a.sample_initial_states(50, vp.RowRng.from_seed(s).derive(3))
        sb = b.sample_initial_states(50, oracle.RowRng.from_seed(s).derive(3))
        np.testing.assert_array_equal(sa.rocks, sb.rocks)
    sy, so = vp.SyntheticModel(seed=4), oracle.SyntheticModel(seed=4)
    np.testing.assert_array_equal(sy.sample_initial_states(20, vp.RowRng.from_seed(1)).word,
                                  so.sample_initial_states(20, oracle.RowRng.from_seed(1)).word)
    la, lb = vp.LightDarkModel(), oracle.LightDarkModel()
    np.testing.assert_array_equal(la.sample_initial_states(20, vp.RowRng.from_seed(1)).x,
                                  lb.sample_initial_states(20, oracle.RowRng.from_seed(1)).x)
    ta, tb = vp.tiger_model(), oracle.tiger_model()
    np.testing.assert_array_equal(ta.pomdp.transitions, tb.pomdp.transitions)
    np.testing.assert_array_equal(ta.pomdp.observations, tb.pomdp.observations)
    np.testing.assert_array_equal(ta.pomdp.rewards, tb.pomdp.rewards)


def test_state_packing_roundtrip():
    m = vp.MarsModel(7, 8, layout_seed=0)
    st = m.sample_initial_states(33, vp.RowRng.from_seed(2))
    st.x[3, 1] = 7
    st.terminal[5] = True
    rec = _device.mars_pack(st)
    assert rec.dtype.itemsize == 16
    back = m._unpack(rec)
    np.testing.assert_array_equal(back.x, st.x)
    np.testing.assert_array_equal(back.y, st.y)
    np.testing.assert_array_equal(back.rocks, st.rocks)
    np.testing.assert_array_equal(back.terminal, st.terminal)
    assert _device.TAB_DTYPE.itemsize == 8 and _device.SYN_DTYPE.itemsize == 16 and _device.LD_DTYPE.itemsize == 24


@pytest.mark.parametrize("native", [True, False])
@pytest.mark.parametrize("n,m", [(4, 3), (11, 11), (20, 30), (20, 60), (20, 64)])
def test_mars_word_packing_equals_field_layout(n, m, native):
    """mars_pack_into writes {x0,y0,x1,y1,terminal,rock bits} as two 64-bit words; every field
    must land where MARS_DTYPE (and the kernel's MarsState) says, for every rock-count path --
    through the library's host packer (vp_pack_mars_states, int64 / bool C-contiguous columns,
    the reference's own dtypes) and through the numpy path (any other dtypes)."""
    model = oracle.MarsModel(n, m, layout_seed=1)
    st = model.sample_initial_states(300, oracle.RowRng.from_seed(3))
    g = np.random.default_rng(0)
    st.x = g.integers(0, n + 1, size=(300, 2)).astype(np.int64 if native else np.int32)
    st.y = g.integers(0, n, size=(300, 2))
    st.terminal = g.random(300) < 0.3
    rec = _device.mars_pack(st)
    assert rec.dtype == _device.MARS_DTYPE
    for i, f in enumerate(("x0", "x1")):
        np.testing.assert_array_equal(rec[f], st.x[:, i])
    for i, f in enumerate(("y0", "y1")):
        np.testing.assert_array_equal(rec[f], st.y[:, i])
    np.testing.assert_array_equal(rec["term"], st.terminal)
    want = (st.rocks.astype(np.uint64) << np.arange(m, dtype=np.uint64)).sum(axis=1, dtype=np.uint64)
    np.testing.assert_array_equal(rec["rocks"], want)
    buf = np.full(16 * 300 + 40, 0xAB, dtype=np.uint8)  # dirty pinned-buffer stand-in
    assert _device.mars_pack_into(st, buf) == 16 * 300
    np.testing.assert_array_equal(buf[: 16 * 300], rec.view(np.uint8))
    assert (buf[16 * 300:] == 0xAB).all()


def test_small_record_packers_match_their_layouts():
    """Navigation / Synthetic / Light-Dark / Tabular records: every field where the dtype (and the
    kernel's struct) puts it, Navigation through its unpacker round trip."""
    g = np.random.default_rng(4)
    nav = oracle.NavigationModel()
    st = nav.sample_initial_states(64, oracle.RowRng.from_seed(2))
    st.terminal = g.random(64) < 0.3
    rec = _device.nav_pack(st)
    assert rec.dtype.itemsize == 24
    back = _device.nav_unpacker(nav.n_unknown, oracle.NavStates)(rec)
    for f in ("pos", "occ", "open_gate", "terminal"):
        np.testing.assert_array_equal(getattr(back, f), getattr(st, f), err_msg=f)
    sy = oracle.SyntheticModel(seed=1).sample_initial_states(50, oracle.RowRng.from_seed(3))
    sy.terminal = g.random(50) < 0.5
    r = _device.syn_pack(sy)
    np.testing.assert_array_equal(r["word"], sy.word)
    np.testing.assert_array_equal(r["term"].astype(bool), sy.terminal)
    ld = oracle.LightDarkModel().sample_initial_states(50, oracle.RowRng.from_seed(3))
    r = _device.ld_pack(ld)
    np.testing.assert_array_equal(r["x"], ld.x)
    np.testing.assert_array_equal(r["y"], ld.y)
    tb = oracle.TabularStates(g.integers(0, 3, size=40), g.random(40) < 0.5)
    r = _device.tab_pack(tb)
    np.testing.assert_array_equal(r["idx"], tb.idx)
    np.testing.assert_array_equal(r["term"].astype(bool), tb.terminal)


@pytest.mark.parametrize("people,tracked", [(300, 6), (17, 8), (320, 1)])
def test_crowdnav_record_roundtrip(people, tracked):
    model = oracle.CrowdNavModel(n_people=people, n_tracked=tracked, p_curious=0.4)
    st = model.sample_initial_states(40, oracle.RowRng.from_seed(2))
    st.terminal[3] = True
    st.last_code[:] = np.arange(40) % (2 ** tracked)
    rec = _device.crowd_pack(st)
    assert rec.dtype.itemsize == _lib.CROWD_STATE_BYTES
    back = _device.crowd_unpacker(people, tracked, oracle.CrowdStates)(rec)
    for f in ("robot", "persons", "curious", "tracked", "prev_dist", "last_code", "terminal"):
        np.testing.assert_array_equal(getattr(back, f), getattr(st, f), err_msg=f)


def test_crowdnav_capacity_is_checked():
    with pytest.raises(ValueError):
        _device.crowdnav_descriptor(oracle.CrowdNavModel(n_people=321))
    with pytest.raises(ValueError):
        _device.crowdnav_descriptor(oracle.CrowdNavModel(n_people=30, n_tracked=9))


def test_solver_config_contract():
    with pytest.raises(ValueError):
        vp.SolverConfig(iterations=None)
    with pytest.raises(ValueError):
        vp.SolverConfig(iterations=3, planning_seconds=1.0)
    with pytest.raises(ValueError):
        vp.SolverConfig(iterations=3, eta=0.0)
    with pytest.raises(ValueError):
        vp.SolverConfig(iterations=0)
    assert vp.SolverConfig(iterations=2).n_parallel == 1024


def test_initial_prefs_rule():
    from paper_2510_27191_b200.solver import initial_prefs

    assert initial_prefs(vp.MarsModel(4, 3), 2.0) is None

    class Skewed(vp.MarsModel):
        def reference_log_probs(self):
            p = np.linspace(1, 2, self.spec.action_count)
            return np.log(p / p.sum())

    ip = initial_prefs(Skewed(4, 3), 2.0)
    assert ip.shape == (64,) and np.all(np.isfinite(ip))


def test_product_never_imports_oracle():
    pkg = os.path.join(REPO, "paper_2510_27191_b200")
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(root, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f


def test_plan_keys_host_function_matches_fold():
    """vp_plan_keys (the library's host key schedule of a fixed-iteration plan) equals
    fold(fold(key, i), site) for the draw (0) and search (1) sites (solver.py:97-102)."""
    import ctypes as C

    for key in (0, 1, 123456789, (1 << 64) - 1):
        out = np.zeros(2 * 13, dtype=np.uint64)
        assert _lib.load().vp_plan_keys(C.c_uint64(key), 13, out.ctypes.data) == 0
        want = [fold(fold(key, i), s) for i in range(13) for s in (0, 1)]
        np.testing.assert_array_equal(out, np.array(want, dtype=np.uint64))


# vecpomdp/__init__.py:10-48 __all__ (the reference's public names)
REFERENCE_ALL = ['BeliefTree', 'BoundRng', 'LeafResult', 'LevelValues', 'ParticleBelief', 'PlanOutcome', 'ProblemModel', 'ProblemSpec', 'RowRng', 'RunRecord', 'SearchBatch', 'SirUpdate', 'SolverConfig', 'StateBatch', 'StepResult', 'action_q_values', 'aggregate_leaves', 'backup', 'init_tree', 'log_sum_exp_rows', 'match_or_append_pairs', 'plan', 'run_episode', 'sample_actions', 'search', 'sir_update', 'softmax_rows', 'systematic_resample']


def test_every_reference_public_name_is_exported():
    missing = [n for n in REFERENCE_ALL if not hasattr(vp, n) or n not in vp.__all__]
    assert missing == []
    envs = ["CrowdNavModel", "MarsModel", "NavigationModel", "TabularModel", "TabularPOMDP", "tiger_model",
            "problem_from_config"]  # vecpomdp/envs/__init__.py __all__
    assert [n for n in envs if not hasattr(vp.envs, n)] == []
