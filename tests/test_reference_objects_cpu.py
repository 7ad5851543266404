"""The drop-in boundary with the REAL reference objects (CPU; skipped when
/root/reference is absent, e.g. on the GPU box).

plan() accepts the reference's own model objects (vecpomdp.envs.MarsModel,
TabularModel, NavigationModel, CrowdNavModel; core.py:84-142).  Here their
host-side binding -- the device descriptor (every scalar field and every
constant table uploaded for the kernels) and the packed particle records --
is built with uploads captured on the host, and compared with the product's
own model classes of the same parameters.  Also: a subclass that overrides
the dynamics the device runs is refused instead of silently planning with its
base's device model (envs/_device.py device_model).
"""

import ctypes as C
import os
import sys

import numpy as np
import pytest

import paper_2510_27191_b200 as vp
from paper_2510_27191_b200 import _lib
from paper_2510_27191_b200.envs import _device

REF_SRC = "/root/reference/pkg/src"
needs_ref = pytest.mark.skipif(not os.path.isdir(os.path.join(REF_SRC, "vecpomdp")),
                               reason="reference sources absent (GPU box)")


@pytest.fixture(scope="module")
def ref():
    sys.dont_write_bytecode = True
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import vecpomdp
    import vecpomdp.envs.crowdnav
    import vecpomdp.envs.mars
    import vecpomdp.envs.navigation
    import vecpomdp.envs.tabular

    return vecpomdp


@pytest.fixture
def host_uploads(monkeypatch):
    """DeviceModel.upload records the table on the host and returns a fake pointer."""
    def upload(self, arr):
        a = np.ascontiguousarray(arr)
        self.tables.append(a)
        return 0x1000 * len(self.tables)

    monkeypatch.setattr(_device.DeviceModel, "upload", upload)
    _device._CACHE.clear()
    yield
    _device._CACHE.clear()


def descriptor_fields(dm):
    out = {}
    for name, ctype in _lib.VpModel._fields_:
        v = getattr(dm.desc, name)
        out[name] = list(v) if isinstance(v, C.Array) else v
    return out


def assert_same_binding(ref_model, own_model, states_ref, states_own):
    a, b = _device.device_model(ref_model), _device.device_model(own_model)
    assert a.kind == b.kind
    assert a.state_dtype == b.state_dtype
    assert descriptor_fields(a) == descriptor_fields(b)  # fake pointers agree too: same upload order
    assert len(a.tables) == len(b.tables)
    for x, y in zip(a.tables, b.tables):
        assert x.dtype == y.dtype and x.shape == y.shape
        np.testing.assert_array_equal(x, y)
    ra, rb = a.pack(states_ref), b.pack(states_own)
    assert ra.dtype == rb.dtype
    np.testing.assert_array_equal(ra.view(np.uint8), rb.view(np.uint8))
    # the packed-into-pinned path writes the same bytes
    buf = np.zeros(ra.nbytes + 16, dtype=np.uint8)
    assert a.pack_into(states_ref, buf) == ra.nbytes
    np.testing.assert_array_equal(buf[: ra.nbytes], ra.view(np.uint8).reshape(-1))
    return a


def sampled(model, n, seed, rng_cls):
    return model.sample_initial_states(n, rng_cls.from_seed(seed).derive(3))


@needs_ref
@pytest.mark.parametrize("n,m,s", [(4, 3, 0), (7, 8, 1), (11, 11, 2), (15, 15, 5)])
def test_reference_mars_binds_like_product(ref, host_uploads, n, m, s):
    rm = ref.envs.mars.MarsModel(n, m, layout_seed=s)
    om = vp.MarsModel(n, m, layout_seed=s)
    a = assert_same_binding(rm, om, sampled(rm, 300, s, ref.RowRng), sampled(om, 300, s, vp.RowRng))
    # stepped reference states (departed agents, sampled rocks, terminal rows) pack the same
    # through both bindings
    sr = sampled(rm, 300, s, ref.RowRng)
    acts = np.arange(300) % rm.spec.action_count
    for t in range(4):
        sr = rm.step_batch(sr, acts, ref.RowRng.from_seed(s).derive(9, t).bind(np.arange(300))).next_states
    b = _device.device_model(om)
    np.testing.assert_array_equal(a.pack(sr).view(np.uint8), b.pack(sr).view(np.uint8))


@needs_ref
def test_reference_tiger_binds_like_product(ref, host_uploads):
    rm, om = ref.envs.tabular.tiger_model(), vp.tiger_model()
    assert_same_binding(rm, om, sampled(rm, 200, 4, ref.RowRng), sampled(om, 200, 4, vp.RowRng))


@needs_ref
def test_reference_navigation_binds_like_product(ref, host_uploads):
    rm, om = ref.envs.navigation.NavigationModel(), vp.NavigationModel()
    assert_same_binding(rm, om, sampled(rm, 200, 5, ref.RowRng), sampled(om, 200, 5, vp.RowRng))


@needs_ref
@pytest.mark.parametrize("people,tracked", [(40, 4), (300, 6)])
def test_reference_crowdnav_binds_like_product(ref, host_uploads, people, tracked):
    rm = ref.envs.crowdnav.CrowdNavModel(p_curious=0.3, n_people=people, n_tracked=tracked)
    om = vp.CrowdNavModel(p_curious=0.3, n_people=people, n_tracked=tracked)
    assert_same_binding(rm, om, sampled(rm, 16, 6, ref.RowRng), sampled(om, 16, 6, vp.RowRng))


@needs_ref
def test_reference_plan_inputs_are_accepted(ref):
    """The reference's SolverConfig passes the product's validation unchanged (solver.py:33-60)."""
    from paper_2510_27191_b200.solver import _validate_config

    _validate_config(ref.SolverConfig(n_parallel=64, iterations=3))
    _validate_config(ref.SolverConfig(n_parallel=64, planning_seconds=0.01))


def test_subclass_overriding_dynamics_is_refused(host_uploads):
    class Louder(vp.MarsModel):
        def step_batch(self, states, actions, rng):  # noqa: D401 - different dynamics
            return super().step_batch(states, actions, rng)

    class Hotter(vp.MarsModel):
        def value_heuristic(self, states):
            return super().value_heuristic(states) * 2

    class Sharper(vp.tiger_model().__class__):
        def observation_log_likelihood(self, states, actions, observations):
            return super().observation_log_likelihood(states, actions, observations)

    for cls, args in [(Louder, (5, 4)), (Hotter, (5, 4))]:
        with pytest.raises(TypeError, match="overrides"):
            _device.device_model(cls(*args, layout_seed=1))
    tiger = vp.tiger_model()
    obj = Sharper.__new__(Sharper)
    obj.__dict__.update(tiger.__dict__)
    with pytest.raises(TypeError, match="observation_log_likelihood"):
        _device.device_model(obj)


def test_subclass_with_host_only_changes_is_accepted(host_uploads):
    class Biased(vp.MarsModel):  # another reference policy: initial PSI is computed on the host
        def reference_log_probs(self):
            p = np.full(self.spec.action_count, -10.0)
            p[0] = 0.0
            return p

    dm = _device.device_model(Biased(5, 4, layout_seed=1))
    assert dm.kind == _lib.VP_MODEL_MARS


@needs_ref
def test_reference_subclass_overriding_step_is_refused(ref, host_uploads):
    class Custom(ref.envs.mars.MarsModel):
        def step_batch(self, states, actions, rng):
            return super().step_batch(states, actions, rng)

    with pytest.raises(TypeError, match="step_batch"):
        _device.device_model(Custom(5, 4, layout_seed=1))
