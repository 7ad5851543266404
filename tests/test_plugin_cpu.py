"""The generic ProblemModel plug-in (plugin.py, csrc/vp_plugin.cuh) on the CPU: a user
model's CUDA source compiles into a plug-in build of the library (nvcc cross-compiles
here), the build exports every symbol the header declares and reports the user State
size; model validation and the record StateBatch.  Device parity: test_gpu_plugin.py."""

import ctypes as C

import numpy as np
import pytest

import oracle
import paper_2510_27191_b200 as vp
from paper_2510_27191_b200 import _lib
from paper_2510_27191_b200.envs.plugin_examples import (TAB_STATE, corridor_cuda_model,
                                                        tabular_cuda_model)
from test_boundary_cpu import header_exports


@pytest.fixture(scope="module")
def tiger():
    return tabular_cuda_model(oracle.tiger_model().pomdp)


def test_plugin_library_builds_and_exports(tiger):
    path = vp.compile_plugin(tiger.source)
    assert path == vp.plugin.plugin_path(tiger.source) and path.endswith(".so")
    lib = _lib.load_plugin(path)
    for name in header_exports():
        assert hasattr(lib, name), name
    size = C.c_int32(0)
    assert lib.vp_plugin_info(C.byref(size)) == 1 and size.value == TAB_STATE.itemsize
    assert _lib.load().vp_plugin_info(C.byref(size)) == 0  # the main build carries no user model
    assert tiger.library() is lib


def test_plugin_path_tracks_the_source(tiger):
    assert vp.plugin.plugin_path(tiger.source) != vp.plugin.plugin_path(tiger.source + "\n// edit")
    assert vp.plugin.plugin_path(tiger.source) == vp.plugin.plugin_path(str(tiger.source))


def test_bad_source_fails_loudly():
    bad = vp.CudaModel(vp.ProblemSpec("bad", 2, 2, 0.9, 10), np.dtype([("terminal", "<i4")]),
                       "struct State { int terminal; };  this is not C++")
    with pytest.raises(RuntimeError, match="failed to compile"):
        bad.library()


def test_state_size_mismatch_is_refused(tiger):
    wrong = vp.CudaModel(tiger.spec, np.dtype([("idx", "<i8"), ("terminal", "<i4")]), tiger.source, tiger.params)
    with pytest.raises(ValueError, match="State"):
        wrong.library()


def test_model_validation():
    with pytest.raises(ValueError, match="terminal"):
        vp.CudaModel(vp.ProblemSpec("x", 2, 2, 0.9, 10), np.dtype([("idx", "<i4")]), "")
    spec = vp.ProblemSpec("x", 2, 2, 0.9, 10)
    with pytest.raises(ValueError, match="pointer"):  # a table needs a '<u8' field of its name in params
        vp.CudaModel(spec, TAB_STATE, "", np.zeros((), dtype=[("S", "<i4"), ("cum_t", "<f8")]),
                     tables={"cum_t": np.zeros(4)})
    with pytest.raises(ValueError, match="pointer"):
        vp.CudaModel(spec, TAB_STATE, "", b"\0" * 16, tables={"cum_t": np.zeros(4)})


def test_record_states_and_packing(tiger):
    b = oracle.ParticleBelief.from_model(oracle.tiger_model(), 50, oracle.RowRng.from_seed(2).derive(3))
    rec = tiger.pack(b.states)  # any object with one attribute per field
    np.testing.assert_array_equal(rec["idx"], b.states.idx)
    np.testing.assert_array_equal(rec["terminal"].astype(bool), b.states.terminal)
    s = vp.RecordStates(rec)
    assert len(s) == 50 and len(s.take([1, 3])) == 2
    np.testing.assert_array_equal(s.take([1, 3]).idx, rec["idx"][[1, 3]])
    assert s.terminal.dtype == bool
    with pytest.raises(AttributeError):
        s.nonexistent
    # the host sampler follows the reference's tabular sample_initial_states
    got = tiger.sample_initial_states(64, vp.RowRng.from_seed(5))
    want = oracle.tiger_model().sample_initial_states(64, oracle.RowRng.from_seed(5))
    np.testing.assert_array_equal(got.idx, want.idx)


def test_corridor_compiles():
    m = corridor_cuda_model()
    lib = m.library()
    size = C.c_int32(0)
    assert lib.vp_plugin_info(C.byref(size)) == 1 and size.value == m.state_dtype.itemsize
