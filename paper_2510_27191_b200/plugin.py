"""User problem models on the device: the generic ``ProblemModel`` plug-in.

The reference plans ANY ``ProblemModel`` subclass (core.py:84-142): ``step_batch``,
``value_heuristic`` and ``observation_log_likelihood`` are numpy there.  The device
cannot call Python once per simulated row, so a user model states those three as
CUDA device functions (the contract is in csrc/vp_plugin.cuh) and ``CudaModel``
compiles them INTO a build of this library: nvcc with ``-DVP_PLUGIN_SOURCE=<file>
-DVP_PLUGIN_ONLY`` instantiates the search, backup, SIR and plan kernels for the
user model exactly as for the built-in ones (no interpretation, no callbacks), into
``plugins/libvpb200_<hash>.so`` in-tree, cached by the hash of the model source and
the library sources.  ``plan()``, ``search()``, ``run_episode()`` and the device SIR
route that model's calls to its library; the tree and backup entry points are
model-independent and stay on the main library.

    class Corridor(vp.CudaModel):
        ...
    model = vp.CudaModel(spec, state_dtype, source, params, initial_states=sampler)
    vp.plan(belief, model, SolverConfig(...), rng)

The source is compiled inside ``namespace vp_user`` and must not ``#include`` anything
(fixed-width integer types and CUDA math are in scope).  ``state_dtype`` is a numpy
structured dtype laid out like the source's ``State``
struct and must have a ``terminal`` field; ``params`` (a structured scalar or raw
bytes) is laid out like ``Params``.  There is no CPU fallback: without nvcc (the
first use of a new source compiles) or a GPU the calls raise.
"""

from __future__ import annotations

import ctypes as C
import hashlib
import os
import shutil
import subprocess
import threading

import numpy as np

from . import _lib
from .core import ProblemModel

_HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(_HERE, "csrc")
PLUGIN_DIR = os.environ.get("VP_PLUGIN_DIR") or os.path.join(_HERE, "plugins")
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17", "-fmad=false",
              "-Xcompiler", "-fPIC,-O2", "--expt-relaxed-constexpr", "-shared"]
_LOCKS_GUARD = threading.Lock()
_BUILD_LOCKS: dict = {}  # one lock per plug-in path: different plug-ins build in parallel


def _library_digest() -> str:
    h = hashlib.sha256()
    for name in sorted(os.listdir(CSRC)):
        with open(os.path.join(CSRC, name), "rb") as f:
            h.update(name.encode() + f.read())
    with open(os.path.join(_HERE, "..", "include", "vpb200.h"), "rb") as f:
        h.update(f.read())
    h.update(" ".join(NVCC_FLAGS).encode())
    return h.hexdigest()


def plugin_path(source: str) -> str:
    """Where the plug-in library of ``source`` lives (whether or not it is built yet)."""
    tag = hashlib.sha256((_library_digest() + "\0" + source).encode()).hexdigest()[:20]
    return os.path.join(PLUGIN_DIR, f"libvpb200_{tag}.so")


def compile_plugin(source: str, *, verbose: bool = False) -> str:
    """Build (once) the library carrying the model ``source``; returns its path."""
    path = plugin_path(source)
    if os.path.exists(path):
        return path
    with _LOCKS_GUARD:
        lock = _BUILD_LOCKS.setdefault(path, threading.Lock())
    with lock:
        if os.path.exists(path):
            return path
        nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
        if not os.path.exists(nvcc):
            raise _lib.LibraryMissing("compiling a CudaModel needs nvcc (CUDA 12.9); there is no CPU fallback")
        os.makedirs(PLUGIN_DIR, exist_ok=True)
        # per-process temporaries, published with an atomic rename: concurrent builders of the
        # same source (e.g. torchrun ranks) never read a half-written file
        stem = f"{path[:-3]}.{os.getpid()}"
        src = stem + ".cuh"
        with open(src, "w") as f:
            f.write(source)
        tmp = stem + ".tmp.so"
        cmd = [nvcc, *NVCC_FLAGS, f'-DVP_PLUGIN_SOURCE="{src}"', "-DVP_PLUGIN_ONLY", "-o", tmp,
               os.path.join(CSRC, "vp_kernels.cu")]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            os.remove(src)
            raise RuntimeError(f"CudaModel source failed to compile:\n{res.stderr[-4000:]}")
        if verbose:
            print(res.stderr)
        os.replace(src, path[:-3] + ".cuh")  # kept beside the library (its -lineinfo source)
        os.replace(tmp, path)
    return path


class RecordStates:
    """A StateBatch (core.py:52-62) of packed device records: a structured numpy array
    with one row per state; every field is readable as an attribute (``.terminal`` as bool)."""

    def __init__(self, records: np.ndarray):
        self.records = np.ascontiguousarray(records)

    def __len__(self) -> int:
        return len(self.records)

    def take(self, indices) -> "RecordStates":
        return RecordStates(self.records[np.asarray(indices, dtype=np.int64)])

    @property
    def terminal(self) -> np.ndarray:
        return self.records["terminal"].astype(bool)

    def __getattr__(self, name):
        rec = self.__dict__.get("records")
        if rec is not None and rec.dtype.names and name in rec.dtype.names:
            return rec[name]
        raise AttributeError(name)


class CudaModel(ProblemModel):
    """A ProblemModel whose dynamics are CUDA device functions (csrc/vp_plugin.cuh).

    ``spec``: ProblemSpec.  ``state_dtype``: structured dtype of the ``State`` record
    (with a ``terminal`` field).  ``source``: the CUDA definitions of ``Params``, ``State``,
    ``step``, ``heuristic``, ``obs_log_likelihood``.  ``params``: the ``Params`` bytes
    (numpy structured scalar / array / bytes).  ``initial_states(n, rng)``: host sampler
    returning a structured array of ``state_dtype`` (sample_initial_states, core.py:101).
    ``reference_log_probs``: optional log pi0 per action (default uniform).
    ``tables``: {field: numpy array} uploaded to HBM once per model; the device address of each
    is written into the ``Params`` field of that name (a pointer in the CUDA struct, a ``<u8``
    field of a structured ``params``) -- constant tables of any size (maps, matrices).
    """

    def __init__(self, spec, state_dtype, source: str, params=None, initial_states=None,
                 reference_log_probs=None, tables=None):
        self.spec = spec
        self.state_dtype = np.dtype(state_dtype)
        if not self.state_dtype.names or "terminal" not in self.state_dtype.names:
            raise ValueError("state_dtype must be a structured dtype with a 'terminal' field")
        self.source = source
        if params is None:
            raw = np.zeros(8, dtype=np.uint8)  # an empty Params struct still has size 1: pad
        elif isinstance(params, (bytes, bytearray)):
            raw = np.frombuffer(bytes(params), dtype=np.uint8)
        else:
            raw = np.ascontiguousarray(np.asarray(params)).view(np.uint8).reshape(-1)
        self.params = raw.copy()
        self.tables = {k: np.ascontiguousarray(v) for k, v in (tables or {}).items()}
        if self.tables:
            names = getattr(np.asarray(params), "dtype", np.dtype([])).names or ()
            missing = [k for k in self.tables if k not in names or np.asarray(params).dtype[k] != np.dtype("<u8")]
            if missing:
                raise ValueError(f"tables {missing} need '<u8' (pointer) fields of the same name in a structured params")
            self._params_dtype = np.asarray(params).dtype
        self._initial = initial_states
        self._ref_logp = None if reference_log_probs is None else np.asarray(reference_log_probs, np.float64)
        self._lib = None

    # -- the plug-in library
    def library(self):
        if self._lib is None:
            lib = _lib.load_plugin(compile_plugin(self.source))
            size = C.c_int32(0)
            if lib.vp_plugin_info(C.byref(size)) != 1:
                raise _lib.LibraryMissing("plug-in library carries no user model")
            if size.value != self.state_dtype.itemsize:
                raise ValueError(f"state_dtype is {self.state_dtype.itemsize} B but the source's State is "
                                 f"{size.value} B")
            self._lib = lib
        return self._lib

    def device_descriptor(self):
        from .envs._device import DeviceModel

        lib = self.library()
        dm = DeviceModel(_lib.VP_MODEL_USER, self.spec, self.state_dtype, self.pack, unpack=RecordStates)
        dm.lib = lib
        raw = self.params
        if self.tables:  # device addresses of the uploaded tables into their pointer fields
            p = raw.view(self._params_dtype)[0].copy()
            for k, v in self.tables.items():
                p[k] = dm.upload(v)
            raw = np.frombuffer(p.tobytes(), dtype=np.uint8).copy()
        dm.desc.user_params = dm.upload(raw)
        dm.desc.user_param_bytes = len(self.params)
        return dm

    def pack(self, states) -> np.ndarray:
        """RecordStates, a structured array, or any object with one attribute per field."""
        if isinstance(states, RecordStates):
            return states.records.astype(self.state_dtype, copy=False)
        if isinstance(states, np.ndarray) and states.dtype.names:
            return np.ascontiguousarray(states).astype(self.state_dtype, copy=False)
        n = len(states)
        out = np.zeros(n, dtype=self.state_dtype)
        for f in self.state_dtype.names:
            if hasattr(states, f):
                out[f] = np.asarray(getattr(states, f)).reshape(out[f].shape)
        return out

    # -- ProblemModel (core.py:84-142), every piece on the device
    def sample_initial_states(self, n: int, rng) -> RecordStates:
        if self._initial is None:
            raise NotImplementedError("CudaModel needs initial_states= to sample initial states")
        return RecordStates(self.pack(self._initial(n, rng)))

    def step_batch(self, states, actions, rng):
        from .envs._device import device_model

        return device_model(self).step(states, actions, rng)

    def value_heuristic(self, states) -> np.ndarray:
        from .envs._device import device_model

        return device_model(self).heuristic(states)

    def observation_log_likelihood(self, next_states, action: int, observation: int) -> np.ndarray:
        from .envs._device import device_model

        if not 0 <= observation <= self.spec.terminal_obs:
            raise ValueError("invalid observation code")
        return device_model(self).obs_loglik(next_states, action, observation)

    def reference_log_probs(self) -> np.ndarray:
        if self._ref_logp is not None:
            return self._ref_logp.copy()
        return super().reference_log_probs()
