"""ctypes binding of the C ABI in include/vpb200.h (libvpb200.so, sm_100a).

This is the "reference-side FFI" of the drop-in: the reference planner is pure
Python (/root/reference/pkg/src/vecpomdp), so the natural binding is ctypes.
There is no fallback: if the library is missing or CUDA is unavailable every
entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("VPB200_LIB") or os.path.join(_HERE, "libvpb200.so")  # override: experiments only

VP_OK, VP_ERR_INVALID, VP_ERR_CAPACITY, VP_ERR_CUDA, VP_ERR_MODEL = range(5)
VP_MODEL_MARS, VP_MODEL_TABULAR, VP_MODEL_SYNTHETIC, VP_MODEL_LIGHTDARK, VP_MODEL_NAVIGATION = 1, 2, 3, 4, 5
VP_MODEL_CROWDNAV = 6
VP_MODEL_USER = 7  # plug-in builds only (plugin.py)
CROWD_MAX_PEOPLE, CROWD_MAX_TRACKED, CROWD_STATE_BYTES = 320, 8, 2704
VP_PSI_F32, VP_PSI_F64 = 0, 1
VP_RNG_SPLITMIX64, VP_RNG_PHILOX = 0, 1
RNG_KINDS = {"splitmix64": VP_RNG_SPLITMIX64, "philox": VP_RNG_PHILOX}
VP_SEARCH_FUSED, VP_SEARCH_TRAJECTORY, VP_SEARCH_INSERT = 0, 1, 2
ABI_VERSION = 9
VP_COUNTERS, VP_COUNTER_ACTIONS, VP_COUNTER_DENSE = 64, 32, 48  # include/vpb200.h
VP_COUNTER_LIVE_B, VP_COUNTER_LIVE_A, VP_COUNTER_DONE = 8, 16, 24
VP_OVERLAY_SLOTS = 4

p_i8, p_i16, p_i32, p_u32, p_f64, p_u8, p_u64 = (
    C.POINTER(C.c_int8), C.POINTER(C.c_int16), C.POINTER(C.c_int32), C.POINTER(C.c_uint32),
    C.POINTER(C.c_double), C.POINTER(C.c_uint8), C.POINTER(C.c_uint64))


class VpModel(C.Structure):
    _fields_ = [
        ("kind", C.c_int32), ("action_count", C.c_int32), ("obs_arity", C.c_int32),
        ("state_bytes", C.c_int32), ("discount", C.c_double),
        ("mars_n", C.c_int32), ("mars_m", C.c_int32), ("mars_ops", C.c_int32), ("mars_pad", C.c_int32),
        ("mars_half_eff", C.c_double), ("mars_rock_at", C.c_void_p), ("mars_acc", C.c_void_p),
        ("mars_gpow", C.c_void_p),
        ("mars_rock_x", C.c_int16 * 64), ("mars_rock_y", C.c_int16 * 64),
        ("tab_states", C.c_int32), ("tab_obs", C.c_int32),
        ("tab_cum_t", C.c_void_p), ("tab_cum_z", C.c_void_p), ("tab_reward", C.c_void_p),
        ("tab_terminal", C.c_void_p), ("tab_log_z", C.c_void_p),
        ("syn_branching", C.c_int32), ("syn_term_per_mille", C.c_int32),
        ("syn_obs_accuracy", C.c_double), ("syn_salt", C.c_uint64),
        ("ld_step", C.c_double), ("ld_light_x", C.c_double), ("ld_goal_radius", C.c_double),
        ("ld_sigma0", C.c_double), ("ld_sigma_slope", C.c_double), ("ld_bin_width", C.c_double),
        ("ld_bins", C.c_int32), ("ld_pad", C.c_int32),
        ("nav_h", C.c_int32), ("nav_w", C.c_int32), ("nav_unknown", C.c_int32), ("nav_pad", C.c_int32),
        ("nav_kind", C.c_void_p), ("nav_aux", C.c_void_p), ("nav_goal", C.c_void_p), ("nav_heur", C.c_void_p),
        ("nav_acc", C.c_double), ("nav_log_acc", C.c_double), ("nav_log_miss", C.c_double),
        ("crowd_people", C.c_int32), ("crowd_tracked", C.c_int32),
        ("crowd_hall_w", C.c_double), ("crowd_hall_d", C.c_double), ("crowd_noise", C.c_double),
        ("crowd_react", C.c_double), ("crowd_r_nearby", C.c_double), ("crowd_v_curious", C.c_double),
        ("crowd_v_shy", C.c_double), ("crowd_v_back", C.c_double), ("crowd_collision", C.c_double),
        ("crowd_heur", C.c_void_p), ("crowd_heur_len", C.c_int32), ("rng_kind", C.c_int32),
        ("user_params", C.c_void_p), ("user_param_bytes", C.c_int64),
    ]


class VpTree(C.Structure):
    _fields_ = [
        ("cap_beliefs", C.c_int32), ("cap_actions", C.c_int32), ("action_count", C.c_int32),
        ("psi_dtype", C.c_int32), ("exact", C.c_int32), ("psi_stride", C.c_int32),
        ("hmask_a", C.c_uint64), ("hmask_b", C.c_uint64),
        ("b_parent_action", C.c_void_p), ("b_parent_obs", C.c_void_p), ("b_parent_belief", C.c_void_p),
        ("b_parent_act", C.c_void_p), ("b_depth", C.c_void_p),
        ("psi", C.c_void_p), ("b_lse", C.c_void_p), ("b_value", C.c_void_p),
        ("b_rows", C.c_void_p), ("b_acc", C.c_void_p), ("b_flags", C.c_void_p), ("b_rec", C.c_void_p),
        ("b_nact", C.c_void_p), ("b_ckey", C.c_void_p),
        ("a_parent_belief", C.c_void_p), ("a_action", C.c_void_p), ("a_reward", C.c_void_p),
        ("a_visits", C.c_void_p), ("a_rows", C.c_void_p), ("a_acc", C.c_void_p), ("a_ckey", C.c_void_p),
        ("a_slot", C.c_void_p),
        ("hash_a", C.c_void_p), ("hash_b", C.c_void_p), ("counters", C.c_void_p),
        ("init_prefs", C.c_void_p), ("init_lse", C.c_void_p), ("init_cdf", C.c_void_p),
        ("psi_cdf", C.c_void_p), ("dense_meta", C.c_void_p), ("bkey_mode", C.c_int32),
        ("cap_dense", C.c_int32), ("overlay_slots", C.c_int32), ("init_uniform", C.c_int32), ("eta", C.c_double),
    ]


class VpWork(C.Structure):
    _fields_ = [
        ("n", C.c_int32), ("max_levels", C.c_int32), ("states", C.c_void_p),
        ("leaves", C.c_void_p), ("leaf_count", C.c_void_p), ("leaf_belief", C.c_void_p),
        ("leaf_value", C.c_void_p), ("stats", C.c_void_p),
        ("trace_action", C.c_void_p), ("trace_obs", C.c_void_p), ("trace_anode", C.c_void_p),
        ("trace_belief", C.c_void_p), ("trace_reward", C.c_void_p),
    ]


class VpSearchArgs(C.Structure):
    _fields_ = [
        ("search_key", C.c_uint64), ("depth0", C.c_int32), ("d_max", C.c_int32),
        ("pass_", C.c_uint32), ("pad0", C.c_int32),
        ("inject_actions", C.c_void_p), ("start_beliefs", C.c_void_p), ("search_key_dev", C.c_void_p),
        ("particles", C.c_void_p), ("cum_weights", C.c_void_p), ("draw_key_dev", C.c_void_p),
        ("draw_key", C.c_uint64), ("m", C.c_int32), ("mode", C.c_int32), ("row0", C.c_int32),
        ("pad1", C.c_int32), ("inject_obs", C.c_void_p), ("inject_reward", C.c_void_p),
        ("inject_leaf", C.c_void_p),
    ]


class VpPlanArgs(C.Structure):
    _fields_ = [
        ("iterations", C.c_int32), ("d_max_cap", C.c_int32), ("m", C.c_int32), ("mode", C.c_int32),
        ("gamma", C.c_double),
        ("particles_host", C.c_void_p), ("particles_dev", C.c_void_p),
        ("cumw_host", C.c_void_p), ("cumw_dev", C.c_void_p),
        ("keys_host", C.c_void_p), ("keys_dev", C.c_void_p),
        ("out_host", C.c_void_p), ("out_dev", C.c_void_p),
    ]


# (name, restype, argtypes) -- exactly the exports of include/vpb200.h
_SIGNATURES = [
    ("vp_abi_version", C.c_int32, []),
    ("vp_status_string", C.c_char_p, [C.c_int32]),
    ("vp_last_cuda_error", C.c_int32, []),
    ("vp_abi_layout", C.c_int32, [p_i32, C.c_int32]),
    ("vp_profile_enable", C.c_int32, [C.c_int32]),
    ("vp_profile_read", C.c_int32, [p_f64, C.POINTER(C.c_int64), C.c_int32]),
    ("vp_launch_count", C.c_int64, []),
    ("vp_tree_init", C.c_int32, [C.POINTER(VpTree), C.c_void_p]),
    ("vp_tree_rehash", C.c_int32, [C.POINTER(VpTree), C.c_void_p]),
    ("vp_tree_build_cdfs", C.c_int32, [C.POINTER(VpTree), C.c_void_p]),
    ("vp_tree_set_eta", C.c_int32, [C.POINTER(VpTree), C.c_void_p]),
    ("vp_probe_latency", C.c_int32, [C.c_void_p, C.c_int32, C.c_int32, C.c_uint64, C.c_void_p, C.c_void_p]),
    ("vp_tree_counts", C.c_int32, [C.POINTER(VpTree), p_i32, C.c_void_p]),
    ("vp_draw_root_states", C.c_int32,
     [C.POINTER(VpModel), C.POINTER(VpWork), C.c_void_p, C.c_void_p, C.c_int32, C.c_uint64, C.c_void_p]),
    ("vp_search", C.c_int32,
     [C.POINTER(VpTree), C.POINTER(VpModel), C.POINTER(VpWork), C.POINTER(VpSearchArgs), C.c_void_p]),
    ("vp_plan", C.c_int32,
     [C.POINTER(VpTree), C.POINTER(VpModel), C.POINTER(VpWork), C.POINTER(VpPlanArgs), C.c_void_p]),
    ("vp_backup", C.c_int32, [C.POINTER(VpTree), C.POINTER(VpWork), C.c_uint32, C.c_double, C.c_void_p]),
    ("vp_root_argmax", C.c_int32, [C.POINTER(VpTree), C.c_void_p, C.c_void_p]),
    ("vp_sir_weigh", C.c_int32,
     [C.POINTER(VpModel), C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_uint32, C.c_uint64, C.c_void_p,
      C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p]),
    ("vp_sir_resample", C.c_int32,
     [C.POINTER(VpModel), C.c_void_p, C.c_void_p, C.c_int32, C.c_double, C.c_void_p, C.c_void_p]),
    ("vp_tree_append_actions", C.c_int32,
     [C.POINTER(VpTree), C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_uint32, C.c_void_p, C.c_void_p]),
    ("vp_tree_append_beliefs", C.c_int32,
     [C.POINTER(VpTree), C.c_void_p, C.c_void_p, C.c_int32, C.c_uint32, C.c_void_p, C.c_void_p]),
    ("vp_broadcast_record", C.c_int32,
     [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p]),
    ("vp_pack_mars_states", C.c_int32,
     [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p]),
    ("vp_plan_keys", C.c_int32, [C.c_uint64, C.c_int32, C.c_void_p]),
    ("vp_rng_uniform", C.c_int32, [C.c_uint64, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_void_p]),
    ("vp_rng_normal", C.c_int32, [C.c_uint64, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_void_p]),
    ("vp_rng_draws", C.c_int32,
     [C.c_uint64, C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p]),
    ("vp_philox4x32_10", C.c_int32, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]),
    ("vp_model_step", C.c_int32,
     [C.POINTER(VpModel), C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p,
      C.c_void_p]),
    ("vp_model_heuristic", C.c_int32, [C.POINTER(VpModel), C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p]),
    ("vp_model_obs_loglik", C.c_int32,
     [C.POINTER(VpModel), C.c_void_p, C.c_int32, C.c_int32, C.c_uint32, C.c_void_p, C.c_void_p]),
    ("vp_plugin_info", C.c_int32, [C.POINTER(C.c_int32)]),
    ("vp_lse_rows", C.c_int32,
     [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_double, C.c_void_p, C.c_void_p]),
    ("vp_sample_rows", C.c_int32,
     [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_double, C.c_void_p, C.c_void_p, C.c_void_p,
      C.c_int32, C.c_void_p, C.c_void_p]),
]

EXPORTED_SYMBOLS = tuple(name for name, _, _ in _SIGNATURES)

KERNEL_KINDS = ("draw", "search", "backup", "tree_init", "rehash", "argmax", "hooks", "cdf_rows")


def profile_enable(on: bool):
    load().vp_profile_enable(1 if on else 0)


def profile_read() -> dict:
    """{kind: (total_ms, launches)} for launches recorded since profile_enable(True)."""
    k = len(KERNEL_KINDS)
    ms = (C.c_double * k)()
    cnt = (C.c_int64 * k)()
    load().vp_profile_read(ms, cnt, k)
    return {name: (ms[i], int(cnt[i])) for i, name in enumerate(KERNEL_KINDS)}


def launch_count() -> int:
    return int(load().vp_launch_count())


class CapacityError(RuntimeError):
    """Device arena or hash index too small (VP_ERR_CAPACITY)."""


class LibraryMissing(ImportError):
    pass


_lib = None


def _open(path: str):
    if not os.path.exists(path):
        raise LibraryMissing(
            f"{path} not found: build the sm_100a library first (`make` or "
            "`python -c 'import __graft_entry__ as g; g.build()'`). There is no CPU fallback.")
    lib = C.CDLL(path)
    for name, res, args in _SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.vp_abi_version() != ABI_VERSION:
        raise LibraryMissing(f"ABI mismatch: library {lib.vp_abi_version()} vs binding {ABI_VERSION}")
    return lib


def load(path: str = LIB_PATH):
    """Load and type the shared library (no CUDA context is created here)."""
    global _lib
    if _lib is None:
        _lib = _open(path)
    return _lib


_PLUGINS: dict = {}


def load_plugin(path: str):
    """A plug-in build of the library (plugin.py), typed like the main one; cached by path."""
    lib = _PLUGINS.get(path)
    if lib is None:
        load()  # the main library first: its status strings and the model-independent entry points
        lib = _PLUGINS[path] = _open(path)
    return lib


def call_on(lib, name: str, *args):
    """``call`` on a given library (None: the main one)."""
    if lib is None:
        return call(name, *args)
    fn = getattr(lib, name)
    st = fn(*args)
    if st != VP_OK:
        raise_status(st, name, lib)


def layout_mismatches() -> list:
    """Compare the ctypes mirrors with the library's own sizeof/offsetof."""
    lib = load()
    m = lib.vp_abi_layout(None, 0)
    buf = (C.c_int32 * m)()
    lib.vp_abi_layout(buf, m)
    mine = [C.sizeof(VpModel), C.sizeof(VpTree), C.sizeof(VpWork), C.sizeof(VpSearchArgs),
            VpModel.tab_states.offset, VpModel.ld_bins.offset, VpTree.eta.offset,
            VpWork.trace_belief.offset, VpSearchArgs.start_beliefs.offset, 16, C.sizeof(VpPlanArgs),
            VpPlanArgs.out_dev.offset, VpTree.init_cdf.offset, VpTree.a_ckey.offset, VpSearchArgs.m.offset,
            VpModel.mars_gpow.offset, VpTree.psi_cdf.offset, VpModel.nav_log_miss.offset,
            VpModel.crowd_heur.offset, CROWD_STATE_BYTES, VpTree.b_rec.offset, VpTree.a_slot.offset,
            VpTree.cap_dense.offset, VpModel.rng_kind.offset, VpModel.user_params.offset,
            VpModel.user_param_bytes.offset]
    names = ["sizeof(vp_model)", "sizeof(vp_tree)", "sizeof(vp_work)", "sizeof(vp_search_args)",
             "vp_model.tab_states", "vp_model.ld_bins", "vp_tree.eta", "vp_work.trace_belief",
             "vp_search_args.start_beliefs", "sizeof(Slot)", "sizeof(vp_plan_args)", "vp_plan_args.out_dev",
             "vp_tree.init_cdf", "vp_tree.a_ckey", "vp_search_args.m", "vp_model.mars_gpow", "vp_tree.psi_cdf", "vp_model.nav_log_miss",
             "vp_model.crowd_heur", "sizeof(CrowdState)", "vp_tree.b_rec", "vp_tree.a_slot", "vp_tree.cap_dense",
             "vp_model.rng_kind", "vp_model.user_params", "vp_model.user_param_bytes"]
    return [(nm, a, b) for nm, a, b in zip(names, list(buf), mine) if a != b]


def check(status: int, what: str = ""):
    """Map a vp_status to the reference's exception convention."""
    if status == VP_OK:
        return
    raise_status(status, what, load())


def raise_status(status: int, what: str, lib):
    msg = f"{what}: {lib.vp_status_string(status).decode()}"
    if status == VP_ERR_INVALID:
        raise ValueError(msg)
    if status == VP_ERR_CAPACITY:
        raise CapacityError(msg)
    if status == VP_ERR_MODEL:
        raise TypeError(msg)
    raise RuntimeError(msg)


_FNS: dict = {}


def call(name: str, *args):
    fn = _FNS.get(name)
    if fn is None:
        fn = _FNS[name] = getattr(load(), name)
    check(fn(*args), name)


_CUDA_OK = False


def torch_cuda():
    """torch, once a CUDA device is known to be present (checked until it is: the product path
    raises rather than fall back to the CPU)."""
    global _CUDA_OK
    import torch

    if not _CUDA_OK:
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2510_27191_b200 needs a CUDA device (B200, sm_100a); there is no CPU fallback")
        _CUDA_OK = True
    return torch
