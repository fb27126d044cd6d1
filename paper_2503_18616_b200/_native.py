"""ctypes binding of the C-ABI in include/tissuesim_b200.h.

The shared library is built in-tree (``paper_2503_18616_b200/_native/``) by
``build.build()``.  There is no fallback: if the library cannot be loaded,
every product entry raises :class:`NativeLibraryError`.
"""

from __future__ import annotations

import ctypes
import os

from .errors import NativeLibraryError, ValidationError

LIB_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_native")
LIB_PATH = os.path.join(LIB_DIR, "libtissuesim_b200.so")

TS_OK, TS_ERR_INVALID, TS_ERR_CUDA, TS_ERR_NOMEM, TS_ERR_UNSUPPORTED = 0, -1, -2, -3, -4
TS_F32, TS_F64 = 0, 1

_P = ctypes.c_void_p
_D = ctypes.c_double
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64


class SceneDesc(ctypes.Structure):
    _fields_ = [
        ("n_vert", _I32), ("n_edge", _I32), ("n_tet", _I32), ("n_face", _I32), ("n_att", _I32),
        ("positions_rest", _P), ("inverse_mass", _P), ("edges", _P), ("rest_length", _P),
        ("tets", _P), ("rest_volume", _P), ("faces", _P),
        ("att_vertex", _P), ("att_faces", _P), ("att_is_face", _P), ("att_anchor", _P),
        ("att_rest", _P), ("att_k", _P),
        ("dt", _D), ("substeps", _I32), ("gravity", _D * 3), ("k_s", _D), ("k_v", _D), ("damping", _D),
        ("k_contact", _D), ("contact_iterations", _I32),
        ("rcm", _D * 3), ("shaft_radius", _D), ("clamp_radius", _D), ("clamp_length", _D),
        ("grasp_radius2", _D),
        ("start_axis", _D * 3), ("start_jaw", _D * 3), ("start_reach", _D), ("start_clamp", _D),
        ("held_clamp_angle", _D), ("held_cos", _D), ("held_sin", _D),
        ("target", _D * 3), ("action_scale", _D), ("success_threshold", _D),
        ("w_distance", _D), ("w_delta", _D), ("w_success", _D), ("reward_scale", _D),
        ("workspace_low", _D * 3), ("workspace_high", _D * 3),
        ("max_episode_steps", _I64),
        ("start_distance", _D), ("target_obs", _D * 3),
    ]


class LayoutOpts(ctypes.Structure):
    _fields_ = [("precision", _I32), ("block_threads", _I32), ("max_chunk_slots", _I32),
                ("schedule_banks", _I32), ("smem_budget", _I32), ("compact", _I32),
                ("edge_gather", _I32), ("cluster_size", _I32), ("refine_iters", _I32)]


class LayoutInfo(ctypes.Structure):
    _fields_ = [("precision", _I32), ("block_threads", _I32), ("vertices_per_thread", _I32),
                ("n_chunks", _I32), ("n_free", _I32), ("n_store", _I32), ("slot_capacity", _I32),
                ("smem_bytes", _I32), ("n_edge_items", _I32), ("n_tet_items", _I32),
                ("n_att_items", _I32), ("n_slots_total", _I32), ("bank_conflicts_p1", _I32),
                ("compact", _I32), ("edge_gather", _I32), ("n_edge_incidences", _I32),
                ("slot_budget", _I32), ("cluster_size", _I32),
                ("program_bytes", _I64)]

    def as_dict(self):
        return {name: getattr(self, name) for name, _ in self._fields_}


class EnvState(ctypes.Structure):
    _fields_ = [("x", _P), ("v", _P), ("tool_axis", _P), ("tool_jaw", _P), ("tool_reach", _P),
                ("tool_clamp", _P), ("grasp_vertex", _P), ("grasped", _P), ("steps", _P),
                ("l_prev", _P), ("ep_return", _P)]


class StepOut(ctypes.Structure):
    _fields_ = [("obs", _P), ("reward", _P), ("terminated", _P), ("truncated", _P),
                ("distance", _P), ("success", _P), ("diverged", _P), ("clipped", _P),
                ("contacts", _P), ("episode_return", _P), ("episode_length", _P),
                ("done_mask", _P), ("final_obs", _P), ("obs_f64", _I32)]


class ToolOverride(ctypes.Structure):
    _fields_ = [("axis", _P), ("jaw", _P), ("reach", _P), ("clamp", _P), ("clipped", _P)]


# ---- typed (DLPack) boundary -------------------------------------------------------------------
ENV_TENSORS = ("x", "v", "tool_axis", "tool_jaw", "tool_reach", "tool_clamp", "grasp_vertex", "grasped",
               "steps", "l_prev", "ep_return")
STEP_OUTS = ("obs", "reward", "terminated", "truncated", "distance", "success", "diverged", "clipped",
             "contacts", "episode_return", "episode_length", "done_mask", "final_obs")
OVERRIDE_TENSORS = ("axis", "jaw", "reach", "clamp", "clipped")


class EnvTensors(ctypes.Structure):
    _fields_ = [(k, _P) for k in ENV_TENSORS]


class StepOutTensors(ctypes.Structure):
    _fields_ = [(k, _P) for k in STEP_OUTS]


class ToolOverrideTensors(ctypes.Structure):
    _fields_ = [(k, _P) for k in OVERRIDE_TENSORS]


_capsule_ptr = ctypes.pythonapi.PyCapsule_GetPointer
_capsule_ptr.restype = ctypes.c_void_p
_capsule_ptr.argtypes = [ctypes.py_object, ctypes.c_char_p]


class DL:
    """A zero-copy DLPack view of a torch tensor (``torch.utils.dlpack.to_dlpack``): ``.ptr`` is the
    ``DLManagedTensor*`` (its first member is the ``DLTensor`` the *_dl entries read).  The capsule
    is kept alive with this object and frees the managed tensor when collected (it is never
    consumed: the library only borrows the view for the call)."""

    __slots__ = ("capsule", "ptr", "tensor")

    def __init__(self, t):
        from torch.utils.dlpack import to_dlpack
        self.tensor = t
        self.capsule = to_dlpack(t)
        self.ptr = _capsule_ptr(self.capsule, b"dltensor")


def dl(t):
    """DL view of `t` (None -> None)."""
    return None if t is None else DL(t)


def dlp(d):
    """DLTensor* of a DL view (None -> NULL).  The caller keeps `d` alive across the C call: a
    collected capsule frees the DLManagedTensor the pointer refers to (never ``dlp(dl(t))``)."""
    return None if d is None else d.ptr


def dl_struct(cls, names, tensors):
    """A ctypes struct of DLTensor* from {name: tensor or None}; keeps the DL views on the struct."""
    s = cls()
    keep = []
    for name in names:
        d = dl(tensors.get(name))
        keep.append(d)
        setattr(s, name, dlp(d))
    s._keep = keep
    return s


# exported symbols (checked by tests/test_abi.py against include/tissuesim_b200.h)
_SIGNATURES = {
    "ts_last_error": ([], ctypes.c_char_p),
    "ts_abi_version": ([], _I32),
    "ts_launch_count": ([], _I64),
    "ts_create": ([_P, _P, _I32, _P], _I32),
    "ts_create_from_program": ([_P, _P, _I64, _P, _I32, _P], _I32),
    "ts_destroy": ([_P], _I32),
    "ts_query": ([_P, _P], _I32),
    "ts_compile_program": ([_P, _P, _P, _P, _P], _I32),
    "ts_env_step": ([_P, _P, _I64, _P, _I32, _P, _P, _P, _P], _I32),
    "ts_env_reset": ([_P, _P, _I64, _P, _P, _I32, _P], _I32),
    "ts_env_observe": ([_P, _P, _I64, _P, _I32, _P], _I32),
    "ts_set_max_grid": ([_P, _I32], _I32),
    "ts_sim_step": ([_P, _P, _I64, _P, _P, _P, _P, _P, _P, _P, _P], _I32),
    "ts_run_substeps": ([_P, _P, _P, _I64, _P, _P, _P, _D, _I32, _D, _P], _I32),
    "ts_detect_contacts": ([_P, _P, _I64, _P, _P, _P, _P, _P, _P, _P, _P], _I32),
    "ts_uniform_actions": ([_P, _I64, _I64, ctypes.c_uint64, ctypes.c_uint64, _P], _I32),
    "ts_smem_probe": ([_I32, _I32, _P], _I32),
    "ts_uniform_actions_dev": ([_P, _I64, _I64, ctypes.c_uint64, _P, _P], _I32),
    "ts_kernel_timing": ([_P, _I32, _I32], _I32),
    "ts_kernel_time": ([_P, _P, _P], _I32),
    "ts_step_kernel_name": ([_P], ctypes.c_char_p),
    "ts_graph_launch_sync": ([_P, _P], _I32),
    "ts_graph_launch": ([_P, _P], _I32),
    "ts_stream_sync": ([_P], _I32),
    "ts_env_step_dl": ([_P, _P, _P, _P, _P, _P, _P], _I32),
    "ts_env_reset_dl": ([_P, _P, _P, _P, _P], _I32),
    "ts_env_observe_dl": ([_P, _P, _P, _P], _I32),
    "ts_sim_step_dl": ([_P, _P, _P, _P, _P, _P, _P, _P, _P, _P], _I32),
    "ts_run_substeps_dl": ([_P, _P, _P, _P, _P, _P, _D, _I32, _D, _P], _I32),
    "ts_detect_contacts_dl": ([_P, _P, _P, _P, _P, _P, _P, _P, _P, _P], _I32),
}

_lib = None


def load():
    """The loaded library (raises NativeLibraryError if it is not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeLibraryError(
            f"sm_100a library not built: {LIB_PATH} is missing "
            "(run `python -c 'import __graft_entry__ as g; g.build()'`)")
    try:
        lib = ctypes.CDLL(LIB_PATH)
    except OSError as exc:
        raise NativeLibraryError(f"cannot load {LIB_PATH}: {exc}") from exc
    for name, (args, res) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def exported_symbols():
    return sorted(_SIGNATURES)


def check(rc, what="call"):
    if rc == TS_OK:
        return
    msg = load().ts_last_error().decode("utf-8", "replace")
    if rc == TS_ERR_INVALID:
        raise ValidationError(f"{what}: {msg}")
    raise NativeLibraryError(f"{what} failed ({rc}): {msg}")


def ptr(t):
    """Device/host address of a torch tensor or numpy array (None -> NULL)."""
    if t is None:
        return None
    if hasattr(t, "data_ptr"):
        return t.data_ptr() if t.numel() else None
    return t.ctypes.data if t.size else None
