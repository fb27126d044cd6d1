"""Scene -> C-ABI scene description, and the device handle that owns the compiled program.

Host-side constants that the reference derives with numpy are derived here
with the same numpy calls, so they are bitwise identical to the reference on
the same host:

* start pose  <- ToolModel.from_config + __post_init__ (tool.py:123-136, 161-173)
* cos/sin of the held clamp angle <- ToolBatch.capsule_rows (tool.py:351-353)
* start distance <- EnvBatch._distances (env.py:103-108)
* normalized target <- EnvBatch._normalize (env.py:99-101)
"""

from __future__ import annotations

import ctypes
import hashlib
import os
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import ValidationError


def _dot(u, w):
    return u[..., 0] * w[..., 0] + u[..., 1] * w[..., 1] + u[..., 2] * w[..., 2]


def _perpendicular(a):
    """perpendicular_unit (tool.py:55-62)."""
    ref = np.zeros_like(a)
    use_z = np.abs(a[..., 0]) > 0.9
    ref[..., 0] = np.where(use_z, 0.0, 1.0)
    ref[..., 2] = np.where(use_z, 1.0, 0.0)
    out = ref - a * _dot(a, ref)[..., None]
    return out / np.sqrt(_dot(out, out))[..., None]


def tool_start_pose(cfg):
    """(axis, jaw_dir, reach, clamp_angle) at reset, exactly as the reference derives them."""
    offset = np.asarray(cfg.tool_start, np.float64) - np.asarray(cfg.rcm, np.float64)
    reach = float(np.linalg.norm(offset))
    axis = offset / reach
    if reach <= 0.0:
        raise ValidationError("tool reach must be positive")
    axis = axis / float(np.sqrt(_dot(axis, axis)))
    return axis, _perpendicular(axis), reach, float(cfg.clamp_angle)


def normalize(p, lo, hi):
    return 2.0 * (p - lo) / (hi - lo) - 1.0


@dataclass
class TaskConstants:
    start_axis: np.ndarray
    start_jaw: np.ndarray
    start_reach: float
    start_clamp: float
    held_cos: float
    held_sin: float
    start_distance: float
    target_obs: np.ndarray


def task_constants(cfg) -> TaskConstants:
    axis, jaw, reach, clamp = tool_start_pose(cfg)
    held = np.full(4, float(cfg.clamp_angle))
    alpha = np.radians(held)
    rcm = np.asarray(cfg.rcm, np.float64)
    drag = rcm[None, :] + np.array([reach])[:, None] * axis[None, :]
    rel = drag - np.asarray(cfg.target, np.float64)[None, :]
    dist = np.sqrt(np.einsum("nq,nq->n", rel, rel))
    lo = np.asarray(cfg.workspace_low, np.float64)
    hi = np.asarray(cfg.workspace_high, np.float64)
    return TaskConstants(axis, jaw, reach, clamp, float(np.cos(alpha)[0]), float(np.sin(alpha)[0]),
                         float(dist[0]), normalize(np.asarray(cfg.target, np.float64)[None, :], lo, hi)[0])


class SceneArrays:
    """Contiguous host arrays of one scene plus the C-ABI description pointing at them."""

    def __init__(self, positions_rest, inverse_mass, edges, rest_length, tets, rest_volume, faces,
                 cfg, attachments=(), surface_faces=None, k_contact=1.0, contact_iterations=8):
        c = np.ascontiguousarray
        self.positions_rest = c(positions_rest, np.float64).reshape(-1, 3)
        self.inverse_mass = c(inverse_mass, np.float64).reshape(-1)
        self.edges = c(edges, np.int32).reshape(-1, 2)
        self.rest_length = c(rest_length, np.float64).reshape(-1)
        self.tets = c(tets, np.int32).reshape(-1, 4)
        self.rest_volume = c(rest_volume, np.float64).reshape(-1)
        self.faces = c(faces, np.int32).reshape(-1, 3)
        atts = list(attachments)
        na = len(atts)
        sf = self.faces if surface_faces is None else c(surface_faces, np.int32).reshape(-1, 3)
        self.att_vertex = np.array([a.vertex for a in atts], np.int32)
        self.att_faces = np.zeros((na, 3), np.int32)
        self.att_is_face = np.zeros(na, np.uint8)
        self.att_anchor = np.zeros((na, 3))
        self.att_rest = np.array([a.rest for a in atts], np.float64)
        self.att_k = np.array([a.stiffness for a in atts], np.float64)
        for i, a in enumerate(atts):
            if a.face is not None:
                self.att_faces[i] = sf[a.face]   # solver.py:297-299
                self.att_is_face[i] = 1
            else:
                self.att_anchor[i] = a.anchor
        self.cfg = cfg
        self.consts = task_constants(cfg) if cfg is not None else None
        self.k_contact = float(k_contact)
        self.contact_iterations = int(contact_iterations)

    @classmethod
    def from_loaded(cls, mesh, rest, cfg, **kw):
        return cls(mesh.positions_rest, rest.inverse_mass, mesh.edges, rest.rest_length, mesh.tets,
                   rest.rest_volume, mesh.surface_faces, cfg, cfg.attachments, **kw)

    @property
    def n_vert(self):
        return len(self.positions_rest)

    def desc(self) -> N.SceneDesc:
        d = N.SceneDesc()
        d.n_vert, d.n_edge, d.n_tet = self.n_vert, len(self.edges), len(self.tets)
        d.n_face, d.n_att = len(self.faces), len(self.att_vertex)
        for name in ("positions_rest", "inverse_mass", "edges", "rest_length", "tets", "rest_volume",
                     "faces", "att_vertex", "att_faces", "att_is_face", "att_anchor", "att_rest", "att_k"):
            setattr(d, name, N.ptr(getattr(self, name)))
        cfg = self.cfg
        d.dt, d.substeps = float(cfg.dt), int(cfg.substeps)
        d.gravity[:] = [float(v) for v in np.asarray(cfg.gravity, np.float64)]
        d.k_s, d.k_v, d.damping = float(cfg.k_s), float(cfg.k_v), float(cfg.damping)
        d.k_contact, d.contact_iterations = self.k_contact, self.contact_iterations
        d.rcm[:] = [float(v) for v in np.asarray(cfg.rcm, np.float64)]
        d.shaft_radius, d.clamp_radius = float(cfg.shaft_radius), float(cfg.clamp_radius)
        d.clamp_length = float(cfg.clamp_length)
        d.grasp_radius2 = float(cfg.grasp_radius) ** 2      # tool.py:385
        k = self.consts
        d.start_axis[:] = [float(v) for v in k.start_axis]
        d.start_jaw[:] = [float(v) for v in k.start_jaw]
        d.start_reach, d.start_clamp = k.start_reach, k.start_clamp
        d.held_clamp_angle, d.held_cos, d.held_sin = float(cfg.clamp_angle), k.held_cos, k.held_sin
        d.target[:] = [float(v) for v in np.asarray(cfg.target, np.float64)]
        d.action_scale, d.success_threshold = float(cfg.action_scale), float(cfg.success_threshold)
        d.w_distance, d.w_delta = float(cfg.reward_distance_weight), float(cfg.reward_delta_weight)
        d.w_success, d.reward_scale = float(cfg.reward_success_weight), float(cfg.reward_scale)
        d.workspace_low[:] = [float(v) for v in np.asarray(cfg.workspace_low, np.float64)]
        d.workspace_high[:] = [float(v) for v in np.asarray(cfg.workspace_high, np.float64)]
        d.max_episode_steps = int(cfg.max_episode_steps)
        d.start_distance = k.start_distance
        d.target_obs[:] = [float(v) for v in k.target_obs]
        return d


def layout_opts(precision="fp32", block_threads=0, max_chunk_slots=0, schedule_banks=True, compact=True,
                edge_gather=None, cluster_size=0, refine_iters=0):
    o = N.LayoutOpts()
    o.precision = N.TS_F64 if precision in ("fp64", "float64", "f64", N.TS_F64) else N.TS_F32
    o.block_threads = int(block_threads)
    o.max_chunk_slots = int(max_chunk_slots)
    o.schedule_banks = 1 if schedule_banks else -1
    o.compact = 1 if compact else -1
    # None: the compiler's choice (owner gather); False: constraint-parallel edge slots
    o.edge_gather = 0 if edge_gather is None else (1 if edge_gather else -1)
    o.cluster_size = int(cluster_size)
    o.refine_iters = int(refine_iters)
    return o


# ---------------------------------------------------------------------------
# compiled-program cache: the thorough bank-schedule search takes seconds, so a program is
# compiled once per (scene, layout options, library build) -- memoised in the process and kept
# under _native/programs/ (TS_PROGRAM_CACHE=0 disables the disk copy)
# ---------------------------------------------------------------------------
_MEMO: dict = {}
_LIB_FP = None
CACHE_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_native", "programs")


def _lib_fingerprint():
    """Hash of what decides a program's bytes: the scene compiler's sources (compiler.cpp, its
    header and the blob format in program.h) -- kernel-only rebuilds keep the cache.  Falls back to
    the library itself when the sources are absent."""
    global _LIB_FP
    if _LIB_FP is None:
        from .build import CSRC, LIB
        h = hashlib.sha1()
        srcs = [os.path.join(CSRC, f) for f in ("compiler.cpp", "compiler.h", "program.h")]
        for f in (srcs if all(os.path.exists(f) for f in srcs) else [LIB]):
            with open(f, "rb") as fh:
                h.update(fh.read())
        _LIB_FP = h.hexdigest()
    return _LIB_FP


def _program_key(arrays: SceneArrays, o) -> str:
    h = hashlib.sha1(_lib_fingerprint().encode())
    for name in ("positions_rest", "inverse_mass", "edges", "rest_length", "tets", "rest_volume", "faces",
                 "att_vertex", "att_faces", "att_is_face", "att_anchor", "att_rest", "att_k"):
        a = np.ascontiguousarray(getattr(arrays, name))
        h.update(f"{name}:{a.dtype}:{a.shape}".encode())
        h.update(a.tobytes())
    d = arrays.desc()
    h.update(repr((d.k_s, d.k_v, d.k_contact, d.contact_iterations)).encode())
    h.update(bytes(o))
    # the compiler's development knobs (environment) change the program too
    h.update(repr([(k, os.environ.get(k)) for k in _COMPILER_ENV]).encode())
    return h.hexdigest()


_COMPILER_ENV = ("TS_SA_FOCUS", "TS_REFINE_ITERS", "TS_TET_HOLES", "TS_SPLIT_CT", "TS_NARROW", "TS_PIN_COPIES",
                 "TS_PIN_SHIFT", "TS_PACK_TETS", "TS_PACK_ITERS", "TS_TET_EXTRA_BATCHES")


def compile_program(arrays: SceneArrays, **layout):
    """Host copy of the compiled program (bytes, info dict) -- no GPU needed.  Cached."""
    blob, info = _compile_cached(arrays, layout_opts(**layout))
    return blob.copy(), info.as_dict()


def _compile_cached(arrays: SceneArrays, o):
    key = _program_key(arrays, o)
    hit = _MEMO.get(key)
    if hit is not None:
        return hit
    prefix = _lib_fingerprint()[:12]
    path = os.path.join(CACHE_DIR, f"{prefix}_{key}.npz")
    use_disk = os.environ.get("TS_PROGRAM_CACHE", "1") != "0"
    if use_disk and os.path.exists(path):
        try:
            z = np.load(path)
            info = N.LayoutInfo.from_buffer_copy(z["info"].tobytes())
            _MEMO[key] = (z["blob"], info)
            return _MEMO[key]
        except Exception:   # a torn / stale file: recompile
            pass
    blob, info = _compile_raw(arrays, o)
    _MEMO[key] = (blob, info)
    if use_disk:
        try:
            os.makedirs(CACHE_DIR, exist_ok=True)
            for old in os.listdir(CACHE_DIR):          # programs of other library builds are stale
                if old.endswith(".npz") and not old.startswith(prefix):
                    os.remove(os.path.join(CACHE_DIR, old))
            tmp = path + f".{os.getpid()}.tmp.npz"
            np.savez(tmp, blob=blob, info=np.frombuffer(bytes(info), np.uint8))
            os.replace(tmp, path)
        except OSError:
            pass
    return blob, info


def _compile_raw(arrays: SceneArrays, o):
    lib = N.load()
    d = arrays.desc()
    info = N.LayoutInfo()
    # generous first guess so the (seconds-long, bank-refined) compile runs once
    guess = (1 << 20) + 512 * (len(arrays.edges) + len(arrays.tets) + len(arrays.att_vertex)) \
        + 256 * arrays.n_vert + 64 * len(arrays.faces)
    for _ in range(2):
        buf = np.zeros(guess, np.uint8)
        size = ctypes.c_int64(guess)
        rc = lib.ts_compile_program(ctypes.byref(d), ctypes.byref(o), N.ptr(buf), ctypes.byref(size),
                                    ctypes.byref(info))
        if rc == N.TS_OK:
            return buf[:size.value].copy(), info
        if size.value <= guess:
            N.check(rc, "ts_compile_program")
        guess = int(size.value)
    N.check(rc, "ts_compile_program")


class DeviceScene:
    """Owns one ts_handle (the compiled program on one GPU)."""

    def __init__(self, arrays: SceneArrays, device_index=0, **layout):
        self.arrays = arrays
        self.lib = N.load()
        self._desc = arrays.desc()
        self._opts = layout_opts(**layout)
        self.precision = "fp64" if self._opts.precision == N.TS_F64 else "fp32"
        blob, pinfo = _compile_cached(arrays, self._opts)
        self.program_key = _program_key(arrays, self._opts)   # equal keys = the same compiled program
        h = ctypes.c_void_p()
        N.check(self.lib.ts_create_from_program(ctypes.byref(self._desc), N.ptr(blob), int(blob.nbytes),
                                                ctypes.byref(pinfo), int(device_index), ctypes.byref(h)),
                "ts_create_from_program")
        self.handle = h
        info = N.LayoutInfo()
        N.check(self.lib.ts_query(h, ctypes.byref(info)), "ts_query")
        self.info = info.as_dict()

    def set_max_grid(self, n):
        N.check(self.lib.ts_set_max_grid(self.handle, int(n)), "ts_set_max_grid")

    def close(self):
        if getattr(self, "handle", None) is not None and self.handle.value:
            self.lib.ts_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
