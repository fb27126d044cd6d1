"""The reference's kernel-backend plugin protocol, served by the sm_100a kernels.

Module attributes and entry points mirror ``tissuesim.backends._kernels``
(_kernels.pyx:28-50, 577-674, 797-947) so code written against the plugin
protocol can call this module with the same numpy arguments:

* ``run_substeps(x, v, w, edges, ..., grasp_vertex, drag_points, g, h,
  substeps, damping, acc, cnt, threads, parallel, scratch)`` -- in place on
  x, v (float64 -> the fp64 build, bitwise equal to the compiled backend;
  float32 -> the fp32 build);
* ``detect_contacts(pos, faces, caps, iters)`` -> (face, cap, depth, dir, bary).

Each call uploads, runs the step kernels once, and downloads; the compiled
topology program is cached per topology.  This is the validation boundary:
production code calls ``EnvBatch`` / ``Simulation``, which keep state resident.
Named "b200", never "cuda" (the reference's registry must keep rejecting
that name, pkg/tests/test_backends.py:30-32).
"""

from __future__ import annotations

import ctypes
import hashlib

import numpy as np
import torch

from . import _native as N
from .mesh import SceneConfig
from .scene import DeviceScene, SceneArrays

NAME = "b200"
SUPPORTS_PARALLEL = False

_CACHE: dict = {}


def make_scratch(n_env, n_vert):
    """State stays on the device; no host scratch is needed."""
    return None


def _key(*arrays, extra=()):
    h = hashlib.sha1()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode() + str(a.shape).encode())
        h.update(a.tobytes())
    h.update(repr(extra).encode())
    return h.hexdigest()


class _AttSpec:
    def __init__(self, vertex, face_row, anchor, rest, k):
        self.vertex, self.face, self.anchor, self.rest, self.stiffness = vertex, face_row, anchor, rest, k


def _scene_for(w, edges, rest_len, ks, tets, rest_vol, kv, att_vertex, att_faces, att_is_face,
               att_anchor, att_rest, att_k, precision, faces=None, iters=8, layout=None):
    layout = dict(layout or {})
    key = _key(w, edges, rest_len, tets, rest_vol, att_vertex, att_faces, att_is_face, att_anchor,
               att_rest, att_k, faces if faces is not None else np.zeros(0),
               extra=(float(ks), float(kv), precision, int(iters), torch.cuda.current_device(),
                      sorted(layout.items())))
    sc = _CACHE.get(key)
    if sc is not None:
        return sc
    nv = len(w)
    cfg = SceneConfig(k_s=float(ks), k_v=float(kv), substeps=1, dt=1.0, total_mass=1.0)
    atts = []
    att_faces = np.asarray(att_faces, np.int32).reshape(-1, 3)
    # attachment face rows are given as vertex triples: expose them as pseudo surface faces
    for i in range(len(att_vertex)):
        face_idx = i if att_is_face[i] else None
        atts.append(_AttSpec(int(att_vertex[i]), face_idx, np.asarray(att_anchor).reshape(-1, 3)[i],
                             float(att_rest[i]), float(att_k[i])))
    arr = SceneArrays(np.zeros((nv, 3)), w, edges, rest_len, tets, rest_vol,
                      np.zeros((0, 3), np.int32) if faces is None else faces, cfg,
                      attachments=atts, surface_faces=att_faces if len(atts) else None,
                      contact_iterations=iters)
    sc = DeviceScene(arr, torch.cuda.current_device(), precision=precision, **layout)
    if len(_CACHE) > 32:
        _CACHE.clear()
    _CACHE[key] = sc
    return sc


def run_substeps(x, v, w, edges, rest_len, ks, tets, rest_vol, kv,
                 att_vertex, att_faces, att_is_face, att_anchor, att_rest, att_k,
                 grasp_vertex, drag_points, g, h, substeps, damping,
                 acc=None, cnt=None, threads=1, parallel=False, scratch=None, *, layout=None):
    """In place on x, v (N, V, 3).  Same arguments as _kernels.run_substeps (_kernels.pyx:577-585)."""
    x_np, v_np = x, v
    if x_np.dtype not in (np.float32, np.float64):
        raise TypeError("x must be float32 or float64")
    precision = "fp64" if x_np.dtype == np.float64 else "fp32"
    n_env, n_vert, _ = x_np.shape
    if n_env == 0 or n_vert == 0:
        return None
    sc = _scene_for(np.asarray(w, np.float64), edges, rest_len, ks, tets, rest_vol, kv, att_vertex,
                    att_faces, att_is_face, att_anchor, att_rest, att_k, precision, layout=layout)
    dev = torch.device("cuda", torch.cuda.current_device())
    xt = torch.as_tensor(np.ascontiguousarray(x_np), device=dev)
    vt = torch.as_tensor(np.ascontiguousarray(v_np), device=dev)
    gv = torch.as_tensor(np.ascontiguousarray(grasp_vertex, np.int64), device=dev)
    drag = torch.as_tensor(np.ascontiguousarray(drag_points, np.float64).reshape(n_env, 3), device=dev)
    grav = (ctypes.c_double * 3)(*[float(a) for a in np.asarray(g, np.float64)])
    stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    views = [N.dl(t) for t in (xt, vt, gv, drag)]
    N.check(sc.lib.ts_run_substeps_dl(sc.handle, *(d.ptr for d in views), grav, float(h), int(substeps),
                                      float(damping), stream), "ts_run_substeps")
    x_np[...] = xt.cpu().numpy()
    v_np[...] = vt.cpu().numpy()
    return None


def detect_contacts(pos, faces, caps, iters=8, *, layout=None):
    """Contacts of one position set (V, 3) against capsule rows (C, 7), capsule-major order.

    float64 positions run the fp64 build (bitwise equal to _kernels.detect_contacts); float32
    positions run the fp32 build's narrow phase -- the production kernel's arithmetic -- like
    ``run_substeps`` dispatches on the dtype of x.  Rows come back as float64 either way."""
    pos = np.asarray(pos)
    precision = "fp32" if pos.dtype == np.float32 else "fp64"
    pos = np.ascontiguousarray(pos, np.float32 if precision == "fp32" else np.float64)
    faces = np.ascontiguousarray(faces, np.int32).reshape(-1, 3)
    caps = np.ascontiguousarray(caps, np.float64).reshape(-1, 7)
    nf, nc = len(faces), len(caps)
    if nf == 0 or nc == 0:
        return (np.zeros(0, np.int32), np.zeros(0, np.int32), np.zeros(0), np.zeros((0, 3)), np.zeros((0, 3)))
    if nc > 3:
        raise ValueError("the device contact kernel handles up to 3 capsules (shaft + 2 clamps)")
    nv = len(pos)
    # rows of absent capsules are parked far away with a tiny radius; they never hit
    rows = np.zeros((3, 7))
    rows[:, 0:3] = 1e30
    rows[:, 3:6] = 1e30 + 1.0
    rows[:, 6] = 1e-30
    rows[:nc] = caps
    sc = _scene_for(np.ones(nv), np.zeros((0, 2), np.int32), np.zeros(0), 1.0, np.zeros((0, 4), np.int32),
                    np.zeros(0), 1.0, np.zeros(0, np.int32), np.zeros((0, 3), np.int32), np.zeros(0, np.uint8),
                    np.zeros((0, 3)), np.zeros(0), np.zeros(0), precision, faces=faces, iters=iters, layout=layout)
    dev = torch.device("cuda", torch.cuda.current_device())
    x = torch.as_tensor(pos[None], device=dev)
    c = torch.as_tensor(rows[None], device=dev)
    cap_n = 3 * nf
    count = torch.zeros(1, dtype=torch.int32, device=dev)
    face = torch.zeros(cap_n, dtype=torch.int32, device=dev)
    capi = torch.zeros(cap_n, dtype=torch.int32, device=dev)
    depth = torch.zeros(cap_n, dtype=torch.float64, device=dev)
    direc = torch.zeros((cap_n, 3), dtype=torch.float64, device=dev)
    bary = torch.zeros((cap_n, 3), dtype=torch.float64, device=dev)
    stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    views = [N.dl(t) for t in (x, c, count, face[None], capi[None], depth[None], direc[None], bary[None])]
    N.check(sc.lib.ts_detect_contacts_dl(sc.handle, *(d.ptr for d in views), stream), "ts_detect_contacts")
    k = int(count.item())
    return (face[:k].cpu().numpy(), capi[:k].cpu().numpy(), depth[:k].cpu().numpy(),
            direc[:k].cpu().numpy(), bary[:k].cpu().numpy())
