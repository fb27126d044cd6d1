"""Batched simulation state on the GPU and its step (mirror of the reference's ``Simulation``).

``Simulation`` keeps the reference's attribute names (``x``, ``v``, ``w``,
``grasped``, ``grasp_vertex``, ``tool``, ``mesh``, ``rest``, ``cfg``,
``params``, ``step_count``) but every per-instance array is a CUDA tensor
that the sm_100a kernels update in place.  One ``step`` is three stream-ordered
launches -- the per-env command kernel (tool command, grasp release, capsule
rows), the fused step kernel (grasp search, substeps, contacts, divergence
flags; one CTA or one thread-block cluster per env) and the per-env epilogue --
see ``csrc/step_kernel.cuh``.  Reference: solver.py:247-381.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .errors import SimulationDiverged, ValidationError
from .scene import DeviceScene, SceneArrays
from .tool import ToolBatch


@dataclass
class SolverParams:
    """solver.py:78-94."""

    dt: float
    substeps: int
    gravity: np.ndarray
    damping: float = 0.0

    def __post_init__(self):
        if self.dt <= 0.0:
            raise ValidationError("dt must be positive")
        if self.substeps < 1:
            raise ValidationError("substeps must be >= 1")
        self.gravity = np.asarray(self.gravity, dtype=np.float64)

    @property
    def h(self):
        return self.dt / self.substeps


def _device(device):
    dev = torch.device(device if device is not None else "cuda")
    if dev.type != "cuda":
        raise ValidationError("the B200 engine runs on CUDA devices only (no CPU fallback)")
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    return dev


# Latency policy for `layout=None` (measured, profiles/r01r/mesh_scaling.json): a thread-block
# cluster costs ~90 us/step of DSMEM halo exchange and cluster barriers at any size, so it only
# pays once one CTA needs more than that (about 768 vertices); it then pays while each CTA keeps
# >= ~200 vertices and the envs x CTAs still fit on the SMs at once.
CLUSTER_MIN_VERTICES = 768
CLUSTER_MIN_VERTICES_PER_CTA = 200


def latency_cluster_size(n_vert, num_instances, sms):
    """CTAs per env for the auto layout: 0 (let the compiler pick the smallest layout that fits,
    which maximises throughput) unless the GPU would otherwise be mostly idle."""
    if n_vert < CLUSTER_MIN_VERTICES or num_instances < 1:
        return 0
    budget = min(16, sms // num_instances)
    k = 0
    for cand in (2, 4, 8, 16):
        if cand <= budget and n_vert // cand >= CLUSTER_MIN_VERTICES_PER_CTA:
            k = cand
    return k


def latency_block_threads(n_free, num_instances, sms, precision):
    """CTA size for the auto layout of a small fp32 batch (at most one env per SM): ~1.3 threads per
    free vertex spreads the tet batches over more warps (one env: 47.0 -> 45.0 us/step, 16 envs:
    53.7 -> 50.5; measured, reach_1170).  0 = the compiler's default (one thread per free vertex),
    which is the throughput choice once envs share SMs."""
    if precision != "fp32" or num_instances > sms or n_free < 1:
        return 0
    b = min(512, -(-int(1.3 * n_free) // 32) * 32)
    return b if b > -(-n_free // 32) * 32 else 0


def _as_device_f64(a, n, dev, name, width=3):
    if isinstance(a, torch.Tensor):
        t = a.to(device=dev, dtype=torch.float64)
    else:
        t = torch.as_tensor(np.asarray(a, dtype=np.float64), device=dev)
    shape = (n, width) if width > 1 else (n,)
    if tuple(t.shape) != shape:
        raise ValidationError(f"{name} must have shape {shape}, got {tuple(t.shape)}")
    return t.contiguous()


class Simulation:
    """N independent scene instances on one GPU (solver.py:247-381).

    ``precision`` selects the solver storage type: "fp32" (throughput build)
    or "fp64" (bitwise-reference build).  Tool, grasp and task state are fp64
    in both.  ``backend``/``mode``/``threads`` are accepted for signature
    compatibility; the only engine is the sm_100a kernel and it is always
    deterministic.
    """

    def __init__(self, mesh, rest, cfg, num_instances=1, backend="auto", mode="deterministic",
                 threads=None, k_contact=1.0, contact_iterations=8, device=None, precision="fp32",
                 layout=None):
        if mode not in ("deterministic", "parallel"):
            raise ValidationError(f"unknown execution mode {mode!r}")
        if backend not in (None, "auto", "b200", "cuda"):
            raise ValidationError(f"unknown backend {backend!r}; this engine is 'b200' only")
        if num_instances < 1:
            raise ValidationError("num_instances must be >= 1")
        self.mesh, self.rest, self.cfg = mesh, rest, cfg
        self.params = SolverParams(cfg.dt, cfg.substeps, cfg.gravity, cfg.damping)
        self.mode = mode
        self.threads = threads
        self.k_contact = k_contact
        self.contact_iterations = contact_iterations
        self.device = _device(device)
        self.precision = "fp64" if precision in ("fp64", "float64") else "fp32"
        self.dtype = torch.float64 if self.precision == "fp64" else torch.float32
        self.arrays = SceneArrays.from_loaded(mesh, rest, cfg, k_contact=k_contact,
                                              contact_iterations=contact_iterations)
        layout = dict(layout or {})
        auto_k = 0
        sms = torch.cuda.get_device_properties(self.device).multi_processor_count
        if "cluster_size" not in layout:
            auto_k = latency_cluster_size(mesh.vertex_count, int(num_instances), sms)
        if not auto_k and "block_threads" not in layout and not layout.get("cluster_size"):
            n_free = mesh.vertex_count - len(np.unique(mesh.pinned))
            b = latency_block_threads(n_free, int(num_instances), sms, self.precision)
            if b:
                layout["block_threads"] = b
        with torch.cuda.device(self.device):
            try:
                self.scene = DeviceScene(self.arrays, self.device.index, precision=self.precision,
                                         **layout, **({"cluster_size": auto_k} if auto_k else {}))
            except RuntimeError:
                if not auto_k:
                    raise
                # the latency layout is smaller than the mesh needs: the compiler's own choice
                self.scene = DeviceScene(self.arrays, self.device.index, precision=self.precision, **layout)
        self.backend = self.scene
        n, nv = int(num_instances), mesh.vertex_count
        self.num_instances = n
        dev = self.device
        rest_x = torch.as_tensor(mesh.positions_rest, dtype=self.dtype, device=dev)
        self.x = rest_x.unsqueeze(0).repeat(n, 1, 1).contiguous()
        self.v = torch.zeros((n, nv, 3), dtype=self.dtype, device=dev)
        self.w = torch.as_tensor(rest.inverse_mass, dtype=torch.float64, device=dev)
        self.grasped = torch.zeros((n, nv), dtype=torch.uint8, device=dev)
        self.grasp_vertex = torch.full((n,), -1, dtype=torch.int64, device=dev)
        k = self.arrays.consts
        self.tool = ToolBatch.from_constants(cfg, k, n, dev)
        # task state lives here too so one kernel owns the whole step
        self._steps = torch.zeros(n, dtype=torch.int64, device=dev)
        self._l_prev = torch.zeros(n, dtype=torch.float64, device=dev)
        self._return = torch.zeros(n, dtype=torch.float64, device=dev)
        self.step_count = 0
        self._state = None

    @classmethod
    def from_scene(cls, path, **kw):
        from .mesh import load_scene
        return cls(*load_scene(path), **kw)

    # -- C-ABI plumbing -----------------------------------------------------
    def state_struct(self):
        """ts_env_tensors: DLPack views of the live state tensors (rebuilt when a tensor was
        replaced; the library checks every view's dtype / shape / device / strides per call)."""
        keys = (self.x, self.v, self.tool.axis, self.tool.jaw_dir, self.tool.reach,
                self.tool.clamp_angle, self.grasp_vertex, self.grasped, self._steps, self._l_prev,
                self._return)
        # (tensor object, storage address): a replaced or reallocated tensor rebuilds the views; shape
        # and stride changes in place are seen through the views (they point at the tensor's own
        # size / stride arrays) and checked by the library on every call
        sig = tuple((id(t), t.data_ptr()) for t in keys)
        if self._state is None or self._state[0] != sig:
            self._state = (sig, N.dl_struct(N.EnvTensors, N.ENV_TENSORS, dict(zip(N.ENV_TENSORS, keys))))
        return self._state[1]

    def stream_ptr(self):
        return ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    # -- reference API --------------------------------------------------------
    def reset_instances(self, idx=None):
        """solver.py:314-320 (x = rest, v = 0, grasp cleared, tool at start pose)."""
        n = self.num_instances
        mask = None
        if idx is not None:
            sel = np.atleast_1d(np.asarray(idx))
            m = np.zeros(n, np.uint8)
            m[sel] = 1
            mask = torch.as_tensor(m, device=self.device)
        st = self.state_struct()
        mask_dl = N.dl(mask)          # the view must outlive the call
        with torch.cuda.device(self.device):
            N.check(self.scene.lib.ts_env_reset_dl(self.scene.handle, ctypes.byref(st), N.dlp(mask_dl), None,
                                                   self.stream_ptr()), "ts_env_reset")

    def step(self, targets=None, angles=None, raise_on_divergence=True, tool_override=None):
        """One outer step (solver.py:322-366).  Returns an info dict of device tensors."""
        n = self.num_instances
        dev = self.device
        info = {}
        t = a = None
        if targets is not None:
            t = _as_device_f64(targets, n, dev, "targets")
            if angles is not None:
                a = _as_device_f64(angles, n, dev, "angles", width=1)
        clipped = torch.empty(n, dtype=torch.bool, device=dev)
        rejected = torch.empty(n, dtype=torch.bool, device=dev)
        diverged = torch.empty(n, dtype=torch.bool, device=dev)
        contacts = torch.empty(n, dtype=torch.int32, device=dev)
        ovr = None
        if tool_override is not None:
            ovr, keep = _override_struct(tool_override, n, dev)
        st = self.state_struct()
        views = [N.dl(x) for x in (t, a, clipped, rejected, diverged, contacts)]
        with torch.cuda.device(dev):
            N.check(self.scene.lib.ts_sim_step_dl(
                self.scene.handle, ctypes.byref(st), N.dlp(views[0]), N.dlp(views[1]),
                ctypes.byref(ovr) if ovr is not None else None,
                *(N.dlp(v) for v in views[2:]), self.stream_ptr()), "ts_sim_step")
        self.step_count += 1
        if targets is not None or tool_override is not None:
            info["clipped"], info["rejected"] = clipped, rejected
        info["contacts_per_env"] = contacts
        info["contacts"] = LazyInt(lambda: int(contacts.sum().item()))
        info["diverged"] = diverged
        if raise_on_divergence and bool(diverged.any().item()):
            bad = int(torch.nonzero(diverged)[0].item())
            raise SimulationDiverged(
                f"instance {bad} produced non-finite positions at step {self.step_count}",
                step=self.step_count)
        return info

    def kinetic_energy(self):
        """Total kinetic energy per instance, joules (solver.py:368-371)."""
        speed2 = (self.v.double() ** 2).sum(-1)
        return 0.5 * speed2 @ torch.as_tensor(self.mesh.vertex_mass, device=self.device)

    def instance_state(self, i):
        from types import SimpleNamespace
        return SimpleNamespace(x=self.x[i], v=self.v[i], w=self.w, grasped=self.grasped[i])

    def tool_model(self, i):
        return self.tool.tool_model(i, int(self.grasp_vertex[i].item()))


class LazyInt:
    """An int computed on first use (keeps the step free of host syncs)."""

    def __init__(self, fn):
        self._fn = fn
        self._v = None

    def value(self):
        if self._v is None:
            self._v = self._fn()
        return self._v

    def __int__(self):
        return self.value()

    def __index__(self):
        return self.value()

    def __eq__(self, other):
        return self.value() == other

    def __add__(self, other):
        return self.value() + other

    __radd__ = __add__

    def __repr__(self):
        return repr(self.value())


def _override_struct(ovr, n, dev):
    """ts_tool_override_tensors from a dict of post-command poses (validation injection)."""
    def t(name, width):
        return _as_device_f64(ovr[name], n, dev, name, width)
    keep = {"axis": t("axis", 3), "jaw": t("jaw", 3), "reach": t("reach", 1), "clamp": t("clamp", 1)}
    clipped = ovr.get("clipped")
    if clipped is not None:
        keep["clipped"] = torch.as_tensor(np.asarray(clipped, np.uint8) if not isinstance(clipped, torch.Tensor)
                                          else clipped.to(torch.uint8), device=dev).contiguous()
    return N.dl_struct(N.ToolOverrideTensors, N.OVERRIDE_TENSORS, keep), keep
