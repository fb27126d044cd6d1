"""Tool pose state on the device (mirror of the reference's ``ToolBatch``, tool.py:263-399).

The pose arrays are fp64 CUDA tensors updated in place by the step kernel
(tool command, tool.py:307-345, runs inside it).  ``drag_points`` and
``capsule_rows`` here are host-side conveniences (inspection/tests) built
from the same formulas; the kernel computes its own copies on chip.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

GRASP_ENGAGE_DEG = 3.0   # tool.py:23
MIN_LEVER_ARM = 1e-9     # tool.py:24
MIN_ROTATION = 1e-9      # tool.py:25


@dataclass
class Capsule:
    p0: np.ndarray
    p1: np.ndarray
    radius: float

    def as_row(self):
        return np.concatenate([np.asarray(self.p0, float), np.asarray(self.p1, float), [self.radius]])


@dataclass
class ToolBatch:
    rcm: np.ndarray            # (3,)
    axis: torch.Tensor         # (N, 3) fp64
    jaw_dir: torch.Tensor      # (N, 3) fp64
    reach: torch.Tensor        # (N,) fp64
    clamp_angle: torch.Tensor  # (N,) fp64, degrees
    shaft_radius: float
    clamp_radius: float
    clamp_length: float
    grasp_radius: float
    workspace_low: np.ndarray
    workspace_high: np.ndarray

    @classmethod
    def from_constants(cls, cfg, consts, n, device):
        f64 = dict(dtype=torch.float64, device=device)
        return cls(
            rcm=np.asarray(cfg.rcm, np.float64).copy(),
            axis=torch.as_tensor(consts.start_axis, **f64).repeat(n, 1).contiguous(),
            jaw_dir=torch.as_tensor(consts.start_jaw, **f64).repeat(n, 1).contiguous(),
            reach=torch.full((n,), consts.start_reach, **f64),
            clamp_angle=torch.full((n,), consts.start_clamp, **f64),
            shaft_radius=float(cfg.shaft_radius), clamp_radius=float(cfg.clamp_radius),
            clamp_length=float(cfg.clamp_length), grasp_radius=float(cfg.grasp_radius),
            workspace_low=np.asarray(cfg.workspace_low, np.float64),
            workspace_high=np.asarray(cfg.workspace_high, np.float64),
        )

    def _rcm(self):
        return torch.as_tensor(self.rcm, dtype=torch.float64, device=self.axis.device)

    def drag_points(self):
        """rcm + reach * axis (tool.py:304-305)."""
        return self._rcm()[None, :] + self.reach[:, None] * self.axis

    def capsule_rows(self):
        """(N, 3, 7) shaft / clamp a / clamp b rows (tool.py:347-370)."""
        n = self.reach.shape[0]
        rcm = self._rcm()
        pivot = rcm[None, :] + (self.reach - self.clamp_length)[:, None] * self.axis
        alpha = self.clamp_angle * (math.pi / 180.0)
        ca = torch.cos(alpha)[:, None]
        sa = torch.sin(alpha)[:, None]
        da = ca * self.axis + sa * self.jaw_dir
        db = ca * self.axis - sa * self.jaw_dir
        base = rcm[None, :].repeat(n, 1)
        degen = torch.linalg.norm(pivot - base, dim=1) < 1e-9
        base = torch.where(degen[:, None], pivot - 1e-6 * self.axis, base)
        rows = torch.empty((n, 3, 7), dtype=torch.float64, device=self.axis.device)
        rows[:, 0, 0:3] = base
        rows[:, 0, 3:6] = pivot
        rows[:, 0, 6] = self.shaft_radius
        rows[:, 1, 0:3] = pivot
        rows[:, 1, 3:6] = pivot + self.clamp_length * da
        rows[:, 1, 6] = self.clamp_radius
        rows[:, 2, 0:3] = pivot
        rows[:, 2, 3:6] = pivot + self.clamp_length * db
        rows[:, 2, 6] = self.clamp_radius
        return rows

    def tool_model(self, i, grasp_vertex=-1):
        """Scalar snapshot of instance i (host numpy), for inspection."""
        from types import SimpleNamespace
        ax = self.axis[i].cpu().numpy()
        reach = float(self.reach[i].item())
        return SimpleNamespace(rcm=self.rcm.copy(), axis=ax, reach=reach,
                               jaw_dir=self.jaw_dir[i].cpu().numpy(),
                               clamp_angle=float(self.clamp_angle[i].item()),
                               drag_point=self.rcm + reach * ax, grasp_vertex=grasp_vertex)
