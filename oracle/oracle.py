"""CPU oracle for the tissue-reach environment step (TEST INFRASTRUCTURE ONLY).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline
leg may import this module, and only as the checker.  The product package
(``paper_2503_18616_b200``) never imports it and has no CPU fallback.

It restates the reference ``tissuesim`` 0.1.0 step (``/root/reference/pkg``):

* numpy (float64, same expression association, same numpy calls where the
  reference's result depends on numpy's own kernels):
    - tool kinematics      <- tool.py:304-389 (apply_commands, update_grasps,
                              capsule_rows, drag_points), tool.py:47-62
                              (rotate_about_axis, perpendicular_unit),
                              tool.py:161-173 (start pose)
    - step orchestration   <- solver.py:322-366 (Simulation.step)
    - reward / obs / done  <- env.py:61-67, 99-115, 123-197
* C (``oracle/ts_oracle.c`` via ctypes), bitwise equal to the compiled backend:
    - substep solver       <- backends/_kernels.pyx:260-352
    - contact detection    <- backends/_kernels.pyx:797-947
    - contact resolution   <- collision.py:55-73

Parity pin: tests/test_oracle.py runs this against the real reference
(built by oracle/build_ref.sh) and against tests/golden/*.npz.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libts_oracle.so")

GRASP_ENGAGE_DEG = 3.0      # tool.py:23
MIN_LEVER_ARM = 1e-9        # tool.py:24
MIN_ROTATION = 1e-9         # tool.py:25
OBS_SIZE = 6
ACT_SIZE = 3

_lib = None


def build_oracle(force=False):
    """Compile ts_oracle.c with the reference's fp flags (pkg/setup.py:20)."""
    src = os.path.join(_HERE, "ts_oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        import subprocess
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-ffp-contract=off",
                               "-fno-math-errno", "-fno-wrapv", src, "-o", _LIB_PATH, "-lm"])
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build_oracle()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        I = ctypes.c_int
        D = ctypes.c_double
        L.tso_run_substeps.argtypes = [I, I, P, P, P, I, P, P, D, I, P, P, D, I, P, P, P, P, P, P,
                                       P, P, P, D, I, D, P, P]
        L.tso_run_substeps.restype = None
        L.tso_detect_contacts.argtypes = [P, I, P, I, P, I, P, P, P, P, P]
        L.tso_detect_contacts.restype = I
        L.tso_resolve_contacts.argtypes = [P, P, P, I, P, P, P, P, D]
        L.tso_resolve_contacts.restype = None
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None and a.size else None


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


# ---------------------------------------------------------------------------
# plugin-level kernels (same argument meaning as the reference backend)
# ---------------------------------------------------------------------------

def run_substeps(x, v, w, edges, rest_len, ks, tets, rest_vol, kv,
                 att_vertex, att_faces, att_is_face, att_anchor, att_rest, att_k,
                 grasp_vertex, drag_points, g, h, substeps, damping):
    """In-place on x, v (N, V, 3) float64; mirrors _kernels.run_substeps."""
    assert x.dtype == np.float64 and x.flags.c_contiguous and v.flags.c_contiguous
    n_env, n_vert, _ = x.shape
    edges = _c(edges, np.int32).reshape(-1, 2)
    tets = _c(tets, np.int32).reshape(-1, 4)
    att_vertex = _c(att_vertex, np.int32).reshape(-1)
    att_faces = _c(att_faces, np.int32).reshape(-1, 3)
    att_is_face = _c(att_is_face, np.uint8).reshape(-1)
    att_anchor = _c(att_anchor, np.float64).reshape(-1, 3)
    att_rest = _c(att_rest, np.float64).reshape(-1)
    att_k = _c(att_k, np.float64).reshape(-1)
    rest_len = _c(rest_len, np.float64)
    rest_vol = _c(rest_vol, np.float64)
    w = _c(w, np.float64)
    gv = _c(grasp_vertex, np.int64)
    drag = _c(drag_points, np.float64).reshape(-1, 3)
    g = _c(g, np.float64)
    acc = np.zeros(n_vert * 3)
    cnt = np.zeros(n_vert)
    lib().tso_run_substeps(n_env, n_vert, _p(x), _p(v), _p(w),
                           len(edges), _p(edges), _p(rest_len), float(ks),
                           len(tets), _p(tets), _p(rest_vol), float(kv),
                           len(att_vertex), _p(att_vertex), _p(att_faces), _p(att_is_face),
                           _p(att_anchor), _p(att_rest), _p(att_k),
                           _p(gv), _p(drag), _p(g), float(h), int(substeps), float(damping),
                           _p(acc), _p(cnt))


def detect_contacts(pos, faces, caps, iters=8):
    """(face, cap, depth, dir, bary) rows, capsule-major; mirrors _kernels.detect_contacts."""
    pos = _c(pos, np.float64)
    faces = _c(faces, np.int32).reshape(-1, 3)
    caps = _c(caps, np.float64).reshape(-1, 7)
    rows = max(1, len(faces) * len(caps))
    of = np.empty(rows, np.int32)
    oc = np.empty(rows, np.int32)
    od = np.empty(rows)
    odir = np.empty((rows, 3))
    ob = np.empty((rows, 3))
    n = lib().tso_detect_contacts(_p(pos), len(faces), _p(faces), len(caps), _p(caps), int(iters),
                                  _p(of), _p(oc), _p(od), _p(odir), _p(ob))
    return of[:n].copy(), oc[:n].copy(), od[:n].copy(), odir[:n].copy(), ob[:n].copy()


def resolve_contacts(pos, w, faces, face_idx, cap_idx, depth, direction, bary, k_c=1.0):
    """In place on pos (V, 3); mirrors collision.resolve_contact_arrays."""
    assert pos.dtype == np.float64 and pos.flags.c_contiguous
    face_idx = _c(face_idx, np.int32)
    if len(face_idx) == 0:
        return
    lib().tso_resolve_contacts(_p(pos), _p(_c(w, np.float64)), _p(_c(faces, np.int32)),
                               len(face_idx), _p(face_idx), _p(_c(depth, np.float64)),
                               _p(_c(direction, np.float64)), _p(_c(bary, np.float64)),
                               float(k_c))


# ---------------------------------------------------------------------------
# tool kinematics (numpy; the transcendental calls are numpy's own)
# ---------------------------------------------------------------------------

def _dot(u, w):
    return u[..., 0] * w[..., 0] + u[..., 1] * w[..., 1] + u[..., 2] * w[..., 2]


def _cross(u, w):
    out = np.empty(np.broadcast(u, w).shape)
    out[..., 0] = u[..., 1] * w[..., 2] - u[..., 2] * w[..., 1]
    out[..., 1] = u[..., 2] * w[..., 0] - u[..., 0] * w[..., 2]
    out[..., 2] = u[..., 0] * w[..., 1] - u[..., 1] * w[..., 0]
    return out


def _norm(u):
    return np.sqrt(_dot(u, u))


def _rodrigues(vec, k, ang):
    c = np.cos(ang)[..., None]
    s = np.sin(ang)[..., None]
    kv = _dot(k, vec)[..., None]
    return vec * c + _cross(k, vec) * s + k * kv * (1.0 - c)


def _some_perpendicular(a):
    ref = np.zeros_like(a)
    z = np.abs(a[..., 0]) > 0.9
    ref[..., 0] = np.where(z, 0.0, 1.0)
    ref[..., 2] = np.where(z, 1.0, 0.0)
    out = ref - a * _dot(a, ref)[..., None]
    return out / _norm(out)[..., None]


def start_pose(rcm, tool_start, clamp_angle):
    """Tool pose at reset: axis, jaw_dir, reach, clamp angle (tool.py:161-173, 123-136)."""
    offset = np.asarray(tool_start, np.float64) - np.asarray(rcm, np.float64)
    reach = float(np.linalg.norm(offset))
    axis = offset / reach
    axis = axis / float(_norm(axis))
    jaw = _some_perpendicular(axis)
    return axis, jaw, reach, float(clamp_angle)


# ---------------------------------------------------------------------------
# batched environment
# ---------------------------------------------------------------------------

class OracleScene:
    """Plain arrays + config for one scene (what the oracle consumes)."""

    def __init__(self, positions_rest, w, edges, rest_length, tets, rest_volume, faces,
                 cfg, att_vertex=None, att_faces=None, att_is_face=None, att_anchor=None,
                 att_rest=None, att_k=None, vertex_mass=None):
        self.positions_rest = _c(positions_rest, np.float64)
        self.w = _c(w, np.float64)
        self.edges = _c(edges, np.int32).reshape(-1, 2)
        self.rest_length = _c(rest_length, np.float64)
        self.tets = _c(tets, np.int32).reshape(-1, 4)
        self.rest_volume = _c(rest_volume, np.float64)
        self.faces = _c(faces, np.int32).reshape(-1, 3)
        self.cfg = cfg
        na = 0 if att_vertex is None else len(att_vertex)
        self.att_vertex = _c(att_vertex if na else np.zeros(0), np.int32)
        self.att_faces = _c(att_faces if na else np.zeros((0, 3)), np.int32).reshape(-1, 3)
        self.att_is_face = _c(att_is_face if na else np.zeros(0), np.uint8)
        self.att_anchor = _c(att_anchor if na else np.zeros((0, 3)), np.float64).reshape(-1, 3)
        self.att_rest = _c(att_rest if na else np.zeros(0), np.float64)
        self.att_k = _c(att_k if na else np.zeros(0), np.float64)
        self.vertex_mass = vertex_mass


class OracleEnv:
    """Restatement of EnvBatch + Simulation (env.py:70-197, solver.py:247-366).

    State arrays are public numpy arrays named like the reference's.
    ``tool_override`` (optional callable) lets a test replace the tool
    command with externally supplied poses; it receives (self, targets,
    angles) and must set axis/jaw/reach/clamp and return (clipped, rejected).
    """

    def __init__(self, scene: OracleScene, num_envs=1, k_contact=1.0, contact_iterations=8):
        cfg = scene.cfg
        self.scene = scene
        self.cfg = cfg
        self.n = n = int(num_envs)
        self.nv = nv = len(scene.positions_rest)
        self.k_contact = k_contact
        self.contact_iterations = contact_iterations
        self.h = cfg.dt / cfg.substeps
        self.rcm = np.asarray(cfg.rcm, np.float64)
        self.x = np.ascontiguousarray(np.tile(scene.positions_rest, (n, 1, 1)))
        self.v = np.zeros((n, nv, 3))
        self.grasped = np.zeros((n, nv), np.uint8)
        self.grasp_vertex = np.full(n, -1, np.int64)
        ax, jaw, reach, clamp = start_pose(cfg.rcm, cfg.tool_start, cfg.clamp_angle)
        self._start = (ax, jaw, reach, clamp)
        self.axis = np.tile(ax, (n, 1))
        self.jaw = np.tile(jaw, (n, 1))
        self.reach = np.full(n, reach)
        self.clamp = np.full(n, clamp)
        self.lo = np.asarray(cfg.workspace_low, np.float64)
        self.hi = np.asarray(cfg.workspace_high, np.float64)
        self.target = np.asarray(cfg.target, np.float64)
        self.steps = np.zeros(n, np.int64)
        self.l_prev = np.zeros(n)
        self.ret = np.zeros(n)
        self.step_count = 0
        self.tool_override = None
        self.last_contacts = None

    # -- tool ---------------------------------------------------------------
    def drag_points(self):
        return self.rcm[None, :] + self.reach[:, None] * self.axis

    def apply_commands(self, targets, angles):
        """tool.py:307-345."""
        targets = np.asarray(targets, np.float64)
        bounded = np.minimum(np.maximum(targets, self.lo), self.hi)
        clipped = np.any(bounded != targets, axis=1)
        v1 = self.drag_points() - self.rcm[None, :]
        v2 = bounded - self.rcm[None, :]
        n1 = _norm(v1)
        n2 = _norm(v2)
        rejected = n2 < MIN_LEVER_ARM
        n2s = np.where(rejected, 1.0, n2)
        theta = np.arccos(np.clip(_dot(v1, v2) / (n1 * n2s), -1.0, 1.0))
        k = _cross(v1, v2)
        kn = _norm(k)
        rot = (theta > MIN_ROTATION) & (kn > 0.0) & ~rejected
        k = np.where(rot[:, None], k / np.where(kn > 0.0, kn, 1.0)[:, None], 0.0)
        flip = (theta > MIN_ROTATION) & (kn == 0.0) & ~rejected
        if np.any(flip):
            k[flip] = _some_perpendicular(v1[flip] / n1[flip][:, None])
            rot = rot | flip
        theta = np.where(rot, theta, 0.0)
        ax = _rodrigues(self.axis, k, theta)
        ax = ax / _norm(ax)[:, None]
        jw = _rodrigues(self.jaw, k, theta)
        jw = jw - ax * _dot(ax, jw)[:, None]
        jw = jw / _norm(jw)[:, None]
        ok = ~rejected
        self.axis[ok] = np.where(rot[ok, None], ax[ok], self.axis[ok])
        self.jaw[ok] = np.where(rot[ok, None], jw[ok], self.jaw[ok])
        self.reach[ok] = self.reach[ok] + (n2 - n1)[ok]
        self.clamp[ok] = np.asarray(angles, np.float64)[ok]
        return clipped, rejected

    def update_grasps(self):
        """tool.py:372-389."""
        rel_release = self.clamp >= GRASP_ENGAGE_DEG
        for i in np.flatnonzero(rel_release & (self.grasp_vertex >= 0)):
            self.grasped[i, self.grasp_vertex[i]] = 0
            self.grasp_vertex[i] = -1
        cand = np.flatnonzero(~rel_release & (self.grasp_vertex < 0))
        if len(cand) == 0:
            return
        drag = self.drag_points()[cand]
        rel = self.x[cand] - drag[:, None, :]
        d2 = np.where(self.scene.w[None, :] > 0.0, _dot(rel, rel), np.inf)
        best = np.argmin(d2, axis=1)
        hit = d2[np.arange(len(cand)), best] <= self.cfg.grasp_radius ** 2
        for r, i in enumerate(cand):
            if hit[r]:
                self.grasp_vertex[i] = best[r]
                self.grasped[i, best[r]] = 1

    def capsule_rows(self):
        """tool.py:347-370."""
        cfg = self.cfg
        n = self.n
        pivot = self.rcm[None, :] + (self.reach - cfg.clamp_length)[:, None] * self.axis
        alpha = np.radians(self.clamp)
        ca = np.cos(alpha)[:, None]
        sa = np.sin(alpha)[:, None]
        da = ca * self.axis + sa * self.jaw
        db = ca * self.axis - sa * self.jaw
        base = np.tile(self.rcm, (n, 1))
        degen = _norm(pivot - base) < 1e-9
        if np.any(degen):
            base[degen] = pivot[degen] - 1e-6 * self.axis[degen]
        rows = np.empty((n, 3, 7))
        rows[:, 0, 0:3] = base
        rows[:, 0, 3:6] = pivot
        rows[:, 0, 6] = cfg.shaft_radius
        for c, d in ((1, da), (2, db)):
            rows[:, c, 0:3] = pivot
            rows[:, c, 3:6] = pivot + cfg.clamp_length * d
            rows[:, c, 6] = cfg.clamp_radius
        return rows

    # -- simulation ---------------------------------------------------------
    def sim_step(self, targets=None, angles=None):
        """solver.py:322-366 with raise_on_divergence=False; returns info dict."""
        info = {}
        if targets is not None:
            if angles is None:
                angles = self.clamp.copy()
            if self.tool_override is not None:
                info["clipped"], info["rejected"] = self.tool_override(self, targets, angles)
            else:
                info["clipped"], info["rejected"] = self.apply_commands(targets, angles)
            # post-command poses, for injecting into a device step (validation builds)
            self.last_cmd = dict(axis=self.axis.copy(), jaw=self.jaw.copy(), reach=self.reach.copy(),
                                 clamp=self.clamp.copy(), clipped=info["clipped"].copy())
        self.update_grasps()
        s = self.scene
        cfg = self.cfg
        run_substeps(self.x, self.v, s.w, s.edges, s.rest_length, cfg.k_s, s.tets, s.rest_volume,
                     cfg.k_v, s.att_vertex, s.att_faces, s.att_is_face, s.att_anchor, s.att_rest,
                     s.att_k, self.grasp_vertex, self.drag_points(), np.asarray(cfg.gravity, np.float64),
                     self.h, cfg.substeps, cfg.damping)
        total = 0
        per_env = np.zeros(self.n, np.int64)
        found_all = []
        if len(s.faces):
            caps = self.capsule_rows()
            for i in range(self.n):
                found = detect_contacts(self.x[i], s.faces, caps[i], self.contact_iterations)
                found_all.append(found)
                if len(found[0]):
                    resolve_contacts(self.x[i], s.w, s.faces, *found, k_c=self.k_contact)
                    per_env[i] = len(found[0])
                    total += len(found[0])
        self.last_contacts = found_all
        info["contacts"] = total
        info["contacts_per_env"] = per_env
        self.step_count += 1
        info["diverged"] = ~np.isfinite(self.x).all(axis=(1, 2))
        return info

    def reset_instances(self, idx):
        ax, jaw, reach, clamp = self._start
        self.x[idx] = self.scene.positions_rest
        self.v[idx] = 0.0
        self.grasped[idx] = 0
        self.grasp_vertex[idx] = -1
        self.axis[idx] = ax
        self.jaw[idx] = jaw
        self.reach[idx] = reach
        self.clamp[idx] = clamp

    # -- env ----------------------------------------------------------------
    def _normalize(self, p):
        return 2.0 * (p - self.lo) / (self.hi - self.lo) - 1.0

    def distances(self, idx=None):
        drag = self.drag_points()
        if idx is not None:
            drag = drag[idx]
        rel = drag - self.target[None, :]
        return np.sqrt(np.einsum("nq,nq->n", rel, rel))

    def observe_rows(self, idx):
        drag = self.drag_points()[idx]
        obs = np.empty((len(idx), OBS_SIZE))
        obs[:, 0:3] = self._normalize(drag)
        obs[:, 3:6] = self._normalize(self.target[None, :])
        return obs

    def reset(self, indices=None):
        idx = np.arange(self.n) if indices is None else np.atleast_1d(indices)
        self.reset_instances(idx)
        self.steps[idx] = 0
        self.ret[idx] = 0.0
        self.l_prev[idx] = self.distances(idx)
        return self.observe_rows(idx)

    def reward(self, distance, delta, success):
        c = self.cfg
        return c.reward_scale * (c.reward_distance_weight * distance + c.reward_delta_weight * delta
                                 + c.reward_success_weight * np.asarray(success, np.float64))

    def step(self, actions):
        """env.py:144-197 (validation omitted: callers pass valid actions)."""
        a = np.clip(np.asarray(actions, np.float64), -1.0, 1.0)
        targets = self.drag_points() + a * self.cfg.action_scale
        angles = np.full(self.n, self.cfg.clamp_angle)
        sinfo = self.sim_step(targets, angles)
        diverged = sinfo["diverged"]
        distance = self.distances()
        success = distance < self.cfg.success_threshold
        reward = self.reward(distance, distance - self.l_prev, success)
        self.steps += 1
        self.ret += reward
        terminated = success & ~diverged
        truncated = (~terminated) & ((self.steps >= self.cfg.max_episode_steps) | diverged)
        done = terminated | truncated
        info = {
            "distance": distance.copy(), "success": success.copy(), "diverged": diverged.copy(),
            "clipped": sinfo.get("clipped"), "contacts": sinfo["contacts"],
            "contacts_per_env": sinfo["contacts_per_env"],
            "episode_return": self.ret.copy(), "episode_length": self.steps.copy(),
            "done_mask": done.copy(), "final_observation": None,
        }
        allidx = np.arange(self.n)
        self.l_prev[~done] = distance[~done]
        if np.any(done):
            fo = np.zeros((self.n, OBS_SIZE))
            fo[done] = self.observe_rows(allidx[done])
            info["final_observation"] = fo
            self.reset(allidx[done])
        return self.observe_rows(allidx), reward, terminated, truncated, info


def scene_from_loaded(mesh, rest, cfg) -> OracleScene:
    """Bundle (TetMesh, RestState, SceneConfig) into oracle arrays (solver.py:280-301)."""
    atts = list(cfg.attachments)
    na = len(atts)
    av = np.array([a.vertex for a in atts], np.int32)
    af = np.zeros((na, 3), np.int32)
    aif = np.zeros(na, np.uint8)
    aa = np.zeros((na, 3))
    for i, a in enumerate(atts):
        if a.face is not None:
            af[i] = mesh.surface_faces[a.face]
            aif[i] = 1
        else:
            aa[i] = a.anchor
    return OracleScene(mesh.positions_rest, rest.inverse_mass, mesh.edges, rest.rest_length,
                       mesh.tets, rest.rest_volume, mesh.surface_faces, cfg,
                       av, af, aif, aa, np.array([a.rest for a in atts]),
                       np.array([a.stiffness for a in atts]), mesh.vertex_mass)
