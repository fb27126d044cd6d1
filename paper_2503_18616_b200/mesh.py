"""Scene ingest: text formats, derived topology and rest state (host side, one-time).

Mirrors the reference's scene API (mesh.py) so a scene that loads there loads
here with bit-identical index arrays and fp64 rest data:

* ``parse_mesh_text``   <- mesh.py:233-285  (``tetmesh 1`` format)
* ``parse_scene_text``  <- mesh.py:445-479  (``key = value``, unknown keys rejected)
* ``derive_topology``   <- mesh.py:139-159  (edges sorted-unique; surface faces =
                           multiplicity-1 faces under the outward tet winding,
                           rows ordered by their sorted vertex triple)
* ``fix_orientation``   <- mesh.py:167-173, ``compute_rest_state`` <- 176-200,
  ``build_mesh`` <- 203-218, ``load_scene`` <- 508-524
* ``make_slab`` / ``slab_pins`` / ``make_slab_scene`` <- mesh.py:316-428 (fixture
  generator only; reach_1170.scene is byte-identical to make_slab_scene(1170))

Topology is derived with integer keys rather than row-wise ``np.unique``; the
ordering contract is the same (tests/test_mesh.py pins it against golden
fixtures produced by the reference).  Everything floating point uses the same
numpy reductions as the reference so fp64 rest data is bitwise identical.
"""

from __future__ import annotations

import os
from dataclasses import dataclass, field, fields

import numpy as np

from .errors import ParseError, ValidationError

MIN_TET_VOLUME = 1e-12  # m^3 (mesh.py:17)

# outward-wound faces of a positively oriented tet (a, b, c, d)  (mesh.py:136)
TET_FACE_CORNERS = ((0, 2, 1), (0, 1, 3), (0, 3, 2), (1, 2, 3))
TET_EDGE_CORNERS = ((0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3))


@dataclass
class TetMesh:
    vertex_count: int
    positions_rest: np.ndarray  # (V, 3) float64
    tets: np.ndarray            # (T, 4) int32, positively oriented
    edges: np.ndarray           # (E, 2) int32, a < b, rows sorted
    surface_faces: np.ndarray   # (F, 3) int32, outward winding
    pinned: np.ndarray          # (P,) int32 sorted
    vertex_mass: np.ndarray     # (V,) float64


@dataclass
class RestState:
    rest_length: np.ndarray   # (E,)
    rest_volume: np.ndarray   # (T,)
    inverse_mass: np.ndarray  # (V,), exactly 0 for pinned


@dataclass
class AttachmentSpec:
    vertex: int
    face: int | None = None
    anchor: np.ndarray | None = None
    rest: float = 0.0
    stiffness: float = 1.0


def _v3(x=0.0, y=0.0, z=0.0):
    return np.array([x, y, z], dtype=np.float64)


@dataclass
class SceneConfig:
    """Scene tunables; field names/defaults are the reference's (mesh.py:58-94)."""

    mesh_path: str = ""
    total_mass: float = 0.08
    dt: float = 0.01
    substeps: int = 10
    gravity: np.ndarray = field(default_factory=lambda: _v3(0.0, -9.81, 0.0))
    k_s: float = 1.0
    k_v: float = 0.9
    damping: float = 0.0
    rcm: np.ndarray = field(default_factory=lambda: _v3(0.04875, 0.09, 0.0225))
    tool_start: np.ndarray = field(default_factory=lambda: _v3(0.04875, 0.03, 0.0225))
    shaft_radius: float = 0.003
    clamp_radius: float = 0.002
    clamp_length: float = 0.008
    clamp_angle: float = 2.0
    grasp_radius: float = 0.005
    target: np.ndarray = field(default_factory=lambda: _v3(0.075, 0.0, 0.030))
    action_scale: float = 0.004
    max_episode_steps: int = 100
    success_threshold: float = 0.003
    reward_distance_weight: float = -1.0
    reward_delta_weight: float = -10.0
    reward_success_weight: float = 100.0
    reward_scale: float = 1.0
    workspace_low: np.ndarray = field(default_factory=lambda: _v3(-0.01, -0.01, -0.01))
    workspace_high: np.ndarray = field(default_factory=lambda: _v3(0.11, 0.08, 0.055))
    attachments: list = field(default_factory=list)

    def validate(self):
        """Range checks of mesh.py:96-128 (same messages)."""
        checks = [
            (self.dt <= 0.0, "dt must be positive"),
            (self.substeps < 1, "substeps must be >= 1"),
            (self.damping < 0.0, "damping must be >= 0"),
            (self.total_mass <= 0.0, "total_mass must be positive"),
        ]
        for bad, msg in checks:
            if bad:
                raise ValidationError(msg)
        for name in ("k_s", "k_v"):
            val = getattr(self, name)
            if not 0.0 <= val <= 1.0:
                raise ValidationError(f"{name} must lie in [0, 1], got {val}")
        if self.damping < 0.0:
            raise ValidationError("damping must be >= 0")
        if not 0.0 < self.clamp_angle < 30.0:
            raise ValidationError("clamp_angle must lie in (0, 30) degrees")
        if self.grasp_radius <= 0.0:
            raise ValidationError("grasp_radius must be positive")
        if min(self.shaft_radius, self.clamp_radius, self.clamp_length) <= 0.0:
            raise ValidationError("tool capsule dimensions must be positive")
        if self.success_threshold <= 0.0:
            raise ValidationError("success_threshold must be positive")
        if self.max_episode_steps < 1:
            raise ValidationError("max_episode_steps must be >= 1")
        if self.action_scale <= 0.0:
            raise ValidationError("action_scale must be positive")
        if not np.all(np.asarray(self.workspace_low) < np.asarray(self.workspace_high)):
            raise ValidationError("workspace_low must be strictly below workspace_high")
        for att in self.attachments:
            if att.rest < 0.0:
                raise ValidationError("attachment rest distance must be >= 0")
            if not 0.0 <= att.stiffness <= 1.0:
                raise ValidationError("attachment stiffness must lie in [0, 1]")
        return self


# ---------------------------------------------------------------------------
# topology
# ---------------------------------------------------------------------------

def derive_topology(tets):
    """(edges (E,2), surface faces (F,3)) of a tet soup, reference ordering."""
    tets = np.asarray(tets, dtype=np.int64).reshape(-1, 4)
    if len(tets) == 0:
        return np.zeros((0, 2), np.int32), np.zeros((0, 3), np.int32)
    base = int(tets.max()) + 1

    # edges: one key per sorted pair; np.unique sorts keys == lexicographic rows
    ea = np.concatenate([tets[:, i] for i, _ in TET_EDGE_CORNERS])
    eb = np.concatenate([tets[:, j] for _, j in TET_EDGE_CORNERS])
    lo, hi = np.minimum(ea, eb), np.maximum(ea, eb)
    ekeys = np.unique(lo * base + hi)
    edges = np.stack([ekeys // base, ekeys % base], axis=1)

    # faces: wound triples, keyed by their sorted triple; boundary = seen once
    wound = np.concatenate([tets[:, list(c)] for c in TET_FACE_CORNERS], axis=0)
    srt = np.sort(wound, axis=1)
    fkeys = (srt[:, 0] * base + srt[:, 1]) * base + srt[:, 2]
    uniq, first, counts = np.unique(fkeys, return_index=True, return_counts=True)
    surface = wound[first[counts == 1]]
    return edges.astype(np.int32), surface.astype(np.int32)


def signed_volumes(positions, tets):
    """(b-a)x(c-a).(d-a)/6 per tet, same numpy reductions as mesh.py:162-164."""
    p = np.asarray(positions, dtype=np.float64)
    t = np.asarray(tets).reshape(-1, 4)
    a, b, c, d = (p[t[:, k]] for k in range(4))
    return np.einsum("ij,ij->i", np.cross(b - a, c - a), d - a) / 6.0


def fix_orientation(positions, tets):
    """Swap corners 2 and 3 of every negatively oriented tet."""
    t = np.asarray(tets, dtype=np.int32).reshape(-1, 4).copy()
    if len(t):
        neg = signed_volumes(positions, t) < 0.0
        t[neg] = t[neg][:, [0, 1, 3, 2]]
    return t


def compute_rest_state(mesh: TetMesh) -> RestState:
    pos = mesh.positions_rest
    if len(mesh.edges):
        rest_length = np.linalg.norm(pos[mesh.edges[:, 0]] - pos[mesh.edges[:, 1]], axis=1)
        if np.any(rest_length <= 0.0):
            raise ValidationError("degenerate edge with zero rest length")
    else:
        rest_length = np.zeros(0)
    rest_volume = signed_volumes(pos, mesh.tets) if len(mesh.tets) else np.zeros(0)
    if np.any(np.abs(rest_volume) < MIN_TET_VOLUME):
        k = int(np.argmin(np.abs(rest_volume)))
        raise ValidationError(f"degenerate tetrahedron {k} (|volume| < {MIN_TET_VOLUME})")
    if np.any(rest_volume <= 0.0):
        raise ValidationError("negatively oriented tetrahedron; run fix_orientation first")
    massless = np.setdiff1d(np.flatnonzero(mesh.vertex_mass <= 0.0), mesh.pinned)
    if len(massless):
        raise ValidationError(f"free vertex {int(massless[0])} has non-positive mass")
    inv = np.zeros(mesh.vertex_count)
    pos_mass = mesh.vertex_mass > 0.0
    inv[pos_mass] = 1.0 / mesh.vertex_mass[pos_mass]
    inv[mesh.pinned] = 0.0
    return RestState(rest_length, rest_volume, inv)


def build_mesh(positions, tets, pinned=(), total_mass=0.08) -> TetMesh:
    positions = np.ascontiguousarray(positions, dtype=np.float64).reshape(-1, 3)
    nv = len(positions)
    t = np.asarray(tets, dtype=np.int64).reshape(-1, 4)
    if len(t) and (t.min() < 0 or t.max() >= nv):
        raise ValidationError(f"tet vertex index out of range [0, {nv})")
    if len(t) and np.any(np.sort(t, axis=1)[:, 1:] == np.sort(t, axis=1)[:, :-1]):
        raise ValidationError("tetrahedron with repeated vertex index")
    pins = np.array(sorted({int(i) for i in pinned}), dtype=np.int32)
    if len(pins) and (pins.min() < 0 or pins.max() >= nv):
        raise ValidationError(f"pinned vertex index out of range [0, {nv})")
    t = fix_orientation(positions, t.astype(np.int32))
    edges, surface = derive_topology(t)
    mass = np.full(nv, total_mass / nv) if nv else np.zeros(0)
    return TetMesh(nv, positions, t, edges, surface, pins, mass)


# ---------------------------------------------------------------------------
# text formats
# ---------------------------------------------------------------------------

def _lines(text):
    for num, raw in enumerate(text.splitlines(), start=1):
        body = raw.split("#", 1)[0].strip()
        if body:
            yield num, body


def parse_mesh_text(text: str):
    """``tetmesh 1`` / counts / V vertex lines / T tet lines / optional ``pinned k i..``."""
    rows = list(_lines(text))
    if not rows or rows[0][1].split() != ["tetmesh", "1"]:
        raise ParseError("mesh file must start with header 'tetmesh 1'")
    if len(rows) < 2:
        raise ParseError("mesh file missing counts line")
    num, counts = rows[1][0], rows[1][1].split()
    if not 2 <= len(counts) <= 4:
        raise ParseError(f"line {num}: counts line needs 2-4 integers")
    try:
        nv, nt = int(counts[0]), int(counts[-1])
    except ValueError as exc:
        raise ParseError(f"line {num}: bad counts line") from exc
    if nv < 0 or nt < 0:
        raise ParseError("negative counts")
    body = rows[2:]
    if len(body) < nv + nt:
        raise ParseError(f"expected {nv} vertex and {nt} tet lines, found {len(body)}")
    try:
        pos = np.array([[float(tok) for tok in body[i][1].split()] for i in range(nv)],
                       dtype=np.float64).reshape(nv, 3)
    except ValueError as exc:
        raise ParseError("bad vertex line (need 3 floats)") from exc
    try:
        tets = np.array([[int(tok) for tok in body[nv + i][1].split()] for i in range(nt)],
                        dtype=np.int64).reshape(nt, 4)
    except ValueError as exc:
        raise ParseError("bad tet line (need 4 indices)") from exc
    pinned: list[int] = []
    for num, line in body[nv + nt:]:
        tok = line.split()
        if tok[0] != "pinned":
            raise ParseError(f"line {num}: unexpected trailing line {tok[0]!r}")
        try:
            k = int(tok[1])
            ids = [int(s) for s in tok[2:]]
        except (IndexError, ValueError) as exc:
            raise ParseError(f"line {num}: bad pinned line") from exc
        if len(ids) != k:
            raise ParseError(f"line {num}: pinned count {k} != {len(ids)} indices")
        pinned += ids
    return pos, tets, pinned


_FLOAT_KEYS = frozenset({
    "total_mass", "dt", "k_s", "k_v", "damping", "shaft_radius", "clamp_radius",
    "clamp_length", "clamp_angle", "grasp_radius", "action_scale", "success_threshold",
    "reward_distance_weight", "reward_delta_weight", "reward_success_weight", "reward_scale",
})
_INT_KEYS = frozenset({"substeps", "max_episode_steps"})
_VEC_KEYS = frozenset({"gravity", "rcm", "tool_start", "target", "workspace_low", "workspace_high"})


def parse_scene_text(text: str, base_dir: str = ".") -> SceneConfig:
    cfg = SceneConfig()
    for num, line in _lines(text):
        if "=" not in line:
            raise ParseError(f"line {num}: expected 'key = value'")
        key, value = (s.strip() for s in line.split("=", 1))
        try:
            if key == "mesh":
                cfg.mesh_path = os.path.normpath(os.path.join(base_dir, value))
            elif key in _FLOAT_KEYS:
                setattr(cfg, key, float(value))
            elif key in _INT_KEYS:
                setattr(cfg, key, int(value))
            elif key in _VEC_KEYS:
                vec = [float(s) for s in value.split()]
                if len(vec) != 3:
                    raise ParseError(f"line {num}: {key} needs 3 components")
                setattr(cfg, key, np.array(vec))
            elif key == "attach_anchor":
                v, x, y, z, rest, k = value.split()
                cfg.attachments.append(AttachmentSpec(int(v), None, np.array([float(x), float(y), float(z)]),
                                                      float(rest), float(k)))
            elif key == "attach_face":
                v, f, rest, k = value.split()
                cfg.attachments.append(AttachmentSpec(int(v), int(f), None, float(rest), float(k)))
            else:
                raise ParseError(f"line {num}: unknown key {key!r}")
        except ParseError:
            raise
        except ValueError as exc:
            raise ParseError(f"line {num}: bad value for {key!r}: {value!r}") from exc
    return cfg


def load_mesh(path: str, total_mass: float = 0.08) -> TetMesh:
    if not os.path.exists(path):
        raise ParseError(f"mesh file not found: {path}")
    with open(path, encoding="utf-8") as fh:
        pos, tets, pinned = parse_mesh_text(fh.read())
    return build_mesh(pos, tets, pinned, total_mass)


def load_scene(path: str):
    """(TetMesh, RestState, SceneConfig) from a scene file (mesh.py:508-524)."""
    if not os.path.exists(path):
        raise ParseError(f"scene file not found: {path}")
    with open(path, encoding="utf-8") as fh:
        cfg = parse_scene_text(fh.read(), base_dir=os.path.dirname(os.path.abspath(path)))
    cfg.validate()
    if not cfg.mesh_path:
        raise ParseError("scene file does not name a mesh")
    mesh = load_mesh(cfg.mesh_path, cfg.total_mass)
    for att in cfg.attachments:
        if not 0 <= att.vertex < mesh.vertex_count:
            raise ValidationError(f"attachment vertex {att.vertex} out of range")
        if att.face is not None and not 0 <= att.face < len(mesh.surface_faces):
            raise ValidationError(f"attachment face {att.face} out of range")
    return mesh, compute_rest_state(mesh), cfg


def write_mesh(path, positions, tets, pinned=()):
    p = np.asarray(positions, dtype=np.float64).reshape(-1, 3)
    t = np.asarray(tets, dtype=np.int64).reshape(-1, 4)
    out = ["tetmesh 1", f"{len(p)} {len(t)}"]
    out += [f"{float(a)!r} {float(b)!r} {float(c)!r}" for a, b, c in p]
    out += [f"{a} {b} {c} {d}" for a, b, c, d in t]
    pins = sorted({int(i) for i in pinned})
    if pins:
        out.append(f"pinned {len(pins)} " + " ".join(map(str, pins)))
    with open(path, "w", encoding="utf-8") as fh:
        fh.write("\n".join(out) + "\n")


def write_scene(path, cfg: SceneConfig, mesh_name=None):
    base = os.path.dirname(os.path.abspath(path))
    rel = mesh_name if mesh_name is not None else os.path.relpath(cfg.mesh_path, base)
    out = [f"mesh = {rel}"]
    for f in fields(SceneConfig):
        if f.name in ("mesh_path", "attachments"):
            continue
        val = getattr(cfg, f.name)
        if f.name in _VEC_KEYS:
            out.append(f"{f.name} = {float(val[0])!r} {float(val[1])!r} {float(val[2])!r}")
        elif f.name in _INT_KEYS:
            out.append(f"{f.name} = {val}")
        else:
            out.append(f"{f.name} = {float(val)!r}")
    for att in cfg.attachments:
        if att.face is not None:
            out.append(f"attach_face = {att.vertex} {att.face} {float(att.rest)!r} {float(att.stiffness)!r}")
        else:
            a = att.anchor
            out.append(f"attach_anchor = {att.vertex} {float(a[0])!r} {float(a[1])!r} {float(a[2])!r} "
                       f"{float(att.rest)!r} {float(att.stiffness)!r}")
    with open(path, "w", encoding="utf-8") as fh:
        fh.write("\n".join(out) + "\n")


# ---------------------------------------------------------------------------
# slab fixtures (the benchmark scene generator)
# ---------------------------------------------------------------------------

SLAB_PRESETS = {1170: (13, 3, 6), 1431: (13, 2, 11), 2880: (12, 4, 12),
                9729: (18, 6, 18), 52359: (34, 11, 28)}
# corner bit patterns (ijk) of the 5-tet split of an even cell; odd cells mirror i
_CELL_EVEN = ((4, 2, 1, 7), (0, 4, 2, 1), (6, 4, 2, 7), (5, 4, 1, 7), (3, 2, 1, 7))
_CELL_ODD = tuple(tuple(c ^ 4 for c in tet) for tet in _CELL_EVEN)
TISSUE_DENSITY = 1050.0


def make_slab(nx, ny, nz, spacing, origin=(0.0, 0.0, 0.0)):
    """Conforming 5-tets-per-cube slab (alternating cell parity)."""
    if min(nx, ny, nz) < 1 or spacing <= 0.0:
        raise ValidationError("slab dimensions must be positive")
    gy, gz = ny + 1, nz + 1
    ii, jj, kk = np.meshgrid(np.arange(nx + 1), np.arange(gy), np.arange(gz), indexing="ij")
    pos = np.stack([ii, jj, kk], axis=-1).reshape(-1, 3) * spacing + np.asarray(origin)
    ci, cj, ck = (a.ravel() for a in np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij"))
    corner = np.stack([((ci + (b >> 2 & 1)) * gy + (cj + (b >> 1 & 1))) * gz + (ck + (b & 1))
                       for b in range(8)], axis=1)
    even = ((ci + cj + ck) % 2 == 0)[:, None, None]
    pat = np.where(even, np.array(_CELL_EVEN)[None], np.array(_CELL_ODD)[None])
    tets = np.take_along_axis(corner[:, None, :].repeat(5, axis=1), pat, axis=2).reshape(-1, 4)
    return pos.astype(np.float64), tets.astype(np.int64)


def slab_pins(nx, ny, nz, side="x0"):
    gx, gy, gz = nx + 1, ny + 1, nz + 1
    i, j, k = (a.ravel() for a in np.meshgrid(np.arange(gx), np.arange(gy), np.arange(gz), indexing="ij"))
    sel = {"x0": i == 0, "x1": i == gx - 1, "y0": j == 0, "y1": j == gy - 1}[side]
    return [int(v) for v in ((i * gy + j) * gz + k)[sel]]


def slab_preset(target_tets):
    if target_tets not in SLAB_PRESETS:
        raise ValidationError(f"no slab preset near {target_tets} tets; have {sorted(SLAB_PRESETS)}")
    return SLAB_PRESETS[target_tets]


def make_slab_scene(out_dir, tets=1170, spacing=0.0075, pin="y0", name=None, **overrides):
    nx, ny, nz = slab_preset(tets)
    pos, tet_arr = make_slab(nx, ny, nz, spacing, origin=(0.0, -ny * spacing, 0.0))
    name = name or f"slab_{5 * nx * ny * nz}"
    os.makedirs(out_dir, exist_ok=True)
    mesh_path = os.path.join(out_dir, f"{name}.mesh")
    write_mesh(mesh_path, pos, tet_arr, slab_pins(nx, ny, nz, pin))
    length, width, depth = nx * spacing, nz * spacing, ny * spacing
    margin = 0.15 * length
    cx, cz = 0.5 * length, 0.5 * width
    cfg = SceneConfig(
        mesh_path=mesh_path, total_mass=length * width * depth * TISSUE_DENSITY,
        rcm=_v3(cx, 0.9 * length, cz), tool_start=_v3(cx, 0.3 * length, cz),
        target=_v3(0.75 * length, 0.0, 2.0 * width / 3.0),
        workspace_low=_v3(-margin, -depth - margin, -margin),
        workspace_high=_v3(length + margin, 0.675 * length, width + margin), damping=1.0)
    for key, value in overrides.items():
        if not hasattr(cfg, key):
            raise ValidationError(f"unknown scene override {key!r}")
        setattr(cfg, key, value)
    cfg.validate()
    path = os.path.join(out_dir, f"{name}.scene")
    write_scene(path, cfg, mesh_name=os.path.basename(mesh_path))
    return path


def default_scene_path():
    """reach_1170.scene shipped in-tree (byte-identical to the reference's pkg/scenes)."""
    return os.path.join(os.path.dirname(os.path.abspath(__file__)), "scenes", "reach_1170.scene")
