"""Generate the golden fixtures in tests/golden/ from the UNMODIFIED reference.

Run in the build container after ``oracle/build_ref.sh`` (which builds the
reference's compiled backend into oracle/_ref/):

    python tests/golden/make_golden.py

The reference is only imported here; the fixtures it writes are what the
tests (and the GPU box, which has no /root/reference) compare against.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))

from tissuesim import backends  # noqa: E402
from tissuesim.env import EnvBatch  # noqa: E402
from tissuesim.mesh import (SceneConfig, build_mesh, compute_rest_state, load_scene, make_slab,  # noqa: E402
                            slab_pins, AttachmentSpec)
from tissuesim.solver import Simulation  # noqa: E402

SCENE = os.path.join(ROOT, "paper_2503_18616_b200", "scenes", "reach_1170.scene")


def small_slab(nx=3, ny=2, nz=2, spacing=0.01, pin="x0", total_mass=0.05, with_attachments=False, **over):
    """Same construction as the reference's test fixture (pkg/tests/conftest.py:10-39)."""
    origin = (0.0, -ny * spacing, 0.0)
    positions, tets = make_slab(nx, ny, nz, spacing, origin=origin)
    pins = slab_pins(nx, ny, nz, pin) if pin else []
    mesh = build_mesh(positions, tets, pins, total_mass=total_mass)
    length = nx * spacing
    cfg = SceneConfig(total_mass=total_mass,
                      rcm=np.array([length / 2, 0.9 * length, nz * spacing / 2]),
                      tool_start=np.array([length / 2, 0.3 * length, nz * spacing / 2]),
                      target=np.array([0.75 * length, 0.0, nz * spacing / 2]),
                      workspace_low=np.array([-0.2 * length, -ny * spacing - 0.2 * length, -0.2 * length]),
                      workspace_high=np.array([1.2 * length, 0.675 * length, nz * spacing * 1.4]),
                      damping=1.0)
    if with_attachments:
        free = int(np.setdiff1d(np.arange(mesh.vertex_count), mesh.pinned)[0])
        cfg.attachments = [
            AttachmentSpec(vertex=free, anchor=positions[free] + [0.0, 0.004, 0.0], rest=0.002, stiffness=0.6),
            AttachmentSpec(vertex=int(mesh.surface_faces[0, 0]), face=len(mesh.surface_faces) - 1,
                           rest=0.01, stiffness=0.4),
        ]
    for k, v in over.items():
        setattr(cfg, k, v)
    cfg.validate()
    return mesh, compute_rest_state(mesh), cfg


def topology(path):
    m, r, c = load_scene(SCENE)
    out = dict(positions_rest=m.positions_rest, tets=m.tets, edges=m.edges, surface_faces=m.surface_faces,
               pinned=m.pinned, vertex_mass=m.vertex_mass, rest_length=r.rest_length,
               rest_volume=r.rest_volume, inverse_mass=r.inverse_mass)
    m2, r2, _ = small_slab(with_attachments=True)
    out.update({f"small_{k}": v for k, v in dict(tets=m2.tets, edges=m2.edges, faces=m2.surface_faces,
                                                  rest_length=r2.rest_length, rest_volume=r2.rest_volume).items()})
    rng = np.random.default_rng(0)
    soup = rng.integers(0, 30, size=(40, 4))
    soup = soup[np.array([len(set(t)) == 4 for t in soup.tolist()])]
    from tissuesim.mesh import derive_topology
    e, f = derive_topology(soup)
    out.update(soup_tets=soup, soup_edges=e, soup_faces=f)
    np.savez_compressed(path, **out)


def trajectory(path, n=8, steps=100, seed=5):
    """EnvBatch rollout with the reference's bench protocol actions (cli.py:70-81)."""
    env = EnvBatch(SCENE, num_envs=n, seed=seed, backend="compiled", threads=1)
    poses = []
    orig = env.sim.tool.apply_commands

    def wrapped(targets, angles):
        res = orig(targets, angles)
        t = env.sim.tool
        poses.append(np.concatenate([t.axis, t.jaw_dir, t.reach[:, None], t.clamp_angle[:, None],
                                     res[0][:, None].astype(np.float64)], axis=1))
        return res
    env.sim.tool.apply_commands = wrapped
    obs0 = env.reset(seed=seed)
    rng = np.random.default_rng(seed)
    rec = {k: [] for k in ("actions", "obs", "reward", "terminated", "truncated", "distance", "grasp_vertex",
                           "contacts", "episode_length", "episode_return", "done_mask")}
    snaps = {}
    for s in range(steps):
        a = rng.uniform(-1.0, 1.0, (n, 3))
        obs, r, te, tr, info = env.step(a)
        for k, v in (("actions", a), ("obs", obs), ("reward", r), ("terminated", te), ("truncated", tr),
                     ("distance", info["distance"]), ("grasp_vertex", env.sim.grasp_vertex.copy()),
                     ("contacts", info["contacts"]), ("episode_length", info["episode_length"]),
                     ("episode_return", info["episode_return"]), ("done_mask", info["done_mask"])):
            rec[k].append(np.asarray(v))
        if s in (0, 9, 49, 98):
            snaps[f"x_{s}"] = env.sim.x.copy()
            snaps[f"v_{s}"] = env.sim.v.copy()
    np.savez_compressed(path, obs0=obs0, poses=np.stack(poses), **{k: np.stack(v) for k, v in rec.items()},
                        **snaps)


def kernels(path):
    """Plugin-level KATs of the compiled backend: run_substeps (with attachments + grasp) and detect_contacts."""
    kb = backends.get_backend("compiled")
    mesh, rest, cfg = small_slab(3, 2, 2, damping=0.6, with_attachments=True)
    cfg.substeps = 4
    sim = Simulation(mesh, rest, cfg, num_instances=3, backend="compiled")
    rng = np.random.default_rng(5)
    sim.v[:] = rng.normal(0, 0.03, sim.v.shape) * (sim.w[None, :, None] > 0)
    free = np.setdiff1d(np.arange(mesh.vertex_count), mesh.pinned)
    sim.grasp_vertex[:] = [int(free[-1]), -1, int(free[3])]
    x0, v0 = sim.x.copy(), sim.v.copy()
    drag = sim.tool.drag_points().copy()
    out = dict(x0=x0, v0=v0, grasp_vertex=sim.grasp_vertex.copy(), drag=drag, w=sim.w,
               edges=sim.edges, rest_length=sim.rest_length, tets=sim.tets, rest_volume=sim.rest_volume,
               att_vertex=sim.att_vertex, att_faces=sim.att_faces, att_is_face=sim.att_is_face,
               att_anchor=sim.att_anchor, att_rest=sim.att_rest, att_k=sim.att_k,
               ks=cfg.k_s, kv=cfg.k_v, g=sim.params.gravity, h=sim.params.h, substeps=cfg.substeps,
               damping=cfg.damping)
    for rep in range(3):
        kb.run_substeps(sim.x, sim.v, sim.w, sim.edges, sim.rest_length, cfg.k_s, sim.tets, sim.rest_volume,
                        cfg.k_v, sim.att_vertex, sim.att_faces, sim.att_is_face, sim.att_anchor, sim.att_rest,
                        sim.att_k, sim.grasp_vertex, drag, sim.params.gravity, sim.params.h, cfg.substeps,
                        cfg.damping, sim._acc, sim._cnt, 1, False, sim._scratch)
        out[f"x_{rep}"] = sim.x.copy()
        out[f"v_{rep}"] = sim.v.copy()
    # contact detection: random triangles against random capsules (test_collision.py:79-97 style)
    rng = np.random.default_rng(14)
    cases = []
    for k in range(40):
        pos = rng.normal(0, 0.2, (9, 3))
        faces = np.array([[0, 1, 2], [3, 4, 5], [6, 7, 8]], dtype=np.int32)
        caps = np.concatenate([rng.normal(0, 0.2, (3, 6)), np.full((3, 1), 0.15)], axis=1)
        res = kb.detect_contacts(np.ascontiguousarray(pos), faces, np.ascontiguousarray(caps), 8)
        out[f"c{k}_pos"] = pos
        out[f"c{k}_caps"] = caps
        for name, arr in zip(("face", "cap", "depth", "dir", "bary"), res):
            out[f"c{k}_{name}"] = arr
        cases.append(len(res[0]))
    out["contact_faces"] = faces
    out["n_contact_cases"] = 40
    np.savez_compressed(path, **out)
    return cases


if __name__ == "__main__":
    assert backends.HAVE_COMPILED, "build the reference first: bash oracle/build_ref.sh"
    topology(os.path.join(HERE, "topology.npz"))
    trajectory(os.path.join(HERE, "trajectory_reach1170_n8_seed5.npz"))
    print("contact rows per case:", kernels(os.path.join(HERE, "kernels.npz")))
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))
