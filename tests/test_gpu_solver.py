"""Simulation-level known answers on the GPU, ported from pkg/tests/test_solver.py, test_tool.py and
test_acceptance.py (P3, P5, P7), run through the sm_100a kernel."""

import numpy as np
import pytest
import torch

import oracle as O
from conftest import build_slab_scene, free_particles_scene
from paper_2503_18616_b200 import Simulation
from paper_2503_18616_b200.errors import SimulationDiverged
from paper_2503_18616_b200.mesh import RestState, SceneConfig, TetMesh, compute_rest_state

pytestmark = pytest.mark.gpu


def np_(t):
    return t.cpu().numpy()


def edge_only_scene(length=2.0, rest=1.0, wa=1.0, wb=1.0, pinned=()):
    positions = np.array([[0.0, 0.0, 0.0], [length, 0.0, 0.0]])
    mesh = TetMesh(vertex_count=2, positions_rest=positions, tets=np.zeros((0, 4), np.int32),
                   edges=np.array([[0, 1]], np.int32), surface_faces=np.zeros((0, 3), np.int32),
                   pinned=np.array(sorted(pinned), np.int32),
                   vertex_mass=np.array([1.0 / wa if wa else 1.0, 1.0 / wb if wb else 1.0]))
    inv = np.array([wa, wb], dtype=float)
    inv[mesh.pinned] = 0.0
    cfg = SceneConfig(dt=0.01, substeps=1, gravity=np.zeros(3), damping=0.0,
                      rcm=np.array([50.0, 50.0, 50.0]), tool_start=np.array([50.0, 49.0, 50.0]),
                      target=np.array([50.0, 48.9, 50.0]), workspace_low=np.array([40.0, 40.0, 40.0]),
                      workspace_high=np.array([60.0, 49.5, 60.0]))
    return mesh, RestState(np.array([rest]), np.zeros(0), inv), cfg


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
@pytest.mark.parametrize("substeps", [1, 5, 10])
def test_free_fall_closed_form(substeps, precision):
    mesh, rest, cfg = free_particles_scene([[0.0, 0.5, 0.0]], substeps=substeps)
    sim = Simulation(mesh, rest, cfg, device="cuda:0", precision=precision)
    sim.step()
    dt, n = cfg.dt, substeps
    tol = 1e-12 if precision == "fp64" else 1e-7
    assert np_(sim.v)[0, 0, 1] == pytest.approx(-9.81 * dt, abs=tol)
    assert np_(sim.x)[0, 0, 1] == pytest.approx(0.5 - 9.81 * dt * dt * (n + 1) / (2 * n), abs=tol)


def test_all_pinned_mesh_static():
    mesh, rest, cfg = build_slab_scene(2, 1, 2)
    mesh.pinned = np.arange(mesh.vertex_count, dtype=np.int32)
    rest = compute_rest_state(mesh)
    sim = Simulation(mesh, rest, cfg, device="cuda:0", precision="fp64")
    x0 = np_(sim.x).copy()
    for _ in range(5):
        sim.step()
    assert np.array_equal(np_(sim.x), x0) and not np_(sim.v).any()


def test_stretched_pair_restores_rest_length():
    mesh, rest, cfg = edge_only_scene()
    sim = Simulation(mesh, rest, cfg, device="cuda:0", precision="fp64")
    sim.step()
    assert abs(np.linalg.norm(np_(sim.x)[0, 0] - np_(sim.x)[0, 1]) - 1.0) < 1e-9


def test_divergence_raises_with_step():
    mesh, rest, cfg = free_particles_scene([[0.0, 0.5, 0.0]])
    sim = Simulation(mesh, rest, cfg, device="cuda:0")
    sim.step()
    sim.v[0, 0, 0] = float("inf")
    with pytest.raises(SimulationDiverged) as err:
        sim.step()
    assert err.value.step == 2


def test_divergence_mask_mode():
    mesh, rest, cfg = free_particles_scene([[0.0, 0.5, 0.0], [1.0, 0.5, 0.0]])
    sim = Simulation(mesh, rest, cfg, num_instances=2, device="cuda:0")
    sim.v[1, 0, 0] = float("nan")
    info = sim.step(raise_on_divergence=False)
    assert np_(info["diverged"]).tolist() == [False, True]


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_pinned_bitwise_constant(precision):
    mesh, rest, cfg = build_slab_scene(3, 2, 2)
    sim = Simulation(mesh, rest, cfg, device="cuda:0", precision=precision)
    rng = np.random.default_rng(6)
    pinned_rest = np_(sim.x)[0, mesh.pinned].copy()
    for _ in range(50):
        sim.step(np_(sim.tool.drag_points()) + rng.normal(0, 0.002, (1, 3)))
    assert np.array_equal(np_(sim.x)[0, mesh.pinned], pinned_rest)
    assert not np_(sim.v)[0, mesh.pinned].any()


@pytest.mark.parametrize("cluster", [0, 2], ids=["one-cta", "cluster2"])
def test_sim_with_attachments_matches_oracle_bitwise(cluster):
    """Attachment constraints (vertex-anchor and vertex-face) run through the kernel bitwise vs the
    oracle -- also split over a 2-CTA cluster (attachment slots only for owned vertices)."""
    scene = build_slab_scene(3, 2, 2, damping=0.8, with_attachments=True)
    n = 2
    sim = Simulation(*scene, num_instances=n, device="cuda:0", precision="fp64",
                     layout={"cluster_size": cluster} if cluster else None)
    ref = O.OracleEnv(O.scene_from_loaded(*scene), n)
    rng = np.random.default_rng(19)
    for _ in range(60):
        targets = ref.drag_points() + rng.normal(0, 0.002, (n, 3))
        ref.sim_step(targets.copy())
        sim.step(targets, tool_override=ref.last_cmd)
        assert np.array_equal(np_(sim.x), ref.x) and np.array_equal(np_(sim.v), ref.v)
        assert np.array_equal(np_(sim.grasp_vertex), ref.grasp_vertex)


def test_full_grasp_drag_release_cycle():
    mesh, rest, cfg = build_slab_scene(3, 2, 2, pin="y0", damping=1.0)
    cfg.clamp_angle = 2.0
    sim = Simulation(mesh, rest, cfg, device="cuda:0", precision="fp64")
    top = float(mesh.positions_rest[:, 1].max())
    for _ in range(60):
        drag = np_(sim.tool.drag_points())
        sim.step(np.array([[0.015, max(top + 0.001, drag[0, 1] - 0.003), 0.01]]))
        if int(sim.grasp_vertex[0]) >= 0:
            break
    held = int(sim.grasp_vertex[0])
    assert held >= 0 and int(sim.grasped[0, held]) == 1
    for _ in range(12):
        sim.step(np_(sim.tool.drag_points()) + [[0.0, 0.0015, 0.0]])
    assert int(sim.grasp_vertex[0]) == held
    assert np.linalg.norm(np_(sim.x)[0, held] - np_(sim.tool.drag_points())[0]) < 0.02
    lifted = np_(sim.x)[0, held, 1]
    assert lifted > top + 0.002
    sim.step(np_(sim.tool.drag_points()), angles=np.array([10.0]))
    assert int(sim.grasp_vertex[0]) == -1 and int(sim.grasped[0, held]) == 0
    for _ in range(120):
        sim.step()
    assert np_(sim.x)[0, held, 1] < lifted


def test_grasped_vertex_tracks_drag_point():
    """Plugin-level: one substep with only the grasp constraint puts the vertex on the drag point."""
    from paper_2503_18616_b200 import backend
    mesh, rest, cfg = build_slab_scene(3, 2, 2)
    free = int(np.setdiff1d(np.arange(mesh.vertex_count), mesh.pinned)[0])
    x = mesh.positions_rest[None].copy()
    v = np.zeros_like(x)
    drag = x[0, free] + np.array([[0.002, 0.001, -0.001]])
    backend.run_substeps(x, v, rest.inverse_mass, np.zeros((0, 2), np.int32), np.zeros(0), 1.0,
                         np.zeros((0, 4), np.int32), np.zeros(0), 1.0, np.zeros(0, np.int32),
                         np.zeros((0, 3), np.int32), np.zeros(0, np.uint8), np.zeros((0, 3)), np.zeros(0),
                         np.zeros(0), np.array([free]), drag, np.zeros(3), cfg.dt, 1, 0.0)
    assert np.linalg.norm(x[0, free] - drag[0]) < 1e-9


def test_p7_slab_settles():
    """Acceptance P7 (test_acceptance.py:170-183): 2000 steps, KE < 1e-8 J, all finite."""
    from paper_2503_18616_b200.mesh import load_scene, make_slab_scene
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        mesh, rest, cfg = load_scene(make_slab_scene(d, tets=1170, pin="x0", name="stab"))
    sim = Simulation(mesh, rest, cfg, device="cuda:0", precision="fp64")
    for _ in range(2000):
        sim.step(raise_on_divergence=False)
    assert torch.isfinite(sim.x).all()
    assert float(sim.kinetic_energy()[0]) < 1e-8


def test_kinetic_energy_matches_definition(small_scene):
    sim = Simulation(*small_scene, num_instances=2, device="cuda:0", precision="fp64")
    sim.step()
    v = np_(sim.v)
    ke = 0.5 * np.einsum("nvq,nvq->nv", v, v) @ small_scene[0].vertex_mass
    assert np.allclose(np_(sim.kinetic_energy()), ke, rtol=1e-12)


@pytest.mark.gpu
def test_tool_command_edge_cases_match_oracle(reach_scene):
    """test_tool.py's command cases on the device command kernel (Simulation.step(targets, angles)):
    identity command, pure advance along the axis, lateral reach, workspace clip, the trocar
    singularity (target at the RCM: rejected, pose held), a sub-threshold rotation (reach changes,
    axis kept) and a quarter turn -- flags exact, pose within 1e-12 of the numpy oracle."""
    import oracle as O
    from paper_2503_18616_b200 import EnvBatch
    import dataclasses
    mesh, rest, cfg = reach_scene
    # the workspace box of the reach scene excludes the RCM; widen it so the singularity is reachable
    cfg = dataclasses.replace(cfg, workspace_high=np.array([0.11, 0.10, 0.055]))
    scene = (mesh, rest, cfg)
    env = EnvBatch(scene, num_envs=7, device="cuda:0", precision="fp64")
    env.reset()
    ref = O.OracleEnv(O.scene_from_loaded(*scene), 7)
    ref.reset()
    rcm = np.asarray(cfg.rcm, np.float64)
    drag = ref.drag_points().copy()
    ax0 = ref.axis[0].copy()
    side = np.cross(ax0, [0.0, 0.0, 1.0])
    side /= np.linalg.norm(side)
    targets = np.stack([
        drag[0],                                   # identity
        drag[1] + 0.005 * ax0,                     # pure advance
        drag[2] + 0.004 * side,                    # lateral reach
        np.array([0.5, -0.5, 0.2]),                # far outside the workspace: clipped
        rcm,                                       # trocar singularity: rejected
        drag[5] + 1e-13 * side,                    # rotation below MIN_ROTATION
        rcm + np.linalg.norm(drag[6] - rcm) * side,  # quarter turn
    ])
    angles = np.array([2.0, 2.0, 5.0, 2.0, 7.0, 2.0, 1.0])
    info = env.sim.step(targets=targets, angles=angles)
    r_clipped, r_rejected = ref.apply_commands(targets, angles)
    assert np.array_equal(info["clipped"].cpu().numpy(), r_clipped)
    assert np.array_equal(info["rejected"].cpu().numpy(), r_rejected)
    assert r_rejected[4] and not r_rejected[:4].any() and r_clipped[3]
    t = env.sim.tool
    for got, want in ((t.axis, ref.axis), (t.jaw_dir, ref.jaw), (t.reach, ref.reach), (t.clamp_angle, ref.clamp)):
        assert np.abs(got.cpu().numpy() - want).max() <= 1e-12
