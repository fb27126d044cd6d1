"""Large-mesh mode on the GPU: one thread-block cluster of K CTAs per environment.

Every CTA owns a block of the mesh (recursive coordinate bisection), keeps a halo of its
neighbours' vertices that the owners refresh over distributed shared memory (DSMEM) every
substep, and takes part in cluster-wide grasp search, contact resolution and the divergence
flag (the reference's constraint-split "parallel" mode, _kernels.pyx:631-674,
is its CPU analogue).  The per-vertex summation order is unchanged, so the fp64 build stays
bitwise equal to the reference.
"""

import tempfile

import numpy as np
import pytest

import oracle as O
from paper_2503_18616_b200 import EnvBatch
from paper_2503_18616_b200.mesh import load_scene, make_slab_scene

pytestmark = pytest.mark.gpu


def _bitwise_rollout(scene, n, steps, seed, layout):
    ref = O.OracleEnv(O.scene_from_loaded(*scene), n)
    ref.reset()
    gpu = EnvBatch(scene, num_envs=n, device="cuda:0", precision="fp64", layout=layout)
    gpu.reset()
    rng = np.random.default_rng(seed)
    interacted = np.zeros(n, bool)
    contacts = 0
    for s in range(steps):
        a = rng.uniform(-1.0, 1.0, (n, 3))
        a[:, 1] = np.clip(a[:, 1] - 0.3, -1, 1)      # lean into the tissue: grasp and contact happen
        ro, rr, rte, rtr, rinfo = ref.step(a)
        go, gr, gte, gtr, ginfo = gpu.step(a, tool_override=ref.last_cmd)
        interacted |= (ref.grasp_vertex >= 0) | (rinfo["contacts_per_env"] > 0)
        contacts += int(rinfo["contacts"])
        assert np.array_equal(gpu.sim.x.cpu().numpy(), ref.x), s
        assert np.array_equal(gpu.sim.v.cpu().numpy(), ref.v), s
        assert np.array_equal(gr.cpu().numpy(), rr) and np.array_equal(go.cpu().numpy(), ro), s
        assert np.array_equal(gte.cpu().numpy(), rte) and np.array_equal(gtr.cpu().numpy(), rtr), s
        assert np.array_equal(gpu.sim.grasp_vertex.cpu().numpy(), ref.grasp_vertex), s
        assert np.array_equal(gpu.sim.grasped.cpu().numpy(), ref.grasped), s
        assert np.array_equal(ginfo["contacts_per_env"].cpu().numpy(), rinfo["contacts_per_env"]), s
    return gpu, interacted, contacts


@pytest.mark.parametrize("k", [2, 4, 8, 16])
def test_cluster_fp64_bitwise_with_injected_tool_poses(reach_scene, k):
    gpu, interacted, contacts = _bitwise_rollout(reach_scene, 12, 60, seed=5, layout=dict(cluster_size=k))
    assert gpu.sim.scene.info["cluster_size"] == k
    assert interacted.sum() >= 2 and contacts > 0


def test_cluster_fp32_positions_and_rewards(reach_scene):
    """fp32 cluster step (4 CTAs per env) against the reference oracle: rewards within 1e-4 every
    step, per-particle positions within 1e-5 relative on envs without tool interaction (the
    north_star's fp32 tolerances, as test_gpu_parity.py::test_fp32_positions_and_rewards)."""
    n, steps = 16, 60
    ref = O.OracleEnv(O.scene_from_loaded(*reach_scene), n)
    ref.reset()
    gpu = EnvBatch(reach_scene, num_envs=n, device="cuda:0", precision="fp32", layout=dict(cluster_size=4))
    gpu.reset()
    assert gpu.sim.scene.info["cluster_size"] == 4
    rng = np.random.default_rng(2)
    interacted = np.zeros(n, bool)
    for _ in range(steps):
        a = rng.uniform(-1.0, 1.0, (n, 3))
        _, rr, rte, rtr, rinfo = ref.step(a)
        _, gr, _, _, _ = gpu.step(a, tool_override=ref.last_cmd)
        interacted |= (ref.grasp_vertex >= 0) | (rinfo["contacts_per_env"] > 0)
        assert np.abs(gr.cpu().numpy() - rr).max() <= 1e-4
    calm = ~interacted
    assert calm.sum() >= 4
    x = gpu.sim.x.cpu().numpy().astype(np.float64)
    rel = np.linalg.norm(x - ref.x, axis=2) / np.maximum(np.linalg.norm(ref.x, axis=2), 1e-3)
    assert rel[calm].max() <= 1e-5, rel[calm].max()


@pytest.fixture(scope="module")
def slab_52359():
    d = tempfile.mkdtemp()
    return load_scene(make_slab_scene(d, tets=52359))


def test_table2_largest_mesh_fp64_bitwise(slab_52359):
    """The 52359-tet preset (Table II-right): a 16-CTA cluster per env, bitwise vs the reference."""
    gpu, _, _ = _bitwise_rollout(slab_52359, 2, 6, seed=1, layout=None)
    assert gpu.sim.scene.info["cluster_size"] == 16


def test_table2_largest_mesh_fp32(slab_52359):
    n, steps = 4, 20
    ref = O.OracleEnv(O.scene_from_loaded(*slab_52359), n)
    ref.reset()
    gpu = EnvBatch(slab_52359, num_envs=n, device="cuda:0", precision="fp32")
    gpu.reset()
    assert gpu.sim.scene.info["cluster_size"] > 1
    rng = np.random.default_rng(4)
    for _ in range(steps):
        a = rng.uniform(-1.0, 1.0, (n, 3))
        _, rr, _, _, rinfo = ref.step(a)
        _, gr, _, _, _ = gpu.step(a, tool_override=ref.last_cmd)
        assert np.abs(gr.cpu().numpy() - rr).max() <= 1e-4
    calm = ref.grasp_vertex < 0
    x = gpu.sim.x.cpu().numpy().astype(np.float64)
    rel = np.linalg.norm(x - ref.x, axis=2) / np.maximum(np.linalg.norm(ref.x, axis=2), 1e-3)
    assert rel[calm].max() <= 1e-5


def test_cluster_plugin_detect_contacts(reach_scene):
    """The cluster-wide contact merge emits rows in the reference's order (capsule-major, face-minor)."""
    from paper_2503_18616_b200 import backend
    ref = O.OracleEnv(O.scene_from_loaded(*reach_scene), 4)
    ref.reset()
    rng = np.random.default_rng(9)
    checked = 0
    for _ in range(60):
        a = rng.uniform(-1, 1, (4, 3))
        a[:, 1] = np.clip(a[:, 1] - 0.6, -1, 1)
        ref.step(a)
        caps = ref.capsule_rows()
        caps[:, :, 6] += 0.0015
        for i in range(4):
            want = O.detect_contacts(ref.x[i], ref.scene.faces, caps[i])
            got = backend.detect_contacts(ref.x[i], ref.scene.faces, caps[i], layout=dict(cluster_size=4))
            for u, w in zip(want, got):
                assert np.array_equal(u, w)
            checked += len(want[0])
    assert checked > 100
