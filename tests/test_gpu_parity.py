"""Parity of the sm_100a env step with the CPU oracle / reference (GPU).

Protocol:
  L0  bit-exact indices: grasp vertex, done/terminated/truncated masks,
      episode lengths, per-env contact counts;
  L2  fp64 build + the oracle's tool poses injected: x, v, rewards, obs
      BITWISE equal to the oracle for 100 interaction-rich steps (and to the
      reference's golden rollout);
  L3  fp32 build: per-particle positions within 1e-5 relative on envs
      without tool interaction after 99 steps (before the step-100 reset);
      rewards within 1e-4 on every step (tolerances stated in the asserts);
  full size (4096 envs): size-independent properties -- row independence
      (a row of the batch equals a batch of one, bitwise), run-to-run
      determinism, pinned vertices never move.
"""

import numpy as np
import pytest
import torch

import oracle as O
from conftest import golden
from paper_2503_18616_b200 import EnvBatch

pytestmark = pytest.mark.gpu

REWARD_TOL = 1e-4          # north_star: per-step rewards within 1e-4
POS_REL_TOL = 1e-5         # north_star: per-particle positions within 1e-5 relative (fp32) after 100 steps


def run_pair(scene, precision, n, steps, seed, inject=True, record=None, layout=None):
    ref = O.OracleEnv(O.scene_from_loaded(*scene), n)
    ref.reset()
    gpu = EnvBatch(scene, num_envs=n, device="cuda:0", precision=precision, layout=layout)
    g_obs0 = gpu.reset().cpu().numpy()
    assert np.allclose(g_obs0, ref.observe_rows(np.arange(n)), atol=1e-7 if precision == "fp32" else 0)
    rng = np.random.default_rng(seed)
    interacted = np.zeros(n, bool)
    out = []
    for s in range(steps):
        a = rng.uniform(-1.0, 1.0, (n, 3))
        ro, rr, rte, rtr, rinfo = ref.step(a)
        go, gr, gte, gtr, ginfo = gpu.step(a, tool_override=ref.last_cmd if inject else None)
        interacted |= (ref.grasp_vertex >= 0) | (rinfo["contacts_per_env"] > 0)
        out.append(dict(step=s, ref=(ro, rr, rte, rtr, rinfo), gpu=(go.cpu().numpy(), gr.cpu().numpy(),
                        gte.cpu().numpy(), gtr.cpu().numpy(), ginfo), interacted=interacted.copy()))
        if record is not None:
            record(s, ref, gpu, out[-1])
    return ref, gpu, out


@pytest.mark.parametrize("edge_gather", [False, True], ids=["edge-slots", "edge-gather"])
def test_fp64_bitwise_with_injected_tool_poses(reach_scene, edge_gather):
    """Both distance-constraint data flows (constraint-parallel slots, owner gather -- the fp32
    default) reproduce the reference bit for bit in the fp64 build."""
    n, steps = 16, 100

    def check(s, ref, gpu, rec):
        go, gr, gte, gtr, ginfo = rec["gpu"]
        ro, rr, rte, rtr, rinfo = rec["ref"]
        assert np.array_equal(gpu.sim.x.cpu().numpy(), ref.x), s
        assert np.array_equal(gpu.sim.v.cpu().numpy(), ref.v), s
        assert np.array_equal(gr, rr) and np.array_equal(go, ro), s
        assert np.array_equal(gte, rte) and np.array_equal(gtr, rtr), s
        assert np.array_equal(gpu.sim.grasp_vertex.cpu().numpy(), ref.grasp_vertex), s
        assert np.array_equal(gpu.sim.grasped.cpu().numpy(), ref.grasped), s
        assert np.array_equal(ginfo["contacts_per_env"].cpu().numpy(), rinfo["contacts_per_env"]), s
        assert np.array_equal(ginfo["episode_length"].cpu().numpy(), rinfo["episode_length"]), s
        assert np.array_equal(ginfo["episode_return"].cpu().numpy(), rinfo["episode_return"]), s
        assert np.array_equal(ginfo["distance"].cpu().numpy(), rinfo["distance"]), s
        if rinfo["final_observation"] is not None:
            assert np.array_equal(ginfo["final_observation"].cpu().numpy(), rinfo["final_observation"]), s
    ref, gpu, out = run_pair(reach_scene, "fp64", n, steps, seed=5, record=check,
                             layout=dict(edge_gather=edge_gather))
    assert gpu.sim.scene.info["edge_gather"] == int(edge_gather)
    assert out[-1]["interacted"].sum() >= 2          # grasp and contact really happened
    assert sum(int(r["ref"][4]["contacts"]) for r in out) > 0


def test_fp64_matches_reference_golden_rollout(reach_scene):
    """The reference's own 100-step rollout (tests/golden) reproduced with its recorded tool poses."""
    g = golden("trajectory_reach1170_n8_seed5.npz")
    n = g["actions"].shape[1]
    gpu = EnvBatch(reach_scene, num_envs=n, device="cuda:0", precision="fp64")
    assert np.array_equal(gpu.reset().cpu().numpy(), g["obs0"])
    for s in range(g["actions"].shape[0]):
        p = g["poses"][s]
        ovr = dict(axis=p[:, 0:3], jaw=p[:, 3:6], reach=p[:, 6], clamp=p[:, 7], clipped=p[:, 8].astype(np.uint8))
        obs, r, te, tr, info = gpu.step(g["actions"][s], tool_override=ovr)
        assert np.array_equal(obs.cpu().numpy(), g["obs"][s]), s
        assert np.array_equal(r.cpu().numpy(), g["reward"][s]), s
        assert np.array_equal(te.cpu().numpy(), g["terminated"][s]), s
        assert np.array_equal(tr.cpu().numpy(), g["truncated"][s]), s
        assert np.array_equal(gpu.sim.grasp_vertex.cpu().numpy(), g["grasp_vertex"][s]), s
        assert info["contacts"] == int(g["contacts"][s]), s
        if f"x_{s}" in g:
            assert np.array_equal(gpu.sim.x.cpu().numpy(), g[f"x_{s}"]), s
            assert np.array_equal(gpu.sim.v.cpu().numpy(), g[f"v_{s}"]), s


def test_fp64_device_kinematics_rewards_and_indices(reach_scene):
    """No injection: CUDA's acos/cos/sin differ from numpy's by ulps; rewards stay within 1e-4 and every
    index (done masks, episode lengths) stays bit-exact on interaction-free envs."""
    n = 32
    ref, gpu, out = run_pair(reach_scene, "fp64", n, 100, seed=7, inject=False)
    for rec in out:
        ro, rr, rte, rtr, _ = rec["ref"]
        go, gr, gte, gtr, _ = rec["gpu"]
        assert np.abs(gr - rr).max() <= REWARD_TOL
        assert np.abs(go - ro).max() <= 1e-9
        calm = ~rec["interacted"]
        assert np.array_equal(gte[calm], rte[calm]) and np.array_equal(gtr[calm], rtr[calm])


def test_fp32_positions_and_rewards(reach_scene):
    n, steps = 32, 99          # compare after 99 steps: step 100 resets every env (max_episode_steps)
    ref, gpu, out = run_pair(reach_scene, "fp32", n, steps, seed=11)
    for rec in out:
        assert np.abs(rec["gpu"][1] - rec["ref"][1]).max() <= REWARD_TOL
        c = ~rec["interacted"]
        assert np.array_equal(rec["gpu"][2][c], rec["ref"][2][c]) and np.array_equal(rec["gpu"][3][c], rec["ref"][3][c])
    calm = ~out[-1]["interacted"]
    assert calm.sum() >= 4
    x = gpu.sim.x.cpu().numpy().astype(np.float64)
    rel = np.linalg.norm(x - ref.x, axis=2) / np.maximum(np.linalg.norm(ref.x, axis=2), 1e-3)
    assert rel[calm].max() <= POS_REL_TOL, rel[calm].max()


def test_fp32_teacher_forced_single_step(reach_scene):
    """From identical (fp64-representable-in-fp32) states, one fp32 step stays within 1e-5 relative."""
    n = 64
    ref = O.OracleEnv(O.scene_from_loaded(*reach_scene), n)
    ref.reset()
    rng = np.random.default_rng(4)
    for _ in range(30):
        ref.step(rng.uniform(-1, 1, (n, 3)))
    gpu = EnvBatch(reach_scene, num_envs=n, device="cuda:0", precision="fp32")
    gpu.reset()
    xf = ref.x.astype(np.float32)
    vf = ref.v.astype(np.float32)
    ref.x[...] = xf
    ref.v[...] = vf
    gpu.sim.x.copy_(torch.as_tensor(xf))
    gpu.sim.v.copy_(torch.as_tensor(vf))
    for name, src in (("axis", ref.axis), ("jaw_dir", ref.jaw), ("reach", ref.reach), ("clamp_angle", ref.clamp)):
        getattr(gpu.sim.tool, name).copy_(torch.as_tensor(src))
    gpu.sim.grasp_vertex.copy_(torch.as_tensor(ref.grasp_vertex))
    gpu.sim.grasped.copy_(torch.as_tensor(ref.grasped))
    gpu.sim._steps.copy_(torch.as_tensor(ref.steps))
    gpu.sim._l_prev.copy_(torch.as_tensor(ref.l_prev))
    a = rng.uniform(-1, 1, (n, 3))
    ref.step(a)
    gpu.step(a, tool_override=ref.last_cmd)
    assert np.array_equal(gpu.sim.grasp_vertex.cpu().numpy(), ref.grasp_vertex)
    x = gpu.sim.x.cpu().numpy().astype(np.float64)
    rel = np.linalg.norm(x - ref.x, axis=2) / np.maximum(np.linalg.norm(ref.x, axis=2), 1e-3)
    assert rel.max() <= POS_REL_TOL, rel.max()


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_full_size_row_independence_and_determinism(reach_scene, precision):
    """4096 envs: row i of the batch equals a batch of one fed the same actions (bitwise), runs repeat
    bitwise, pinned vertices never move."""
    n, steps = 4096, 30
    rng = np.random.default_rng(2)
    acts = rng.uniform(-1, 1, (steps, n, 3))

    def run(num, cols):
        env = EnvBatch(reach_scene, num_envs=num, device="cuda:0", precision=precision)
        env.reset()
        rew = []
        for s in range(steps):
            _, r, _, _, _ = env.step(acts[s][cols])
            rew.append(r.cpu().numpy())
        return env.sim.x.cpu().numpy(), env.sim.v.cpu().numpy(), np.stack(rew)

    xa, va, ra = run(n, slice(None))
    xb, vb, rb = run(n, slice(None))
    assert np.array_equal(xa, xb) and np.array_equal(va, vb) and np.array_equal(ra, rb)
    for i in (0, 1234, n - 1):
        x1, v1, r1 = run(1, slice(i, i + 1))
        assert np.array_equal(x1[0], xa[i]) and np.array_equal(v1[0], va[i]) and np.array_equal(r1[:, 0], ra[:, i])
    mesh = reach_scene[0]
    pinned_rest = mesh.positions_rest[mesh.pinned].astype(xa.dtype)
    assert np.array_equal(xa[:, mesh.pinned], np.broadcast_to(pinned_rest, xa[:, mesh.pinned].shape))
    assert not np.any(va[:, mesh.pinned])


def test_plugin_run_substeps_bitwise_vs_reference_golden():
    from paper_2503_18616_b200 import backend
    g = golden("kernels.npz")
    x, v = g["x0"].copy(), g["v0"].copy()
    for rep in range(3):
        backend.run_substeps(x, v, g["w"], g["edges"], g["rest_length"], float(g["ks"]), g["tets"],
                             g["rest_volume"], float(g["kv"]), g["att_vertex"], g["att_faces"], g["att_is_face"],
                             g["att_anchor"], g["att_rest"], g["att_k"], g["grasp_vertex"], g["drag"], g["g"],
                             float(g["h"]), int(g["substeps"]), float(g["damping"]))
        assert np.array_equal(x, g[f"x_{rep}"]) and np.array_equal(v, g[f"v_{rep}"]), rep


def test_plugin_detect_contacts_bitwise_vs_reference_golden():
    from paper_2503_18616_b200 import backend
    g = golden("kernels.npz")
    for k in range(int(g["n_contact_cases"])):
        res = backend.detect_contacts(g[f"c{k}_pos"], g["contact_faces"], g[f"c{k}_caps"], 8)
        for name, arr in zip(("face", "cap", "depth", "dir", "bary"), res):
            assert np.array_equal(arr, g[f"c{k}_{name}"]), (k, name)


def test_contacts_detected_on_random_tissue_states(reach_scene):
    """Contact rows of the kernel equal the oracle's, bitwise, on many deformed states (capsules are
    inflated by 1.5 mm because the step already pushed the tissue out of the real ones)."""
    from paper_2503_18616_b200 import backend
    ref = O.OracleEnv(O.scene_from_loaded(*reach_scene), 8)
    ref.reset()
    rng = np.random.default_rng(9)
    checked = 0
    for _ in range(150):
        a = rng.uniform(-1, 1, (8, 3))
        a[:, 1] = np.clip(a[:, 1] - 0.6, -1, 1)     # drive the tool into the tissue
        ref.step(a)
        caps = ref.capsule_rows()
        caps[:, :, 6] += 0.0015
        for i in range(8):
            a = O.detect_contacts(ref.x[i], ref.scene.faces, caps[i])
            b = backend.detect_contacts(ref.x[i], ref.scene.faces, caps[i])
            for u, w in zip(a, b):
                assert np.array_equal(u, w)
            checked += len(a[0])
    assert checked > 1000


def test_config1_single_env_1000_steps_bitwise(reach_scene):
    """BASELINE config 1: one env, a 1000-step random-action rollout (ten 100-step episodes with
    auto-resets) -- fp64 build with the oracle's tool poses: bitwise at every step."""
    ref, gpu, out = run_pair(reach_scene, "fp64", 1, 1000, seed=21)
    assert np.array_equal(gpu.sim.x.cpu().numpy(), ref.x) and np.array_equal(gpu.sim.v.cpu().numpy(), ref.v)
    for rec in out:
        ro, rr, rte, rtr, _ = rec["ref"]
        go, gr, gte, gtr, _ = rec["gpu"]
        assert np.array_equal(gr, rr) and np.array_equal(go, ro), rec["step"]
        assert np.array_equal(gte, rte) and np.array_equal(gtr, rtr), rec["step"]
    assert sum(int(rec["gpu"][2][0] or rec["gpu"][3][0]) for rec in out) >= 10   # >= 10 episodes ended


def test_config2_distance_only_bitwise(reach_scene):
    """BASELINE config 2: distance constraints only (tets emptied for the solver, as the reference's
    tests do) -- the kernel's no-slot path (one barrier per substep), fp64 bitwise vs the oracle."""
    import dataclasses
    mesh, rest, cfg = reach_scene
    scene = (dataclasses.replace(mesh, tets=np.zeros((0, 4), np.int32)),
             dataclasses.replace(rest, rest_volume=np.zeros(0)), cfg)
    ref, gpu, out = run_pair(scene, "fp64", 16, 60, seed=4)
    assert gpu.sim.scene.info["n_chunks"] == 0
    assert np.array_equal(gpu.sim.x.cpu().numpy(), ref.x) and np.array_equal(gpu.sim.v.cpu().numpy(), ref.v)
    for rec in out:
        assert np.array_equal(rec["gpu"][1], rec["ref"][1]), rec["step"]


def test_p4_rcm_invariance_device_tool_state(reach_scene):
    """Acceptance P4 (pkg/tests/test_acceptance.py, test_tool.py:rcm_invariance_random_walk) on the
    device command kernel: over a 150-step random walk (auto-resets included) the tool axis stays a
    unit vector through the RCM, the jaw stays orthonormal to it, the clamp angle stays in range, the
    drag point stays in the workspace box -- and the pose equals the numpy oracle's within 1e-9
    (the reference pins its own tool kinematics to 1e-9..1e-12, test_tool.py:35-44)."""
    import torch
    n = 64
    mesh, rest, cfg = reach_scene
    ref = O.OracleEnv(O.scene_from_loaded(*reach_scene), n)
    ref.reset()
    gpu = EnvBatch(reach_scene, num_envs=n, device="cuda:0", precision="fp64")
    gpu.reset()
    rng = np.random.default_rng(4)
    rcm = np.asarray(cfg.rcm)
    lo, hi = np.asarray(cfg.workspace_low), np.asarray(cfg.workspace_high)
    for _ in range(150):
        a = rng.uniform(-1.0, 1.0, (n, 3))
        ref.step(a)
        gpu.step(a)
        t = gpu.sim.tool
        ax, jw = t.axis.cpu().numpy(), t.jaw_dir.cpu().numpy()
        reach, clamp = t.reach.cpu().numpy(), t.clamp_angle.cpu().numpy()
        assert np.abs(np.linalg.norm(ax, axis=1) - 1.0).max() <= 1e-12
        assert np.abs(np.linalg.norm(jw, axis=1) - 1.0).max() <= 1e-12
        assert np.abs(np.einsum("ij,ij->i", ax, jw)).max() <= 1e-12
        assert np.all(clamp > 0.0) and np.all(clamp < 30.0)
        drag = rcm + reach[:, None] * ax
        assert np.all(drag >= lo - 1e-12) and np.all(drag <= hi + 1e-12)
        assert np.abs(ax - ref.axis).max() <= 1e-9 and np.abs(jw - ref.jaw).max() <= 1e-9
        assert np.abs(reach - ref.reach).max() <= 1e-9 and np.abs(clamp - ref.clamp).max() <= 1e-9
    torch.cuda.synchronize()
