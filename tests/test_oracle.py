"""Pin the CPU oracle before trusting it.

* bitwise against golden vectors produced by the UNMODIFIED reference
  (tests/golden/make_golden.py): a 100-step 8-env reach rollout with grasp
  and contact, plugin-level run_substeps (attachments + grasp) and
  detect_contacts KATs;
* the reference's own known-answer tests (pkg/tests/test_solver.py,
  test_collision.py) restated against the oracle kernels;
* when the reference is built in this container (oracle/_ref), a fresh
  bitwise rollout comparison.
"""

import os
import sys

import numpy as np
import pytest

import oracle as O
from conftest import ROOT, build_slab_scene, golden


def oracle_env(scene, n):
    env = O.OracleEnv(O.scene_from_loaded(*scene), n)
    env.reset()
    return env


def test_blas_dot_association_assumption():
    """collision.py:64 computes b2 = b @ b through BLAS ddot; the oracle and the kernel assume the
    fused chain fma(b2,b2, fma(b1,b1, b0*b0)).  Pin that on this host."""
    rng = np.random.default_rng(3)
    B = rng.dirichlet(np.ones(3), 2000) * rng.uniform(0.1, 2.0, (2000, 1))
    from fractions import Fraction as Fr

    def fma(a, b, c):
        return float(Fr(a) * Fr(b) + Fr(c))
    assert all(float(b @ b) == fma(b[2], b[2], fma(b[1], b[1], b[0] * b[0])) for b in B)


def test_golden_rollout_bitwise(reach_scene):
    g = golden("trajectory_reach1170_n8_seed5.npz")
    n = g["actions"].shape[1]
    env = oracle_env(reach_scene, n)
    assert np.array_equal(env.observe_rows(np.arange(n)), g["obs0"])
    for s in range(g["actions"].shape[0]):
        obs, r, te, tr, info = env.step(g["actions"][s])
        assert np.array_equal(obs, g["obs"][s]), s
        assert np.array_equal(r, g["reward"][s]), s
        assert np.array_equal(te, g["terminated"][s]) and np.array_equal(tr, g["truncated"][s]), s
        assert np.array_equal(env.grasp_vertex, g["grasp_vertex"][s]), s
        assert info["contacts"] == g["contacts"][s], s
        assert np.array_equal(info["episode_length"], g["episode_length"][s])
        if f"x_{s}" in g:
            assert np.array_equal(env.x, g[f"x_{s}"]) and np.array_equal(env.v, g[f"v_{s}"]), s
    assert g["grasp_vertex"].max() >= 0 and g["contacts"].sum() > 0   # the rollout exercises grasp + contact


def test_golden_plugin_substeps_bitwise():
    g = golden("kernels.npz")
    x, v = g["x0"].copy(), g["v0"].copy()
    for rep in range(3):
        O.run_substeps(x, v, g["w"], g["edges"], g["rest_length"], float(g["ks"]), g["tets"], g["rest_volume"],
                       float(g["kv"]), g["att_vertex"], g["att_faces"], g["att_is_face"], g["att_anchor"],
                       g["att_rest"], g["att_k"], g["grasp_vertex"], g["drag"], g["g"], float(g["h"]),
                       int(g["substeps"]), float(g["damping"]))
        assert np.array_equal(x, g[f"x_{rep}"]) and np.array_equal(v, g[f"v_{rep}"])


def test_golden_contacts_bitwise():
    g = golden("kernels.npz")
    for k in range(int(g["n_contact_cases"])):
        res = O.detect_contacts(g[f"c{k}_pos"], g["contact_faces"], g[f"c{k}_caps"], 8)
        for name, arr in zip(("face", "cap", "depth", "dir", "bary"), res):
            assert np.array_equal(arr, g[f"c{k}_{name}"]), (k, name)


# --- reference KATs (pkg/tests/test_solver.py, test_collision.py) on the oracle kernels ---------------

def _pair_substep(xa, xb, rest, wa=1.0, wb=1.0, substeps=1):
    x = np.array([[xa, xb]], float)
    v = np.zeros_like(x)
    O.run_substeps(x, v, np.array([wa, wb]), np.array([[0, 1]]), np.array([rest]), 1.0, np.zeros((0, 4)),
                   np.zeros(0), 1.0, np.zeros(0), np.zeros((0, 3)), np.zeros(0), np.zeros((0, 3)), np.zeros(0),
                   np.zeros(0), np.array([-1]), np.zeros((1, 3)), np.zeros(3), 0.01, substeps, 0.0)
    return x[0], v[0]


def test_stretched_pair_restores_rest_length():
    x, _ = _pair_substep([0, 0, 0], [2, 0, 0], 1.0)
    assert abs(np.linalg.norm(x[0] - x[1]) - 1.0) < 1e-9
    assert np.allclose(x[0], [0.5, 0, 0]) and np.allclose(x[1], [1.5, 0, 0])


def test_pinned_endpoint_full_correction():
    x, _ = _pair_substep([0, 0, 0], [2, 0, 0], 1.0, wa=0.0)
    assert np.array_equal(x[0], [0, 0, 0]) and np.allclose(x[1], [1, 0, 0], atol=1e-15)


@pytest.mark.parametrize("substeps", [1, 5, 10])
def test_free_fall_closed_form(substeps):
    x = np.array([[[0.0, 0.5, 0.0]]])
    v = np.zeros_like(x)
    dt = 0.01
    O.run_substeps(x, v, np.ones(1), np.zeros((0, 2)), np.zeros(0), 1.0, np.zeros((0, 4)), np.zeros(0), 1.0,
                   np.zeros(0), np.zeros((0, 3)), np.zeros(0), np.zeros((0, 3)), np.zeros(0), np.zeros(0),
                   np.array([-1]), np.zeros((1, 3)), np.array([0.0, -9.81, 0.0]), dt / substeps, substeps, 0.0)
    assert v[0, 0, 1] == pytest.approx(-9.81 * dt, abs=1e-12)
    assert x[0, 0, 1] == pytest.approx(0.5 - 9.81 * dt * dt * (substeps + 1) / (2 * substeps), abs=1e-12)


def test_tet_scaling_kat():
    """s = 1/3 and dx_d = (0,0,-1/18) for the stretched right tet (test_solver.py:121-129)."""
    x = np.array([[[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 2]]], float)
    v = np.zeros_like(x)
    w = np.array([0.0, 0.0, 0.0, 1.0])
    O.run_substeps(x, v, w, np.zeros((0, 2)), np.zeros(0), 1.0, np.array([[0, 1, 2, 3]]), np.array([1 / 6]), 1.0,
                   np.zeros(0), np.zeros((0, 3)), np.zeros(0), np.zeros((0, 3)), np.zeros(0), np.zeros(0),
                   np.array([-1]), np.zeros((1, 3)), np.zeros(3), 0.001, 1, 0.0)
    assert np.allclose(x[0, 3], [0, 0, 2 - 1 / 18], atol=1e-14)


class TestContactKAT:
    AXIS = np.array([[0.0, 0.0, 0.0, 0.0, 0.0, 1.0, 0.1]])

    def test_far_face_empty(self):
        res = O.detect_contacts(np.array([[5, 5, 5], [6, 5, 5], [5, 6, 5]], float), np.array([[0, 1, 2]]), self.AXIS)
        assert len(res[0]) == 0

    def test_penetrating_vertex(self):
        res = O.detect_contacts(np.array([[0.05, 0, 0.5], [0.5, 0, 0.5], [0.5, 0.4, 0.5]]), np.array([[0, 1, 2]]),
                                self.AXIS)
        assert len(res[0]) == 1 and res[2][0] >= 0.05 - 1e-9
        assert np.linalg.norm(res[3][0]) == pytest.approx(1.0) and res[4][0].sum() == pytest.approx(1.0)

    def test_sliver_fallback(self):
        res = O.detect_contacts(np.array([[0.0, 0, 0.5], [1e-9, 0, 0.5], [2e-9, 0, 0.5]]), np.array([[0, 1, 2]]),
                                self.AXIS)
        assert len(res[0]) == 1 and res[2][0] == pytest.approx(0.1, rel=1e-6)

    def test_witness_displacement_equals_depth(self):
        rng = np.random.default_rng(15)
        for _ in range(50):
            pos = rng.normal(size=(3, 3))
            bary = rng.dirichlet(np.ones(3))
            d = rng.normal(size=3)
            d /= np.linalg.norm(d)
            depth = rng.uniform(0.001, 0.05)
            before = bary @ pos
            O.resolve_contacts(pos, np.ones(3), np.array([[0, 1, 2]]), np.array([0]), np.array([0]),
                               np.array([depth]), d[None], bary[None])
            assert np.linalg.norm(bary @ pos - (before + depth * d)) < 1e-9


def test_oracle_batch_rows_independent(small_scene):
    env4 = oracle_env(small_scene, 4)
    env1 = oracle_env(small_scene, 1)
    rng = np.random.default_rng(20)
    for _ in range(25):
        a = rng.uniform(-1, 1, 3)
        env4.step(np.tile(a, (4, 1)))
        env1.step(a[None])
    for i in range(4):
        assert np.array_equal(env4.x[i], env1.x[0]) and np.array_equal(env4.v[i], env1.v[0])


def _ref_available():
    d = os.path.join(ROOT, "oracle", "_ref", "tissuesim", "backends")
    return os.path.isdir(d) and any(f.startswith("_kernels") and f.endswith(".so") for f in os.listdir(d))


@pytest.mark.skipif(not _ref_available(), reason="reference not built here (oracle/build_ref.sh)")
def test_live_reference_rollout_bitwise(reach_scene_path):
    sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))
    from tissuesim.env import EnvBatch as RefEnv
    from paper_2503_18616_b200.mesh import load_scene
    n = 6
    ref = RefEnv(reach_scene_path, num_envs=n, seed=3, backend="compiled", threads=2)
    ref.reset(seed=3)
    env = oracle_env(load_scene(reach_scene_path), n)
    rng = np.random.default_rng(3)
    for s in range(120):
        a = rng.uniform(-1, 1, (n, 3))
        r1 = ref.step(a)
        r2 = env.step(a)
        assert np.array_equal(ref.sim.x, env.x) and np.array_equal(ref.sim.v, env.v), s
        assert np.array_equal(r1[1], r2[1]) and np.array_equal(r1[0], r2[0]), s
        assert r1[4]["contacts"] == r2[4]["contacts"], s
