"""Gym-convention bindings and the reference's conformance checks
(reference bindings/src/tissuesim_gym/conformance.py:17-71, bindings/tests/test_bindings.py)."""

import numpy as np
import pytest
import torch

from paper_2503_18616_b200.bindings import Box, make
from paper_2503_18616_b200.bindings.conformance import main as conformance_main, run_checks
from paper_2503_18616_b200.mesh import default_scene_path


def test_box_contains_cpu():
    from paper_2503_18616_b200.bindings import _unit_box
    b = _unit_box(3)
    assert isinstance(b, Box) and b.contains(np.zeros(3)) and not b.contains(np.full(3, 1.5))
    assert not b.contains(np.zeros(4)) and b.contains(torch.zeros(3))


@pytest.mark.gpu
@pytest.mark.parametrize("tensors", [False, True])
def test_conformance_passes(tensors):
    ok, results = run_checks(default_scene_path(), num_envs=4, seed=0, verbose=False, tensors=tensors)
    assert ok, [name for name, good in results if not good]
    assert len(results) == 15


@pytest.mark.gpu
def test_conformance_cli():
    assert conformance_main(["--num-envs", "3"]) == 0


@pytest.mark.gpu
def test_bound_env_matches_native_batch():
    """The binding adds no arithmetic: its five-tuple equals EnvBatch.step_numpy's, bit for bit."""
    from paper_2503_18616_b200 import EnvBatch
    env = make(default_scene_path(), num_envs=5, seed=3)
    ref = EnvBatch(default_scene_path(), num_envs=5, seed=3, obs_dtype=torch.float64)
    assert np.array_equal(env.reset(seed=3), ref.reset(seed=3).cpu().numpy())
    rng = np.random.default_rng(0)
    for _ in range(20):
        a = rng.uniform(-1, 1, (5, 3))
        got, want = env.step(a), ref.step_numpy(a)
        for g, w in zip(got[:4], want[:4]):
            assert np.array_equal(g, w)
