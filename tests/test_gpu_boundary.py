"""The typed (DLPack) C-ABI rejects mismatched tensors before anything launches.

The reference's compiled entry takes typed memoryviews, so a wrong buffer fails at the call
(`/root/reference/pkg/src/tissuesim/backends/_kernels.pyx:577-585`); the *_dl entries of
include/tissuesim_b200.h check device, dtype, shape and strides of every DLTensor the same way and
return TS_ERR_INVALID (ValidationError here) naming the tensor -- and leave the state untouched.
"""

import ctypes

import numpy as np
import pytest
import torch

from conftest import build_slab_scene
from paper_2503_18616_b200 import EnvBatch
from paper_2503_18616_b200 import _native as N
from paper_2503_18616_b200 import backend as B
from paper_2503_18616_b200.errors import ValidationError

pytestmark = pytest.mark.gpu


def _env(precision="fp32", n=3):
    env = EnvBatch(build_slab_scene(), num_envs=n, device="cuda:0", precision=precision)
    env.reset()
    return env


def _call_step(env, state=None, actions=None, outs=None):
    """ts_env_step_dl with the env's own tensors, any of which the caller replaces."""
    n = env.num_envs
    sim = env.sim
    st = {k: t for k, t in zip(N.ENV_TENSORS, (sim.x, sim.v, sim.tool.axis, sim.tool.jaw_dir, sim.tool.reach,
                                               sim.tool.clamp_angle, sim.grasp_vertex, sim.grasped, sim._steps,
                                               sim._l_prev, sim._return))}
    st.update(state or {})
    o = {"obs": torch.empty((n, 6), dtype=torch.float32, device=env.device),
         "reward": torch.empty(n, dtype=torch.float64, device=env.device)}
    o.update(outs or {})
    a = actions if actions is not None else torch.zeros((n, 3), dtype=torch.float64, device=env.device)
    sts = N.dl_struct(N.EnvTensors, N.ENV_TENSORS, st)
    so = N.dl_struct(N.StepOutTensors, N.STEP_OUTS, o)
    ad = N.dl(a)
    N.check(sim.scene.lib.ts_env_step_dl(sim.scene.handle, ctypes.byref(sts), ad.ptr, ctypes.byref(so), None, None,
                                         sim.stream_ptr()), "ts_env_step")
    torch.cuda.synchronize()
    return o


def test_well_typed_call_runs():
    env = _env()
    x0 = env.sim.x.clone()
    o = _call_step(env, actions=torch.full((3, 3), 0.5, dtype=torch.float64, device="cuda:0"))
    assert torch.isfinite(o["reward"]).all()
    assert not torch.equal(env.sim.x, x0)          # the step ran
    o = _call_step(env, actions=torch.zeros((3, 3), dtype=torch.float32, device="cuda:0"))   # f32 actions too


@pytest.mark.parametrize("case", ["x_f64_on_fp32", "x_f32_on_fp64", "x_cpu", "x_shape", "x_noncontig",
                                  "grasped_i32", "steps_f64", "axis_shape", "obs_i32", "obs_final_mismatch",
                                  "actions_i64", "actions_noncontig", "actions_cpu", "reward_f32"])
def test_mismatch_rejected_and_state_untouched(case):
    precision = "fp64" if case == "x_f32_on_fp64" else "fp32"
    env = _env(precision)
    sim, n, dev = env.sim, env.num_envs, env.device
    V = sim.x.shape[1]
    state, outs, actions = {}, {}, None
    if case == "x_f64_on_fp32":
        state["x"] = sim.x.double()
    elif case == "x_f32_on_fp64":
        state["x"] = sim.x.float()
    elif case == "x_cpu":
        state["x"] = sim.x.cpu()
    elif case == "x_shape":
        state["x"] = sim.x[:, :-1].contiguous()
    elif case == "x_noncontig":
        state["x"] = torch.empty((n, 3, V), dtype=sim.x.dtype, device=dev).transpose(1, 2)
    elif case == "grasped_i32":
        state["grasped"] = sim.grasped.int()
    elif case == "steps_f64":
        state["steps"] = sim._steps.double()
    elif case == "axis_shape":
        state["tool_axis"] = sim.tool.axis[:, :2].contiguous()
    elif case == "obs_i32":
        outs["obs"] = torch.empty((n, 6), dtype=torch.int32, device=dev)
    elif case == "obs_final_mismatch":
        outs["final_obs"] = torch.empty((n, 6), dtype=torch.float64, device=dev)
    elif case == "actions_i64":
        actions = torch.zeros((n, 3), dtype=torch.int64, device=dev)
    elif case == "actions_noncontig":
        actions = torch.zeros((3, n), dtype=torch.float64, device=dev).t()
    elif case == "actions_cpu":
        actions = torch.zeros((n, 3), dtype=torch.float64)
    elif case == "reward_f32":
        outs["reward"] = torch.empty(n, dtype=torch.float32, device=dev)
    x0, steps0 = sim.x.clone(), sim._steps.clone()
    with pytest.raises(ValidationError) as ei:
        _call_step(env, state, actions, outs)
    name = {"x_f64_on_fp32": "x", "x_f32_on_fp64": "x", "x_cpu": "x", "x_shape": "x", "x_noncontig": "x",
            "grasped_i32": "grasped", "steps_f64": "steps", "axis_shape": "tool_axis", "obs_i32": "obs",
            "obs_final_mismatch": "final_obs", "actions_i64": "actions", "actions_noncontig": "actions",
            "actions_cpu": "actions", "reward_f32": "reward"}[case]
    assert str(ei.value).startswith(f"ts_env_step: {name}:"), str(ei.value)
    torch.cuda.synchronize()
    assert torch.equal(sim.x, x0) and torch.equal(sim._steps, steps0)


def test_reset_and_observe_typed():
    env = _env("fp64")
    obs = env.reset()
    assert obs.dtype == torch.float64
    sim = env.sim
    st = sim.state_struct()
    bad_mask = N.dl(torch.ones(env.num_envs + 1, dtype=torch.uint8, device=env.device))
    with pytest.raises(ValidationError, match="mask"):
        N.check(sim.scene.lib.ts_env_reset_dl(sim.scene.handle, ctypes.byref(st), bad_mask.ptr, None,
                                              sim.stream_ptr()), "ts_env_reset")
    bad_obs = N.dl(torch.empty((env.num_envs, 5), dtype=torch.float64, device=env.device))
    with pytest.raises(ValidationError, match="obs"):
        N.check(sim.scene.lib.ts_env_observe_dl(sim.scene.handle, ctypes.byref(st), bad_obs.ptr,
                                                sim.stream_ptr()), "ts_env_observe")


def test_replaced_state_tensor_is_checked():
    """Replacing a state tensor with a wrongly typed one fails at the next call, not silently."""
    env = _env()
    env.sim.x = env.sim.x.double()
    with pytest.raises(ValidationError, match="x: dtype"):
        env.step(np.zeros((env.num_envs, 3)))


def test_plugin_entries_typed():
    """run_substeps / detect_contacts plugin entries: shapes are checked (wrong caps row count)."""
    mesh, rest, cfg = build_slab_scene()
    x = np.repeat(mesh.positions_rest[None], 2, 0).astype(np.float64)
    v = np.zeros_like(x)
    sc = B._scene_for(rest.inverse_mass.astype(np.float64), mesh.edges, rest.rest_length, 0.5, mesh.tets,
                      rest.rest_volume, 0.5, np.zeros(0, np.int32), np.zeros((0, 3), np.int32), np.zeros(0, np.uint8),
                      np.zeros((0, 3)), np.zeros(0), np.zeros(0), "fp64")
    dev = torch.device("cuda", 0)
    xt, vt = torch.as_tensor(x, device=dev), torch.as_tensor(v, device=dev)
    gv = torch.full((3,), -1, dtype=torch.int64, device=dev)           # N mismatch (3 vs 2)
    drag = torch.zeros((2, 3), dtype=torch.float64, device=dev)
    grav = (ctypes.c_double * 3)(0.0, -9.81, 0.0)
    views = [N.dl(t) for t in (xt, vt, gv, drag)]
    with pytest.raises(ValidationError, match="grasp_vertex: shape"):
        N.check(sc.lib.ts_run_substeps_dl(sc.handle, *(d.ptr for d in views), grav, 1e-3, 2, 0.0, None),
                "ts_run_substeps")
    views[2] = N.dl(gv[:2])
    N.check(sc.lib.ts_run_substeps_dl(sc.handle, *(d.ptr for d in views), grav, 1e-3, 2, 0.0, None),
            "ts_run_substeps")
    torch.cuda.synchronize()
    assert not torch.equal(xt, torch.as_tensor(x, device=dev))


def test_pinned_host_actions_and_outputs_zero_copy():
    """ts_env_step_dl reads actions from / writes outputs to page-locked host memory in place (the
    zero-copy path of step_numpy): same results as device buffers; pageable host memory is rejected."""
    envs = [_env("fp32", n=4) for _ in range(2)]
    rng = np.random.default_rng(5)
    for _ in range(5):
        a = rng.uniform(-1, 1, (4, 3))
        outs = []
        for k, env in enumerate(envs):
            pin = k == 1
            act = torch.as_tensor(a).pin_memory() if pin else torch.as_tensor(a, device="cuda:0")
            mk = (lambda shape, dt: torch.empty(shape, dtype=dt).pin_memory()) if pin else \
                 (lambda shape, dt: torch.empty(shape, dtype=dt, device="cuda:0"))
            o = {"obs": mk((4, 6), torch.float64), "reward": mk(4, torch.float64), "done_mask": mk(4, torch.bool)}
            outs.append(_call_step(env, actions=act, outs=o))
        for key in ("obs", "reward", "done_mask"):
            assert torch.equal(outs[0][key].cpu(), outs[1][key].cpu()), key
        assert torch.equal(envs[0].sim.x, envs[1].sim.x)
    with pytest.raises(ValidationError, match="reward: expected a CUDA tensor or pinned host memory"):
        _call_step(envs[0], outs={"reward": torch.empty(4, dtype=torch.float64)})
