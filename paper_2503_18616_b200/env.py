"""Batched episodic reach task on the GPU -- drop-in for the reference ``EnvBatch`` (env.py:70-197).

Same constructor, ``reset``/``step``/``observe``, attributes and error
behaviour; the return values are CUDA tensors:

* observations (N, 6): float32 (``precision="fp32"``, the policy dtype) or
  float64 (``precision="fp64"``), overridable with ``obs_dtype``;
* rewards (N,) float64; terminated / truncated (N,) bool;
* ``info``: ``distance, success, diverged, clipped, contacts, episode_return,
  episode_length, done_mask, final_observation`` (+ ``contacts_per_env``).
  ``final_observation`` is always an (N, 6) tensor whose rows are zero where
  ``done_mask`` is false (the reference returns None when no row is done);
  ``contacts`` is evaluated lazily so a step never blocks the host.

Every call to ``step`` is three stream-ordered launches -- the per-env command
kernel, the fused sm_100a step kernel and the per-env epilogue
(``csrc/step_kernel.cuh``) -- plus a one-block action check when the actions
are already on the device and ``validate=True``; ``capture_step`` records them
as one CUDA graph and ``step_numpy`` returns host arrays like the reference.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from .errors import ValidationError
from .mesh import SceneConfig, load_scene
from .solver import LazyInt, Simulation, _override_struct

OBSERVATION_SIZE = 6
ACTION_SIZE = 3


@dataclass
class EnvConfig:
    """env.py:24-58."""

    w_distance: float = -1.0
    w_delta: float = -10.0
    w_success: float = 100.0
    success_threshold: float = 0.003
    max_episode_steps: int = 200
    action_scale: float = 0.005
    reward_scale: float = 1.0
    start: np.ndarray = field(default_factory=lambda: np.zeros(3))
    target: np.ndarray = field(default_factory=lambda: np.zeros(3))
    workspace_low: np.ndarray = field(default_factory=lambda: -np.ones(3))
    workspace_high: np.ndarray = field(default_factory=lambda: np.ones(3))
    held_clamp_angle: float = 2.0

    @classmethod
    def from_scene(cls, cfg: SceneConfig):
        out = cls(w_distance=cfg.reward_distance_weight, w_delta=cfg.reward_delta_weight,
                  w_success=cfg.reward_success_weight, success_threshold=cfg.success_threshold,
                  max_episode_steps=cfg.max_episode_steps, action_scale=cfg.action_scale,
                  reward_scale=cfg.reward_scale, start=np.asarray(cfg.tool_start, np.float64),
                  target=np.asarray(cfg.target, np.float64),
                  workspace_low=np.asarray(cfg.workspace_low, np.float64),
                  workspace_high=np.asarray(cfg.workspace_high, np.float64),
                  held_clamp_angle=cfg.clamp_angle)
        for name, p in (("tool_start", out.start), ("target", out.target)):
            if np.any(p < out.workspace_low) or np.any(p > out.workspace_high):
                raise ValidationError(f"{name} lies outside the workspace box")
        return out


def compute_reward(distance, delta, success, cfg: EnvConfig):
    """env.py:61-67 (numpy or torch)."""
    if isinstance(distance, torch.Tensor):
        s = success.to(torch.float64) if isinstance(success, torch.Tensor) else torch.as_tensor(success, dtype=torch.float64)
    else:
        s = np.asarray(success, dtype=np.float64)
    return cfg.reward_scale * (cfg.w_distance * distance + cfg.w_delta * delta + cfg.w_success * s)


class StepInfo(dict):
    """info dict whose ``contacts`` total is computed on first access."""

    def __getitem__(self, key):
        val = dict.__getitem__(self, key)
        return val.value() if isinstance(val, LazyInt) else val


# output buffer layout of one step: (name, dtype, trailing shape)
# final_obs last: step_numpy copies the block without it and fetches it only when a row is done
_OUTS = [("reward", torch.float64, ()), ("distance", torch.float64, ()),
         ("episode_return", torch.float64, ()), ("episode_length", torch.int64, ()),
         ("obs", None, (OBSERVATION_SIZE,)),
         ("contacts", torch.int32, ()), ("terminated", torch.bool, ()), ("truncated", torch.bool, ()),
         ("success", torch.bool, ()), ("diverged", torch.bool, ()), ("clipped", torch.bool, ()),
         ("done_mask", torch.bool, ()), ("final_obs", None, (OBSERVATION_SIZE,))]


class EnvBatch:
    """N independent reach-task instances stepped as one batch on one GPU."""

    observation_size = OBSERVATION_SIZE
    action_size = ACTION_SIZE
    # step_numpy: True = the kernels read actions / write outputs in pinned host memory directly.
    # Measured slower on B200 (0.695 vs 0.658 ms per 4096-env step: the epilogue's scattered writes
    # over the bus cost more than one bulk D2H copy), so the default keeps the two copies.
    numpy_zero_copy = False

    def __init__(self, scene, num_envs: int = 1, seed: int = 0, backend: str = "auto",
                 mode: str = "deterministic", threads: int | None = None, device=None,
                 precision: str = "fp32", obs_dtype=None, layout=None):
        if isinstance(scene, str):
            mesh, rest, cfg = load_scene(scene)
        else:
            mesh, rest, cfg = scene
        if num_envs < 1:
            raise ValidationError("num_envs must be >= 1")
        self.scene_config = cfg
        self.config = EnvConfig.from_scene(cfg)
        self.sim = Simulation(mesh, rest, cfg, num_instances=num_envs, backend=backend, mode=mode,
                              threads=threads, device=device, precision=precision, layout=layout)
        self.num_envs = num_envs
        self.device = self.sim.device
        self.precision = self.sim.precision
        if obs_dtype is None:
            obs_dtype = torch.float64 if self.precision == "fp64" else torch.float32
        if obs_dtype not in (torch.float32, torch.float64):
            raise ValidationError("obs_dtype must be torch.float32 or torch.float64")
        self.obs_dtype = obs_dtype
        self._ready = False
        self.seed_value = seed
        self._rng = None
        self._bad_flag = torch.zeros(1, dtype=torch.int32, device=self.device)
        self._bad_flag_dl = N.dl(self._bad_flag)
        self._pinned_actions = None
        self._dev_actions = None
        self._layout = self._out_layout()
        self._numpy_layout = self._out_layout(torch.float64)
        # D2H bytes of a step_numpy call: the block without final_obs, + final_obs when a row is done
        self.numpy_block_bytes = self._numpy_layout[0][-1][3]
        self.numpy_final_obs_bytes = self._numpy_layout[0][-1][4]
        self.numpy_d2h_bytes = 0   # running total over step_numpy calls

    # -- reference-named state (views of the device state) ------------------
    @property
    def _steps(self):
        return self.sim._steps

    @property
    def _l_prev(self):
        return self.sim._l_prev

    @property
    def _return(self):
        return self.sim._return

    # -- helpers ------------------------------------------------------------
    def _normalize(self, p):
        lo = torch.as_tensor(self.config.workspace_low, dtype=torch.float64, device=self.device)
        hi = torch.as_tensor(self.config.workspace_high, dtype=torch.float64, device=self.device)
        if not isinstance(p, torch.Tensor):
            p = torch.as_tensor(np.asarray(p, np.float64), device=self.device)
        return 2.0 * (p - lo) / (hi - lo) - 1.0

    def _distances(self, idx=None):
        drag = self.sim.tool.drag_points()
        if idx is not None:
            drag = drag[torch.as_tensor(np.atleast_1d(idx), device=self.device)]
        rel = drag - torch.as_tensor(self.config.target, dtype=torch.float64, device=self.device)[None, :]
        return torch.sqrt((rel[:, 0] * rel[:, 0] + rel[:, 2] * rel[:, 2]) + rel[:, 1] * rel[:, 1])

    def _observe_all(self):
        obs = torch.empty((self.num_envs, OBSERVATION_SIZE), dtype=self.obs_dtype, device=self.device)
        st = self.sim.state_struct()
        obs_dl = N.dl(obs)            # the view must outlive the call
        with torch.cuda.device(self.device):
            N.check(self.sim.scene.lib.ts_env_observe_dl(self.sim.scene.handle, ctypes.byref(st),
                                                         obs_dl.ptr, self.sim.stream_ptr()), "ts_env_observe")
        return obs

    def _observe_rows(self, idx):
        return self._observe_all()[torch.as_tensor(np.asarray(idx), device=self.device)]

    def observe(self, instance: int):
        return self._observe_all()[int(instance)]

    # -- episodic API ---------------------------------------------------------
    def reset(self, indices=None, seed=None):
        """env.py:123-142: restore rows to rest, tool at start; returns their observations."""
        n = self.num_envs
        if seed is not None:
            self.seed_value = seed
        if self._rng is None or seed is not None:
            # per-instance RNGs are reserved by the reference (unused): keep the seeding contract
            self._rng = np.random.SeedSequence(self.seed_value).generate_state(n)
        mask = None
        idx = None
        if indices is not None:
            idx = np.atleast_1d(np.asarray(indices))
            m = np.zeros(n, np.uint8)
            m[idx] = 1
            mask = torch.as_tensor(m, device=self.device)
        obs = torch.empty((n, OBSERVATION_SIZE), dtype=self.obs_dtype, device=self.device)
        st = self.sim.state_struct()
        mask_dl, obs_dl = N.dl(mask), N.dl(obs)   # the views must outlive the call
        with torch.cuda.device(self.device):
            N.check(self.sim.scene.lib.ts_env_reset_dl(self.sim.scene.handle, ctypes.byref(st), N.dlp(mask_dl),
                                                       obs_dl.ptr, self.sim.stream_ptr()), "ts_env_reset")
        self._ready = True
        return obs if idx is None else obs[torch.as_tensor(idx, device=self.device)]

    def _out_layout(self, obs_dtype=None):
        n = self.num_envs
        off = 0
        layout = []
        for name, dt, shape in _OUTS:
            dt = (obs_dtype or self.obs_dtype) if dt is None else dt
            numel = n * int(np.prod(shape)) if shape else n
            nbytes = numel * torch.tensor([], dtype=dt).element_size()
            layout.append((name, dt, (n, *shape), off, nbytes))
            off += (nbytes + 15) // 16 * 16
        return layout, off

    def _alloc_outputs(self):
        layout, total = self._layout
        buf = torch.empty(total, dtype=torch.uint8, device=self.device)
        self._last_buf = buf
        return {name: buf[off:off + nb].view(dt).view(shape) for name, dt, shape, off, nb in layout}

    def _stage_actions(self, actions):
        """(device pointer, is_f32, keepalive) for actions; validates like env.py:151-160."""
        n = self.num_envs
        if isinstance(actions, torch.Tensor) and actions.is_cuda:
            if tuple(actions.shape) != (n, ACTION_SIZE):
                raise ValidationError(f"actions must have shape {(n, ACTION_SIZE)}, got {tuple(actions.shape)}")
            a = actions
            if a.device != self.device:
                a = a.to(self.device)
            if a.dtype not in (torch.float32, torch.float64):
                a = a.to(torch.float64)
            a = a.contiguous()
            return a, a.dtype == torch.float32, True
        a = np.asarray(actions.cpu().numpy() if isinstance(actions, torch.Tensor) else actions, dtype=np.float64)
        if a.shape != (n, ACTION_SIZE):
            raise ValidationError(f"actions must have shape {(n, ACTION_SIZE)}, got {a.shape}")
        if not np.all(np.isfinite(a)):
            raise ValidationError("actions must be finite")
        if self._pinned_actions is None:
            self._pinned_actions = torch.empty((n, ACTION_SIZE), dtype=torch.float64, pin_memory=True)
            self._dev_actions = torch.empty((n, ACTION_SIZE), dtype=torch.float64, device=self.device)
            self._copy_done = torch.cuda.Event()
        else:
            self._copy_done.synchronize()   # previous H2D copy must have drained the pinned buffer
        self._pinned_actions.numpy()[...] = a
        with torch.cuda.device(self.device):
            self._dev_actions.copy_(self._pinned_actions, non_blocking=True)
            self._copy_done.record()
        return self._dev_actions, False, False

    def capture_step(self, actions, pre=None, warmup=2):
        """CUDA-graph one whole env step (command, fused step and epilogue kernels) for the
        device-resident ``actions`` tensor, which the caller refills in place between replays
        (or ``pre``, a callable captured in front of the step -- e.g. an on-device action draw).

        Runs ``warmup`` real steps first (graph capture needs the lazily-grown device buffers to
        exist), then captures.  Returns ``replay() -> (obs, reward, terminated, truncated, info)``;
        the outputs live in fixed buffers that every replay overwrites.
        """
        if not self._ready:
            raise RuntimeError("step called before reset")
        if not (isinstance(actions, torch.Tensor) and actions.is_cuda):
            raise ValidationError("capture_step needs device-resident actions")
        dev = self.device
        side = torch.cuda.Stream(dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):
            for _ in range(warmup):
                if pre is not None:
                    pre()
                self.step(actions, validate=False)
        torch.cuda.current_stream(dev).wait_stream(side)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            if pre is not None:
                pre()
            out = self.step(actions, validate=False)
        self.sim.step_count -= 1          # the capture itself executes nothing

        def replay():
            graph.replay()
            self.sim.step_count += 1
            return out
        replay.graph = graph
        return replay

    def step_numpy(self, actions):
        """``step`` with the reference's host semantics (env.py:144-197): numpy actions in; numpy
        float64 obs (whatever the build precision, like the reference's ``_observe_rows``),
        reward / terminated / truncated and an info dict of numpy arrays out
        (``final_observation`` is None when no row is done, ``contacts`` an int).

        The first call runs eagerly and then records the device side of a step as a CUDA graph;
        later calls validate the actions on the host, fill the pinned action buffer, replay the
        graph and wait for it.  The graph holds the H2D copy of the actions from a pinned buffer,
        the three step kernels and ONE D2H copy of the packed output block into pinned memory --
        all of it but final_obs, which is fetched after the wait only when a row is done (with
        max_episode_steps = 100 that is one step in a hundred).  (``numpy_zero_copy = True``
        instead lets the kernels read the actions and write the block in pinned host memory
        directly -- measured slower, off by default.)  The graph is re-recorded if a state tensor
        was replaced.  The returned arrays are views of one fresh host copy of the block (never
        aliased with the next step's output).
        """
        if not self._ready:
            raise RuntimeError("step called before reset")
        n = self.num_envs
        a = np.asarray(actions.cpu().numpy() if isinstance(actions, torch.Tensor) else actions)
        if a.shape != (n, ACTION_SIZE):
            raise ValidationError(f"actions must have shape {(n, ACTION_SIZE)}, got {a.shape}")
        fx = getattr(self, "_np_fast", None)
        if fx is None:
            zc = self.numpy_zero_copy
            layout, total = self._numpy_layout
            host = torch.empty(total, dtype=torch.uint8, pin_memory=True)
            dev_buf = host if zc else torch.empty(total, dtype=torch.uint8, device=self.device)
            views = {name: dev_buf[off:off + nb].view(dt).view(shape) for name, dt, shape, off, nb in layout}
            # float64 observations, as the reference returns: the obs views are float64 (_numpy_layout)
            so = N.dl_struct(N.StepOutTensors, N.STEP_OUTS, views)
            hv = [(name, torch.empty(0, dtype=dt).numpy().dtype, shape, off, nb) for name, dt, shape, off, nb in layout]
            fo_off = self.numpy_block_bytes   # final_obs: the block's tail
            pin_a = torch.empty((n, ACTION_SIZE), dtype=torch.float64, pin_memory=True)
            dev_a = pin_a if zc else torch.empty((n, ACTION_SIZE), dtype=torch.float64, device=self.device)
            fx = self._np_fast = {"dev_buf": dev_buf, "so": so, "host": host, "raw": host.numpy()[:fo_off],
                                  "hv": hv[:-1], "fo": hv[-1], "fo_host": host[fo_off:], "fo_dev": dev_buf[fo_off:],
                                  "pin_a": pin_a, "pin_np": pin_a.numpy(), "dev_a": dev_a, "dl_a": N.dl(dev_a),
                                  "done": torch.cuda.Event(), "graph": None, "sig": None, "zc": zc}
        pin = fx["pin_np"]
        np.copyto(pin, a, casting="unsafe")
        if not np.isfinite(pin).all():
            raise ValidationError("actions must be finite")
        st = self.sim.state_struct()
        dev = self.device
        fo_len = self.numpy_block_bytes

        def device_side():
            if not fx["zc"]:
                fx["dev_a"].copy_(fx["pin_a"], non_blocking=True)
            N.check(self.sim.scene.lib.ts_env_step_dl(self.sim.scene.handle, ctypes.byref(st), fx["dl_a"].ptr,
                                                      ctypes.byref(fx["so"]), None, None, self.sim.stream_ptr()),
                    "ts_env_step")
            if not fx["zc"]:
                fx["host"][:fo_len].copy_(fx["dev_buf"][:fo_len], non_blocking=True)

        if fx["graph"] is not None and fx["sig"] is self.sim._state and torch.cuda.current_device() == dev.index:
            # the steady state: launch the recorded graph on the current stream; while it runs, take
            # (and page in) the fresh host block this step's outputs are copied to; then wait
            lib = self.sim.scene.lib
            stream = torch._C._cuda_getCurrentRawStream(dev.index)
            N.check(lib.ts_graph_launch(fx["exec"], stream), "step_numpy")
            block = np.empty(fx["raw"].shape, np.uint8)
            block.fill(0)
            N.check(lib.ts_stream_sync(stream), "step_numpy")
        else:
            with torch.cuda.device(dev):
                self._step_numpy_record(fx, device_side)
                fx["done"].record()
            fx["done"].synchronize()
            block = np.empty(fx["raw"].shape, np.uint8)
        self.sim.step_count += 1
        np.copyto(block, fx["raw"])       # one host copy of the packed block; the arrays are views of it
        out = {name: np.ndarray(shape, dt, block, off) for name, dt, shape, off, nb in fx["hv"]}
        done = out["done_mask"]
        d2h = fo_len
        final = None
        if done.any():                    # final_obs only now (its rows are zero where not done)
            if not fx["zc"]:
                fx["fo_host"].copy_(fx["fo_dev"])
                d2h += self.numpy_final_obs_bytes
            _, dt, shape, off, nb = fx["fo"]
            final = np.ndarray(shape, dt, fx["host"].numpy()[off:off + nb].copy())
        self.numpy_d2h_bytes += d2h
        info = {
            "distance": out["distance"], "success": out["success"], "diverged": out["diverged"],
            "clipped": out["clipped"], "contacts": int(out["contacts"].sum()),
            "contacts_per_env": out["contacts"], "episode_return": out["episode_return"],
            "episode_length": out["episode_length"], "done_mask": done,
            "final_observation": final,
        }
        return out["obs"], out["reward"], out["terminated"], out["truncated"], info

    def _step_numpy_record(self, fx, device_side):
        """step_numpy off the steady state: replay on another current device, or -- first call /
        a state tensor replaced -- one eager step, then the graph of the device side."""
        if fx["graph"] is not None and fx["sig"] is self.sim._state:
            fx["graph"].replay()
            return
        device_side()
        fx["done"].record()
        fx["done"].synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            device_side()
        ex = graph.raw_cuda_graph_exec()                 # cudaGraphExec_t (an address)
        fx["graph"], fx["sig"], fx["exec"] = graph, self.sim._state, ex if isinstance(ex, int) else int(ex)

    def step(self, actions, validate=True, tool_override=None):
        """env.py:144-197 on the GPU.  Returns (obs, reward, terminated, truncated, info).

        Device-resident actions are checked for finiteness on the GPU; with
        ``validate=True`` the call then waits for that verdict so a bad batch
        raises ``ValidationError`` before returning (no state is modified).
        """
        if not self._ready:
            raise RuntimeError("step called before reset")
        n = self.num_envs
        a, is_f32, on_device = self._stage_actions(actions)
        out = self._alloc_outputs()
        so = N.dl_struct(N.StepOutTensors, N.STEP_OUTS, out)
        ovr = None
        if tool_override is not None:
            ovr, _keep = _override_struct(tool_override, n, self.device)
        check = on_device and validate
        st = self.sim.state_struct()
        a_dl = N.dl(a)
        with torch.cuda.device(self.device):
            N.check(self.sim.scene.lib.ts_env_step_dl(
                self.sim.scene.handle, ctypes.byref(st), a_dl.ptr, ctypes.byref(so),
                ctypes.byref(ovr) if ovr is not None else None,
                self._bad_flag_dl.ptr if check else None, self.sim.stream_ptr()), "ts_env_step")
        if check and int(self._bad_flag.item()) != 0:
            raise ValidationError("actions must be finite")
        self.sim.step_count += 1
        contacts = out["contacts"]
        info = StepInfo(
            distance=out["distance"], success=out["success"], diverged=out["diverged"],
            clipped=out["clipped"], contacts=LazyInt(lambda: int(contacts.sum().item())),
            contacts_per_env=contacts, episode_return=out["episode_return"],
            episode_length=out["episode_length"], done_mask=out["done_mask"],
            final_observation=out["final_obs"])
        return out["obs"], out["reward"], out["terminated"], out["truncated"], info
