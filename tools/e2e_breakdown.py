"""Where the step_numpy time goes beyond the kernels (4096 envs): wall clock of the recorded
graph replay + sync, the same graph's device time (CUDA events around the replay), a graph of the
kernels alone, and the two copies alone.

    gpurun -- python tools/e2e_breakdown.py
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_2503_18616_b200 import EnvBatch, load_scene  # noqa: E402
from paper_2503_18616_b200.mesh import default_scene_path  # noqa: E402

n = 4096
env = EnvBatch(load_scene(default_scene_path()), num_envs=n, device="cuda:0")
env.reset()
rng = np.random.default_rng(0)
for i in range(5):
    env.step_numpy(rng.uniform(-1, 1, (n, 3)))
torch.cuda.synchronize()
fx = env._np_fast
K = 300


def wall(fn):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(K):
        fn()
        fx["done"].record(); fx["done"].synchronize()
    return (time.perf_counter() - t0) / K * 1e3


def dev(fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn(); torch.cuda.synchronize()
    e0.record()
    for _ in range(K):
        fn()
    e1.record(); e1.synchronize()
    return e0.elapsed_time(e1) / K


g = fx["graph"]
print(f"full graph      wall {wall(g.replay):.4f} ms  device (back to back) {dev(g.replay):.4f} ms")
st = env.sim.state_struct()
import ctypes
from paper_2503_18616_b200 import _native as N
lib = env.sim.scene.lib


def kernels():
    N.check(lib.ts_env_step_dl(env.sim.scene.handle, ctypes.byref(st), fx["dl_a"].ptr, ctypes.byref(fx["so"]), None,
                               None, env.sim.stream_ptr()), "step")


gk = torch.cuda.CUDAGraph()
with torch.cuda.graph(gk):
    kernels()
print(f"kernels graph   wall {wall(gk.replay):.4f} ms  device {dev(gk.replay):.4f} ms")
gc = torch.cuda.CUDAGraph()
with torch.cuda.graph(gc):
    fx["dev_a"].copy_(fx["pin_a"], non_blocking=True)
    fx["host"].copy_(fx["dev_buf"], non_blocking=True)
print(f"copies graph    wall {wall(gc.replay):.4f} ms  device {dev(gc.replay):.4f} ms  "
      f"(H2D {fx['pin_a'].numel() * 8} B, D2H {fx['host'].numel()} B)")
ge = torch.cuda.CUDAGraph()
tiny = torch.zeros(1, device="cuda:0")
with torch.cuda.graph(ge):
    tiny.add_(1)
print(f"one-kernel graph wall {wall(ge.replay):.4f} ms")
a = rng.uniform(-1, 1, (n, 3))
t0 = time.perf_counter()
for _ in range(K):
    env.step_numpy(a)
print(f"step_numpy      wall {(time.perf_counter() - t0) / K * 1e3:.4f} ms")
t0 = time.perf_counter()
for _ in range(K):
    rng.uniform(-1, 1, (n, 3))
print(f"rng.uniform     wall {(time.perf_counter() - t0) / K * 1e3:.4f} ms")

# where the Python time of step_numpy goes
import cProfile
import pstats
pr = cProfile.Profile()
pr.enable()
for _ in range(K):
    env.step_numpy(a)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
t0 = time.perf_counter()
for _ in range(K):
    env.sim.state_struct()
print(f"state_struct    wall {(time.perf_counter() - t0) / K * 1e3:.4f} ms")
