"""Where the host time of EnvBatch.step_numpy goes (4096 envs): per-phase wall clock.

    gpurun -- python tools/e2e_profile.py
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_2503_18616_b200 import EnvBatch, load_scene  # noqa: E402
from paper_2503_18616_b200.mesh import default_scene_path  # noqa: E402

n = 4096
if len(sys.argv) > 1 and sys.argv[1] == "zero-copy":
    EnvBatch.numpy_zero_copy = True      # A/B: kernels read / write pinned host memory directly
env = EnvBatch(load_scene(default_scene_path()), num_envs=n, device="cuda:0")
env.reset()
rng = np.random.default_rng(0)
for i in range(5):
    env.step_numpy(rng.uniform(-1, 1, (n, 3)))
torch.cuda.synchronize()
K = 200
t0 = time.perf_counter()
for i in range(K):
    a = rng.uniform(-1, 1, (n, 3))
t_draw = (time.perf_counter() - t0) / K
t0 = time.perf_counter()
for i in range(K):
    env.step_numpy(a)
t_step = (time.perf_counter() - t0) / K
t0 = time.perf_counter()
for i in range(K):
    env.step_numpy(rng.uniform(-1, 1, (n, 3)))
t_both = (time.perf_counter() - t0) / K
fx = env._np_fast
g = fx["graph"]
torch.cuda.synchronize()
t0 = time.perf_counter()
for i in range(K):
    g.replay()
    fx["done"].record()
    fx["done"].synchronize()
t_graph = (time.perf_counter() - t0) / K
raw = fx["raw"]
t0 = time.perf_counter()
for i in range(K):
    raw.copy()
t_copy = (time.perf_counter() - t0) / K
pin = fx["pin_np"]
t0 = time.perf_counter()
for i in range(K):
    np.copyto(pin, a, casting="unsafe")
    np.isfinite(pin).all()
t_stage = (time.perf_counter() - t0) / K
print(f"draw {t_draw*1e3:.4f} ms  step_numpy {t_step*1e3:.4f}  draw+step {t_both*1e3:.4f}  "
      f"graph replay+sync {t_graph*1e3:.4f}  block copy {t_copy*1e3:.4f} ({raw.nbytes} B)  stage {t_stage*1e3:.4f}")
