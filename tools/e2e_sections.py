"""Per-section host time of EnvBatch.step_numpy's steady state (4096 envs), by replaying its code
with timers (development tool)."""
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
fx = env._np_fast
a = rng.uniform(-1, 1, (n, 3))
K = 300
T = np.zeros(7)
for _ in range(K):
    t = [time.perf_counter()]
    pin = fx["pin_np"]
    np.copyto(pin, a, casting="unsafe")
    ok = np.isfinite(pin).all()
    t.append(time.perf_counter())
    st = env.sim.state_struct()
    t.append(time.perf_counter())
    cond = fx["graph"] is not None and fx["sig"] is env.sim._state and torch.cuda.current_device() == env.device.index
    t.append(time.perf_counter())
    fx["graph"].replay()
    t.append(time.perf_counter())
    fx["done"].record()
    t.append(time.perf_counter())
    fx["done"].synchronize()
    t.append(time.perf_counter())
    block = fx["raw"].copy()
    out = {name: np.ndarray(shape, dt, block, off) for name, dt, shape, off, nb in fx["hv"]}
    done = out["done_mask"]
    info = {"contacts": int(out["contacts"].sum()), "any": done.any()}
    t.append(time.perf_counter())
    T += np.diff(t) * 1e6
names = ["stage+check", "state_struct", "graph cond", "replay", "record", "sync (GPU)", "outputs"]
print("  ".join(f"{k} {v / K:.1f}" for k, v in zip(names, T)), "us; total", f"{T.sum() / K:.1f}")
