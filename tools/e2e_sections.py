"""Per-section host time of EnvBatch.step_numpy's steady state (4096 envs), by replaying its code
with timers (development tool)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_2503_18616_b200 import EnvBatch, load_scene  # noqa: E402
from paper_2503_18616_b200 import _native as N  # noqa: E402
from paper_2503_18616_b200.mesh import default_scene_path  # noqa: E402

n = 4096
env = EnvBatch(load_scene(default_scene_path()), num_envs=n, device="cuda:0")
env.reset()
rng = np.random.default_rng(0)
for i in range(5):
    env.step_numpy(rng.uniform(-1, 1, (n, 3)))
fx = env._np_fast
lib = env.sim.scene.lib
a = rng.uniform(-1, 1, (n, 3))
K = 300
names = ["stage+check", "state_struct", "launch", "alloc+fault", "sync (GPU)", "copy", "views+info"]
T = np.zeros(len(names))
for _ in range(K):
    t = [time.perf_counter()]
    pin = fx["pin_np"]
    np.copyto(pin, a, casting="unsafe")
    ok = np.isfinite(pin).all()
    t.append(time.perf_counter())
    st = env.sim.state_struct()
    t.append(time.perf_counter())
    stream = torch._C._cuda_getCurrentRawStream(0)
    N.check(lib.ts_graph_launch(fx["exec"], stream), "launch")
    t.append(time.perf_counter())
    block = np.empty(fx["raw"].shape, np.uint8)
    block.fill(0)
    t.append(time.perf_counter())
    N.check(lib.ts_stream_sync(stream), "sync")
    t.append(time.perf_counter())
    np.copyto(block, fx["raw"])
    t.append(time.perf_counter())
    out = {name: np.ndarray(shape, dt, block, off) for name, dt, shape, off, nb in fx["hv"]}
    done = out["done_mask"]
    info = {"contacts": int(out["contacts"].sum()), "any": done.any()}
    t.append(time.perf_counter())
    T += np.diff(t) * 1e6
print("  ".join(f"{k} {v / K:.1f}" for k, v in zip(names, T)), "us; total", f"{T.sum() / K:.1f}")
t0 = time.perf_counter()
for _ in range(K):
    env.step_numpy(a)
print(f"step_numpy {(time.perf_counter() - t0) / K * 1e6:.1f} us")
import cProfile
import pstats
pr = cProfile.Profile()
pr.enable()
for _ in range(K):
    env.step_numpy(a)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
t0 = time.perf_counter()
for _ in range(100):
    fx["fo_host"].copy_(fx["fo_dev"])
print(f"final_obs torch copy_ {(time.perf_counter() - t0) / 100 * 1e6:.1f} us")
t0 = time.perf_counter()
for _ in range(100):
    fx["fo_host"].copy_(fx["fo_dev"], non_blocking=True)
    torch.cuda.current_stream().synchronize()
print(f"final_obs torch copy_ non_blocking + sync {(time.perf_counter() - t0) / 100 * 1e6:.1f} us")
t0 = time.perf_counter()
for _ in range(100):
    np.ndarray((n, 6), np.float64, fx["host"].numpy()[fx["fo"][3]:fx["fo"][3] + fx["fo"][4]].copy())
print(f"final_obs host copy {(time.perf_counter() - t0) / 100 * 1e6:.1f} us")
