import sys, time, cProfile, pstats
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2503_18616_b200 import EnvBatch, load_scene
from paper_2503_18616_b200.mesh import default_scene_path
n = 4096
env = EnvBatch(load_scene(default_scene_path()), num_envs=n, device="cuda:0")
env.reset()
rng = np.random.default_rng(0)
acts = [rng.uniform(-1, 1, (n, 3)) for _ in range(60)]
for i in range(5): env.step_numpy(acts[i])
torch.cuda.synchronize()
t0 = time.perf_counter()
for i in range(50): env.step_numpy(acts[i])
print("e2e ms/step", (time.perf_counter() - t0) / 50 * 1e3)
pr = cProfile.Profile(); pr.enable()
for i in range(50): env.step_numpy(acts[i])
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
