"""One env of a slab preset (TS_TETS, default 52359) for ncu: a few steps of the cluster kernel."""
import ctypes, os, sys, tempfile
import numpy as np, torch
sys.path.insert(0, '.')
from paper_2503_18616_b200 import EnvBatch, _native as N
from paper_2503_18616_b200.mesh import load_scene, make_slab_scene
d = tempfile.mkdtemp()
scene = load_scene(make_slab_scene(d, tets=int(os.environ.get("TS_TETS", "52359")), name="s"))
env = EnvBatch(scene, num_envs=1, device="cuda:0")
env.reset()
acts = torch.zeros((1, 3), dtype=torch.float64, device="cuda:0")
for i in range(6):
    env.step(acts, validate=False)
torch.cuda.synchronize()
print(env.sim.scene.info)
