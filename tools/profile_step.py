"""Minimal driver for ncu: N envs, a few env steps (step kernel launches are the profiled ones)."""
import ctypes
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2503_18616_b200 import EnvBatch, _native as N  # noqa: E402
from paper_2503_18616_b200.mesh import default_scene_path, load_scene  # noqa: E402


def main():
    n = int(os.environ.get("TS_ENVS", "4096"))
    steps = int(os.environ.get("TS_STEPS", "6"))
    prec = os.environ.get("TS_PREC", "fp32")
    layout = {}
    if os.environ.get("TS_CHUNK"):
        layout["max_chunk_slots"] = int(os.environ["TS_CHUNK"])
    if os.environ.get("TS_BLOCK"):
        layout["block_threads"] = int(os.environ["TS_BLOCK"])
    if os.environ.get("TS_CLUSTER"):
        layout["cluster_size"] = int(os.environ["TS_CLUSTER"])
    scene = load_scene(default_scene_path())
    if os.environ.get("TS_DIST_ONLY"):   # config 2: tets emptied (bench.distance_only)
        import dataclasses
        import numpy as np
        mesh, rest, cfg = scene
        scene = (dataclasses.replace(mesh, tets=np.zeros((0, 4), np.int32)),
                 dataclasses.replace(rest, rest_volume=np.zeros(0)), cfg)
    env = EnvBatch(scene, num_envs=n, device="cuda:0", precision=prec, layout=layout)
    env.reset()
    acts = torch.empty((n, 3), dtype=torch.float64, device="cuda:0")
    lib = N.load()
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    for i in range(steps):
        lib.ts_uniform_actions(acts.data_ptr(), n, 0, 7, i, s)
        env.step(acts, validate=False)
    torch.cuda.synchronize()
    print("layout", env.sim.scene.info)


if __name__ == "__main__":
    main()
