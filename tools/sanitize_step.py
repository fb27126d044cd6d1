"""A few env steps for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
one-CTA fp32 and fp64 steps, a 2-CTA cluster step, plugin run_substeps / detect_contacts.

    compute-sanitizer --tool racecheck python tools/sanitize_step.py
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2503_18616_b200 import EnvBatch, backend  # noqa: E402
from paper_2503_18616_b200.mesh import default_scene_path, load_scene  # noqa: E402


def main():
    scene = load_scene(default_scene_path())
    n = int(os.environ.get("TS_ENVS", "4"))
    rng = np.random.default_rng(0)
    for prec, layout in (("fp32", None), ("fp64", None), ("fp32", {"cluster_size": 2})):
        env = EnvBatch(scene, num_envs=n, device="cuda:0", precision=prec, layout=layout)
        env.reset()
        for _ in range(int(os.environ.get("TS_STEPS", "3"))):
            a = rng.uniform(-1, 1, (n, 3))
            a[:, 1] -= 0.5          # into the tissue: grasp and contacts run too
            env.step(np.clip(a, -1, 1))
        torch.cuda.synchronize()
        print(prec, layout, "ok", flush=True)
    mesh, rest, cfg = scene
    pos = mesh.positions_rest.copy()
    caps = np.array([[0.04, 0.01, 0.02, 0.04, -0.002, 0.02, 0.003]] * 3)
    out = backend.detect_contacts(pos, mesh.surface_faces, caps)
    print("detect_contacts", len(out[0]), flush=True)


if __name__ == "__main__":
    main()
