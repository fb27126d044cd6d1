"""Quick GPU sanity / parity / timing probe (development tool)."""
import os
import subprocess
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle as O  # noqa: E402

from paper_2503_18616_b200 import EnvBatch, load_scene  # noqa: E402
from paper_2503_18616_b200.mesh import default_scene_path  # noqa: E402


def parity(precision, n=16, steps=100, override=True, seed=5):
    scene = load_scene(default_scene_path())
    ref = O.OracleEnv(O.scene_from_loaded(*scene), n)
    ref.reset()
    gpu = EnvBatch(scene, num_envs=n, device="cuda:0", precision=precision)
    gpu.reset()
    rng = np.random.default_rng(seed)
    first_bad = None
    max_r = 0.0
    grasped_ever = np.zeros(n, bool)
    for s in range(steps):
        a = rng.uniform(-1, 1, (n, 3))
        o_ref, r_ref, te_ref, tr_ref, info_ref = ref.step(a)
        grasped_ever |= ref.grasp_vertex >= 0
        o, r, te, tr, info = gpu.step(a, tool_override=ref.last_cmd if override else None)
        r = r.cpu().numpy()
        max_r = max(max_r, np.abs(r - r_ref).max())
        x = gpu.sim.x.cpu().numpy().astype(np.float64)
        v = gpu.sim.v.cpu().numpy().astype(np.float64)
        same = (np.array_equal(x, ref.x) and np.array_equal(v, ref.v)
                and np.array_equal(gpu.sim.grasp_vertex.cpu().numpy(), ref.grasp_vertex)
                and np.array_equal(te.cpu().numpy(), te_ref) and np.array_equal(tr.cpu().numpy(), tr_ref))
        if not same and first_bad is None:
            first_bad = s
            d = np.abs(x - ref.x).max(axis=(1, 2))
            print(f"  first mismatch at step {s}: per-env max|dx| {np.array2string(d, precision=2)}")
            print("  gv gpu", gpu.sim.grasp_vertex.cpu().numpy(), "ref", ref.grasp_vertex)
    x = gpu.sim.x.cpu().numpy().astype(np.float64)
    rel = np.abs(x - ref.x).max(axis=2) / np.maximum(np.linalg.norm(ref.x, axis=2), 1e-3)
    print(f"[{precision}] first_bad={first_bad} max|dr|={max_r:.3e} "
          f"never-grasped envs max rel dx={rel[~grasped_ever].max() if (~grasped_ever).any() else float('nan'):.3e} "
          f"all envs max rel dx={rel.max():.3e}")


def timing(precision, n=4096, steps=20, warmup=5):
    scene = load_scene(default_scene_path())
    env = EnvBatch(scene, num_envs=n, device="cuda:0", precision=precision)
    env.reset()
    acts = torch.empty((n, 3), dtype=torch.float64, device="cuda:0")
    lib = env.sim.scene.lib
    import ctypes
    for i in range(warmup):
        lib.ts_uniform_actions(acts.data_ptr(), n, 0, 1, i, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
        env.step(acts, validate=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(steps):
        lib.ts_uniform_actions(acts.data_ptr(), n, 0, 1, 100 + i, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
        env.step(acts, validate=False)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    print(f"[{precision}] N={n}: {ms:.3f} ms/step -> {n / ms * 1e3:,.0f} env-steps/s  layout={env.sim.scene.info}")


if __name__ == "__main__":
    print(torch.cuda.get_device_name(0), torch.version.cuda)
    print(subprocess.run(["bash", "-c", "lscpu | head -20; nproc"], capture_output=True, text=True).stdout)
    for prec, ovr in (("fp64", True), ("fp64", False), ("fp32", True), ("fp32", False)):
        try:
            print("override" if ovr else "device tool kinematics")
            parity(prec, override=ovr)
        except Exception as exc:  # keep probing
            import traceback; traceback.print_exc()
            print(f"[{prec}] parity failed: {exc!r}")
    for prec in ("fp32", "fp64"):
        for n in (1, 1024, 4096):
            try:
                timing(prec, n=n)
            except Exception as exc:
                print(f"[{prec}] timing failed: {exc!r}")
