"""Mesh-size scaling (the paper's Table II-right): env-steps/s of one
environment (and of a batch) versus the slab presets' tet count, one CTA per env where the mesh
fits and a thread-block cluster of K CTAs per env otherwise, next to the unmodified CPU
reference (compiled backend, 1 thread for 1 env) on this host.

    python tools/bench_mesh.py [--out gpurun_out/mesh.json] [--steps 200] [--batch 256]

Each GPU figure replays the CUDA-graph-captured step (action draw + command + step +
epilogue kernels), timed with CUDA events over `steps` replays (state resident, L2 warm: the
single-env state is tens of KB).
"""
import argparse
import ctypes
import json
import os
import sys
import tempfile
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2503_18616_b200 import EnvBatch, _native as N  # noqa: E402
from paper_2503_18616_b200.mesh import SLAB_PRESETS, load_scene, make_slab_scene  # noqa: E402


def gpu_rate(scene, n, steps, layout=None, precision="fp32"):
    env = EnvBatch(scene, num_envs=n, device="cuda:0", precision=precision, layout=layout)
    env.reset()
    lib = N.load()
    acts = torch.empty((n, 3), dtype=torch.float64, device="cuda:0")
    counter = torch.zeros(1, dtype=torch.int64, device="cuda:0")

    def draw():
        N.check(lib.ts_uniform_actions_dev(N.ptr(acts), n, 0, 7, N.ptr(counter),
                                           ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)), "draw")
    replay = env.capture_step(acts, pre=draw, warmup=3)
    for _ in range(5):
        replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        replay()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    return n / ms * 1e3, ms, env.sim.scene.info


def cpu_rate(scene_path, n, seconds=4.0):
    sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))
    try:
        from tissuesim.env import EnvBatch as RefEnv
    except ImportError:
        return None, 0
    threads = min(16, n)
    env = RefEnv(scene_path, num_envs=n, seed=0, backend="compiled", mode="deterministic", threads=threads)
    env.reset(seed=0)
    rng = np.random.default_rng(0)
    env.step(rng.uniform(-1, 1, (n, 3)))
    k, t0 = 0, time.perf_counter()
    while time.perf_counter() - t0 < seconds:
        env.step(rng.uniform(-1, 1, (n, 3)))
        k += 1
    return n * k / (time.perf_counter() - t0), threads


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "mesh_scaling.json"))
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--cpu-seconds", type=float, default=4.0)
    args = ap.parse_args()
    rows = []
    d = tempfile.mkdtemp()
    for tets in sorted(SLAB_PRESETS):
        path = make_slab_scene(d, tets=tets, name=f"slab_{tets}")
        scene = load_scene(path)
        row = {"tets": tets, "vertices": scene[0].vertex_count}
        variants = [("auto", None)] + [(f"cluster{k}", {"cluster_size": k}) for k in (2, 4, 8, 16)]
        for name, layout in variants:
            try:
                fps, ms, info = gpu_rate(scene, 1, args.steps, layout)
                row[f"gpu_1env_{name}"] = {"env_steps_per_s": fps, "ms_per_step": ms,
                                           "ctas_per_env": info["cluster_size"]}
            except Exception as exc:   # a cluster size may not fit / not help this mesh
                row[f"gpu_1env_{name}"] = {"error": str(exc)[:200]}
        try:
            fps, ms, info = gpu_rate(scene, args.batch, max(20, args.steps // 4))
            row[f"gpu_{args.batch}env"] = {"env_steps_per_s": fps, "ms_per_step": ms,
                                          "ctas_per_env": info["cluster_size"]}
        except Exception as exc:
            row[f"gpu_{args.batch}env"] = {"error": str(exc)[:200]}
        cps, threads = cpu_rate(path, 1, args.cpu_seconds)
        row["cpu_reference_1env"] = {"env_steps_per_s": cps, "threads": threads}
        rows.append(row)
        print(json.dumps(row), flush=True)
    out = {"what": "single-env (and batch) env-steps/s vs mesh size, slab presets (Table II-right)",
           "gpu": torch.cuda.get_device_name(0), "host_cores": os.cpu_count(), "rows": rows}
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
