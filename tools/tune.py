"""Layout sweep: ms/step of the fused env-step kernel for several compiler layouts (development tool)."""
import ctypes
import itertools
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2503_18616_b200 import EnvBatch, _native as N  # noqa: E402
from paper_2503_18616_b200.mesh import default_scene_path, load_scene  # noqa: E402


def time_layout(scene, n, precision, layout, steps=20, warmup=4, grid=0):
    env = EnvBatch(scene, num_envs=n, device="cuda:0", precision=precision, layout=layout)
    if grid:
        env.sim.scene.set_max_grid(grid)
    env.reset()
    acts = torch.empty((n, 3), dtype=torch.float64, device="cuda:0")
    lib = N.load()
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    for i in range(warmup):
        lib.ts_uniform_actions(acts.data_ptr(), n, 0, 3, i, s)
        env.step(acts, validate=False)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * steps)]
    tot = 0.0
    for i in range(steps):
        lib.ts_uniform_actions(acts.data_ptr(), n, 0, 3, 100 + i, s)
        ev[2 * i].record()
        env.step(acts, validate=False)
        ev[2 * i + 1].record()
    torch.cuda.synchronize()
    tot = sum(ev[2 * i].elapsed_time(ev[2 * i + 1]) for i in range(steps)) / steps
    return tot, env.sim.scene.info


def main():
    scene = load_scene(default_scene_path())
    n = int(os.environ.get("TS_ENVS", "4096"))
    precs = os.environ.get("TS_PRECS", "fp32,fp64").split(",")
    chunks = [int(c) for c in os.environ.get("TS_CHUNKS", "0,4160,3000,2200,1600,1100").split(",")]
    blocks = [int(b) for b in os.environ.get("TS_BLOCKS", "0").split(",")]
    gathers = [int(g) for g in os.environ.get("TS_GATHER", "1").split(",")]
    cts = os.environ.get("TS_CTS", "").split(",") if os.environ.get("TS_CTS") else [None]
    holes = os.environ.get("TS_HOLES", "").split(",") if os.environ.get("TS_HOLES") else [None]
    ablates = os.environ.get("TS_ABLATES", "").split(",") if os.environ.get("TS_ABLATES") else [None]
    iters = os.environ.get("TS_ITERS", "").split(",") if os.environ.get("TS_ITERS") else [None]
    for prec, ch, bl, ga, ct, ho, ab, itn in itertools.product(precs, chunks, blocks, gathers, cts, holes, ablates,
                                                               iters):
        if ab is not None:
            os.environ["TS_ABLATE"] = ab
        if itn is not None:
            os.environ["TS_REFINE_ITERS"] = itn
        if ct is not None:
            os.environ["TS_SPLIT_CT"] = ct
        if ho is not None:
            os.environ["TS_TET_HOLES"] = ho
        layout = {"edge_gather": bool(ga)}
        if ch:
            layout["max_chunk_slots"] = ch
        if bl:
            layout["block_threads"] = bl
        try:
            ms, info = time_layout(scene, n, prec, layout, grid=int(os.environ.get("TS_GRID", "0")))
            print(f"{prec} gather={ga} ct={ct} holes={ho} ablate={ab} iters={itn} chunk={ch:5d} block={bl:4d}: {ms:.3f} ms/step  {n / ms * 1e3:12,.0f} env-steps/s  "
                  f"chunks={info['n_chunks']} slots={info['slot_capacity']} smem={info['smem_bytes']} "
                  f"conf={info['bank_conflicts_p1']}", flush=True)
        except Exception as exc:
            print(f"{prec} chunk={ch} block={bl}: failed {exc}", flush=True)


if __name__ == "__main__":
    main()
