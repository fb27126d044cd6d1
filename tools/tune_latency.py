"""Single-env (config 1) step time for several CTA sizes and phase-1 split weights: graph replays
timed back to back with CUDA events (development tool).

    gpurun -- python tools/tune_latency.py
"""
import ctypes
import itertools
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2503_18616_b200 import EnvBatch, _native as N  # noqa: E402
from paper_2503_18616_b200.mesh import default_scene_path, load_scene  # noqa: E402

scene = load_scene(default_scene_path())
n = int(os.environ.get("TS_ENVS", "1"))
lib = N.load()
blocks = [int(b) for b in os.environ.get("TS_BLOCKS", "320,384,448,512").split(",")]
cts = os.environ.get("TS_CTS", "4").split(",")
for bl, ct in itertools.product(blocks, cts):
    os.environ["TS_SPLIT_CT"] = ct
    env = EnvBatch(scene, num_envs=n, device="cuda:0", layout={"block_threads": bl})
    env.reset()
    acts = torch.empty((n, 3), dtype=torch.float64, device="cuda:0")
    counter = torch.zeros(1, dtype=torch.int64, device="cuda:0")

    def draw():
        N.check(lib.ts_uniform_actions_dev(N.ptr(acts), n, 0, 7, N.ptr(counter),
                                           ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)), "draw")

    replay = env.capture_step(acts, pre=draw, warmup=5)
    for _ in range(20):
        replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    K = 500
    torch.cuda._sleep(10_000_000)
    e0.record()
    for _ in range(K):
        replay()
    e1.record()
    e1.synchronize()
    print(f"block {bl} ct {ct}: {e0.elapsed_time(e1) / K * 1e3:.1f} us/step  "
          f"({lib.ts_step_kernel_name(env.sim.scene.handle).decode()})", flush=True)
