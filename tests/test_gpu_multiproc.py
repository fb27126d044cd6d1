"""Multi-rank paths on the real kernels, on ONE B200 (gloo: NCCL needs one GPU per rank).

* ``bench.py --gpus 2`` (the driver's command form) launches 2 ranks and reports ``n_gpus == 2``;
* the distributed PPO loop -- ``_allreduce_grads`` (one flat all-reduce per minibatch) and
  ``_gather_window`` (episode statistics across ranks), reference ppo.py:254-303, 405-413 -- runs on
  the actual EnvBatch: every rank steps its own env shard and the replicas stay bit-identical.
"""

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.timeout(600)
def test_bench_two_ranks_on_one_gpu():
    env = dict(os.environ, TS_BENCH_DIST="gloo")
    env.pop("WORLD_SIZE", None)
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "5",
                          "--warmup", "3", "--no-cpu-baseline", "--no-extras"],
                         capture_output=True, text=True, env=env, timeout=550)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, res.stdout
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["config"]["global_envs"] == 8192
    assert line["value"] > 0 and line["e2e"]["value"] > 0
    assert line["roofline"]["kernel"] == "tsk::fast_step_kernel<float>"


def _ppo_worker(rank, world, port, out):
    import torch
    import torch.distributed as dist
    from paper_2503_18616_b200 import EnvBatch
    from paper_2503_18616_b200.mesh import default_scene_path, load_scene
    from paper_2503_18616_b200.ppo import PPOConfig, train
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    n = 256
    env = EnvBatch(load_scene(default_scene_path()), num_envs=n, seed=rank, device="cuda:0")
    cfg = PPOConfig.for_num_envs(n, horizon=8, minibatches=4, seed=1, stop_window=64)
    cfg.total_steps = 4 * cfg.steps_before_update
    stats = train(env, cfg)
    flat = torch.cat([p.detach().reshape(-1) for p in stats.model.parameters()]).cpu()
    out[rank] = (flat.numpy().copy(), [r["mean_ep_reward"] for r in stats.rows],
                 [r["env_steps"] for r in stats.rows])
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_ppo_two_ranks_real_env():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_ppo_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    (w0, r0, s0), (w1, r1, s1) = out[0], out[1]
    assert np.isfinite(w0).all()
    assert np.array_equal(w0, w1)                     # gradients averaged: replicas identical
    assert np.allclose(r0, r1, equal_nan=True)        # gathered episode window: same statistics
    assert s0 == s1 == [256 * 8 * 2 * (u + 1) for u in range(4)]   # env steps counted over both ranks
