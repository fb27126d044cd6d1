"""Multi-process host logic on CPU (gloo, world_size 2): env sharding, max-over-ranks timing, and that
sharded oracle rollouts reproduce the unsharded rows (envs are independent)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2503_18616_b200.shard import job_throughput, job_time, shard_range, weak_range


def test_shard_ranges_partition():
    for total in (1, 7, 4096, 65536):
        for world in (1, 2, 3, 8):
            if total < world:
                continue
            ranges = [shard_range(total, r, world) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
            sizes = [b - a for a, b in ranges]
            assert max(sizes) - min(sizes) <= 1
    assert weak_range(4096, 3) == (12288, 16384)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    t = job_time(1.0 + rank)                         # rank 1 is slower
    thr = job_throughput(100 * (rank + 1), 1.0 + rank)
    # each rank steps its own shard of an oracle batch; rows must equal the single-process run
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, os.path.join(os.path.dirname(here), "oracle"))
    import oracle as O
    from paper_2503_18616_b200.mesh import default_scene_path, load_scene
    total = 4
    first, last = shard_range(total, rank, world)
    env = O.OracleEnv(O.scene_from_loaded(*load_scene(default_scene_path())), last - first)
    env.reset()
    rng = np.random.default_rng(0)
    for _ in range(3):
        a = rng.uniform(-1, 1, (total, 3))[first:last]
        env.step(a)
    out[rank] = (t, thr, env.x.copy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_gloo_two_ranks():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    assert out[0][0] == out[1][0] == 2.0               # max over ranks
    assert abs(out[0][1] - 300 / 2.0) < 1e-9           # sum of work / max time
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, os.path.join(os.path.dirname(here), "oracle"))
    import oracle as O
    from paper_2503_18616_b200.mesh import default_scene_path, load_scene
    env = O.OracleEnv(O.scene_from_loaded(*load_scene(default_scene_path())), 4)
    env.reset()
    rng = np.random.default_rng(0)
    for _ in range(3):
        env.step(rng.uniform(-1, 1, (4, 3)))
    assert np.array_equal(np.concatenate([out[0][2], out[1][2]]), env.x)


class _FakeReachEnv:
    """CPU stand-in with EnvBatch's step contract (torch tensors, info keys, auto-reset) so the
    distributed PPO loop (gradient all-reduce, episode-window gather) runs under gloo on CPU."""

    observation_size, action_size = 6, 3

    def __init__(self, n, rank):
        import torch
        self.num_envs, self.device = n, torch.device("cpu")
        g = torch.Generator().manual_seed(100 + rank)
        self.target = torch.rand((n, 3), generator=g, dtype=torch.float64)
        self.pos = torch.zeros((n, 3), dtype=torch.float64)
        self.steps = torch.zeros(n, dtype=torch.int64)
        self.ret = torch.zeros(n, dtype=torch.float64)

    def _obs(self):
        import torch
        return torch.cat([self.pos, self.target], 1).float()

    def reset(self, seed=None, indices=None):
        self.pos.zero_(), self.steps.zero_(), self.ret.zero_()
        return self._obs()

    def step(self, action, validate=True):
        import torch
        self.pos += 0.1 * action.double().clamp(-1, 1)
        d = (self.pos - self.target).norm(dim=1)
        term = d < 0.1
        reward = -d + 10.0 * term
        self.steps += 1
        self.ret += reward
        trunc = ~term & (self.steps >= 20)
        done = term | trunc
        final = torch.where(done[:, None], self._obs(), torch.zeros_like(self._obs()))
        info = {"final_observation": final, "diverged": torch.zeros_like(done), "done_mask": done,
                "episode_return": self.ret.clone(), "episode_length": self.steps.clone()}
        self.pos[done] = 0.0
        self.steps[done] = 0
        self.ret[done] = 0.0
        return self._obs(), reward, term, trunc, info


def _ppo_worker(rank, world, port, out):
    import torch
    import torch.distributed as dist
    from paper_2503_18616_b200.ppo import PPOConfig, train
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.set_num_threads(1)
    env = _FakeReachEnv(16, rank)
    cfg = PPOConfig(total_steps=16 * 8 * 4, steps_before_update=16 * 8, minibatch_size=32, epochs=2,
                    hidden_sizes=(16, 16), seed=3, stop_window=8)
    stats = train(env, cfg)
    flat = torch.cat([p.detach().reshape(-1) for p in stats.model.parameters()])
    out[rank] = (flat.numpy().copy(), [r["mean_ep_reward"] for r in stats.rows])
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_ppo_gradient_allreduce_two_ranks():
    """Multi-GPU PPO logic (config 5) on CPU/gloo: each rank rolls its own env shard, gradients are
    averaged with one all-reduce per minibatch, so the replicas stay bit-identical; the reward window
    is gathered across ranks, so both ranks log the same statistics."""
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_ppo_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    w0, r0 = out[0]
    w1, r1 = out[1]
    assert np.array_equal(w0, w1)
    assert np.allclose(r0, r1, equal_nan=True)


@pytest.mark.timeout(300)
def test_bench_gpus_two_launches_two_ranks():
    """`bench.py --gpus 2` outside torchrun re-launches itself as 2 ranks (the driver's command form
    at N > 1); --dry-run exercises the rank / shard / max-over-ranks plumbing on CPU with gloo."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, TS_BENCH_DIST="gloo")
    env.pop("WORLD_SIZE", None)
    res = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--steps", "3",
                          "--warmup", "3", "--dry-run"], capture_output=True, text=True, env=env, timeout=240)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, res.stdout           # rank 0 alone prints
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2
    assert line["shards"] == [[0, 4096], [4096, 8192]]   # weak scaling: 4096 envs per rank
    assert line["job_time"] == 0.002                    # max over ranks


def test_bench_rejects_world_mismatch():
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import bench
    bench.check_world(2, 2)
    with pytest.raises(SystemExit):
        bench.check_world(1, 2)
