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
