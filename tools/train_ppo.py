"""Config 4 / 5: on-GPU PPO on the 4096-env tissue reach to the reward-80 threshold (wall clock).

    python tools/train_ppo.py [--envs 4096] [--horizon 16] [--max-updates 200]
    python -m torch.distributed.run --nproc-per-node N tools/train_ppo.py ...   (NCCL gradient all-reduce)

Prints one JSON line: env steps and wall-clock seconds when the trailing
100-episode mean first held above 80 for 5 updates (ppo.py:405-413 rule),
plus a greedy evaluation of the final policy.
"""
import argparse
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2503_18616_b200 import EnvBatch  # noqa: E402
from paper_2503_18616_b200.mesh import default_scene_path, load_scene  # noqa: E402
from paper_2503_18616_b200.ppo import PPOConfig, evaluate, train  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--envs", type=int, default=4096)
    ap.add_argument("--horizon", type=int, default=16)
    ap.add_argument("--minibatches", type=int, default=4)
    ap.add_argument("--epochs", type=int, default=5)
    ap.add_argument("--lr", type=float, default=1e-3)
    ap.add_argument("--clip", type=float, default=0.2)
    ap.add_argument("--anneal-frac", type=float, default=0.5)
    ap.add_argument("--max-updates", type=int, default=150)
    ap.add_argument("--stop", type=float, default=80.0)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--window", type=int, default=0,
                    help="episodes in the trailing reward mean (0 = one per env of the whole job; "
                         "100 = the reference's rule, ppo.py:405-413)")
    ap.add_argument("--precision", default="fp32")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    env = EnvBatch(load_scene(default_scene_path()), num_envs=args.envs, seed=args.seed + rank, device=dev,
                   precision=args.precision)
    cfg = PPOConfig.for_num_envs(args.envs, horizon=args.horizon, minibatches=args.minibatches, epochs=args.epochs,
                                 learning_rate=args.lr, clip_range=args.clip, log_std_anneal_frac=args.anneal_frac,
                                 seed=args.seed, stop_at_reward=args.stop,
                                 stop_window=args.window or args.envs * world)
    cfg.total_steps = args.max_updates * cfg.steps_before_update
    t0 = time.perf_counter()
    stats = train(env, cfg, out_dir=args.out, verbose=(rank == 0))
    wall = time.perf_counter() - t0
    ev = evaluate(env, stats.model, episodes=500, seed=123) if rank == 0 else None
    if rank == 0:
        print(json.dumps({
            "metric": f"wall-clock to trailing-{cfg.stop_window}-episode mean reward > 80 (on-GPU PPO, tissue reach)",
            "reward_crossed_at_env_steps": stats.reward_crossed_at, "reward_crossed_wall_s": stats.reward_crossed_wall,
            "stopped_early_at": stats.stopped_early_at, "wall_s": wall, "updates": len(stats.rows),
            "n_gpus": world, "envs_per_gpu": args.envs, "stop_window": cfg.stop_window,
            "config": {k: getattr(cfg, k) for k in (
                "steps_before_update", "minibatch_size", "epochs", "learning_rate", "clip_range", "gamma",
                "gae_lambda", "log_std_final", "log_std_anneal_frac", "total_steps")},
            "final_mean_reward": stats.rows[-1]["mean_ep_reward"] if stats.rows else None,
            "eval": ev}), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
