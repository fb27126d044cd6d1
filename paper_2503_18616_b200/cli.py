"""Command line with the reference's commands and report format (reference
cli.py:22-128 for the CSV columns and the `bench` protocol, 131-170 for `--set` overrides,
173-215 for train / eval, 222-321 for the parser).

    python -m paper_2503_18616_b200.cli bench --num-envs 1,64,4096 [--tets 9729] [--csv out.csv]
    python -m paper_2503_18616_b200.cli bench --mode rl --num-envs 4096
    python -m paper_2503_18616_b200.cli train --num-envs 4096 --out runs/a [--set ppo.learning_rate=1e-3]
    python -m paper_2503_18616_b200.cli eval --checkpoint runs/a/policy.pt --episodes 100
    python -m paper_2503_18616_b200.cli make-scene --tets 52359 --out scenes/

`--set KEY=VALUE` (repeatable) overrides a SceneConfig field, or a PPOConfig field as
`ppo.NAME`, with the reference's casting rules; `--backend` / `--threads` are accepted for
command-line compatibility (the only engine is the sm_100a kernel).

`bench --mode sim` follows the reference's _bench_one_sim protocol (host numpy
uniform(-1, 1) actions, `warmup` untimed batches, ceil(steps / N) timed batches
through the public `EnvBatch.step` API, steps/s = batches x N / wall time), one row
per env count with the mean / std over `runs` seeds; the backend column reads "b200".
"""

from __future__ import annotations

import argparse
import math
import os
import sys
import tempfile
import time
from dataclasses import dataclass, field

import numpy as np

from .errors import CheckpointError, ParseError, SimulationDiverged, ValidationError
from .mesh import SLAB_PRESETS, load_scene, make_slab_scene

CSV_HEADER = "envs,tets,mode,backend,mean_sps,std_sps,available"


@dataclass
class BenchRow:
    envs: int
    tets: int
    mode: str
    backend: str
    mean_sps: float
    std_sps: float
    available: bool = True


@dataclass
class BenchReport:
    rows: list = field(default_factory=list)

    def to_csv(self, path):
        with open(path, "w", encoding="utf-8") as fh:
            fh.write(CSV_HEADER + "\n")
            for r in self.rows:
                fh.write(f"{r.envs},{r.tets},{r.mode},{r.backend},{float(r.mean_sps)!r},"
                         f"{float(r.std_sps)!r},{int(r.available)}\n")

    @classmethod
    def from_csv(cls, path):
        rep = cls()
        with open(path, encoding="utf-8") as fh:
            if not fh.readline().startswith("envs,"):
                raise ParseError(f"{path} is not a benchmark report")
            for line in fh:
                e, t, m, b, mu, sd, av = line.strip().split(",")
                rep.rows.append(BenchRow(int(e), int(t), m, b, float(mu), float(sd), bool(int(av))))
        return rep

    def pretty(self):
        out = [f"{'envs':>6} {'tets':>7} {'mode':>4} {'backend':>8} {'steps/s':>14} {'std':>12}"]
        for r in self.rows:
            val = f"{r.mean_sps:>14.1f} {r.std_sps:>12.1f}" if r.available else f"{'--':>14} {'--':>12}"
            out.append(f"{r.envs:>6} {r.tets:>7} {r.mode:>4} {r.backend:>8} {val}")
        return "\n".join(out)


def _cast_like(current, value):
    """Parse VALUE as the type of the field it replaces (reference cli.py:151-165)."""
    if isinstance(current, bool):
        return value.lower() in ("1", "true", "yes")
    if isinstance(current, int):
        return int(value)
    if isinstance(current, float):
        return float(value)
    if isinstance(current, np.ndarray):
        return np.array([float(t) for t in value.split()], dtype=np.float64)
    if isinstance(current, (tuple, list)):
        return type(current)(int(t) for t in value.split())
    if current is None:
        return float(value)
    return value


def apply_overrides(pairs, scene_cfg, ppo_cfg=None):
    """`--set key=value` pairs onto the scene config, or the PPO config for `ppo.` keys
    (reference cli.py:131-148; same messages)."""
    for pair in pairs or []:
        if "=" not in pair:
            raise ValidationError(f"--set expects key=value, got {pair!r}")
        key, value = pair.split("=", 1)
        key = key.strip()
        if key.startswith("ppo."):
            name = key[4:]
            if ppo_cfg is None or not hasattr(ppo_cfg, name):
                raise ValidationError(f"unknown ppo setting {name!r}")
            setattr(ppo_cfg, name, _cast_like(getattr(ppo_cfg, name), value))
        else:
            if not hasattr(scene_cfg, key):
                raise ValidationError(f"unknown scene setting {key!r}")
            setattr(scene_cfg, key, _cast_like(getattr(scene_cfg, key), value))


def load_scene_with_overrides(scene_path, set_pairs, ppo_cfg=None):
    mesh, rest, cfg = load_scene(scene_path)
    apply_overrides(set_pairs, cfg, ppo_cfg)
    cfg.validate()
    return mesh, rest, cfg


def run_training(scene, out_dir, num_envs=8, seed=0, steps=None, set_pairs=None, verbose=True,
                 precision="fp32") -> int:
    """reference cli.py:173-195: PPO on the GPU env; writes train_log.csv, reward_curve.csv and
    policy.pt under out_dir.  At >= 64 envs the config is the large-batch one
    (`PPOConfig.for_num_envs`); `--set ppo.*` applies on top of either."""
    from . import ppo
    from .env import EnvBatch
    ppo_cfg = ppo.PPOConfig.for_num_envs(num_envs, seed=seed) if num_envs >= 64 else ppo.PPOConfig(seed=seed)
    scene_tuple = load_scene_with_overrides(scene, set_pairs, ppo_cfg)
    if steps is not None:
        ppo_cfg.total_steps = steps
    env = EnvBatch(scene_tuple, num_envs=num_envs, seed=seed, precision=precision)
    try:
        stats = ppo.train(env, ppo_cfg, out_dir=out_dir, verbose=verbose)
    except SimulationDiverged as exc:
        print(f"training aborted: {exc}", file=sys.stderr)
        return 3
    last = stats.rows[-1]
    print(f"finished: {last['env_steps']} env steps, mean episode reward {last['mean_ep_reward']:.2f}, "
          f"wall clock {stats.wall_clock:.1f}s")
    if stats.reward_crossed_at is not None:
        print(f"trailing mean first exceeded 80 at {stats.reward_crossed_at} env steps")
    return 0


def run_eval(checkpoint, scene, episodes=100, num_envs=8, seed=0, set_pairs=None, precision="fp32"):
    """reference cli.py:198-215: greedy episodes of a saved policy."""
    from . import ppo
    from .env import EnvBatch
    if episodes < 1:
        raise ValidationError("episodes must be >= 1")
    scene_tuple = load_scene_with_overrides(scene, set_pairs)
    env = EnvBatch(scene_tuple, num_envs=num_envs, seed=seed, precision=precision)
    model, _ = ppo.load_checkpoint(checkpoint, expect_obs_dim=env.observation_size,
                                   expect_act_dim=env.action_size, device=env.device)
    result = ppo.evaluate(env, model, episodes=episodes, seed=seed)
    print(f"success rate {result['success_rate']:.3f}  mean episode reward {result['mean_reward']:.2f}  "
          f"mean length {result['mean_length']:.1f}")
    return result


def bench_sim(scene, num_envs, steps, seed, warmup=100, precision="fp32"):
    from .env import EnvBatch
    env = EnvBatch(scene, num_envs=num_envs, seed=seed, precision=precision)
    rng = np.random.default_rng(seed)
    env.reset(seed=seed)
    batches = max(1, math.ceil(steps / num_envs))
    for _ in range(warmup):
        env.step(rng.uniform(-1.0, 1.0, (num_envs, 3)))
    import torch
    torch.cuda.synchronize(env.device)
    t0 = time.perf_counter()
    for _ in range(batches):
        env.step(rng.uniform(-1.0, 1.0, (num_envs, 3)))
    torch.cuda.synchronize(env.device)
    return batches * num_envs / (time.perf_counter() - t0)


def bench_rl(scene, num_envs, steps, seed):
    from . import ppo
    from .env import EnvBatch
    env = EnvBatch(scene, num_envs=num_envs, seed=seed)
    cfg = ppo.PPOConfig.for_num_envs(num_envs, seed=seed) if num_envs >= 64 else ppo.PPOConfig(seed=seed)
    cfg.total_steps = max(cfg.steps_before_update, steps)
    stats = ppo.train(env, cfg)
    total = stats.rows[-1]["env_steps"] if stats.rows else cfg.total_steps
    return total / stats.wall_clock


def run_benchmark(mode, env_counts, scene, steps, seeds, warmup=100, precision="fp32") -> BenchReport:
    if steps < 1:
        raise ValidationError("steps must be >= 1")
    if mode not in ("sim", "rl"):
        raise ValidationError("mode must be 'sim' or 'rl'")
    n_tets = len((load_scene(scene) if isinstance(scene, str) else scene)[0].tets)
    rep = BenchReport()
    for count in env_counts:
        rates, available = [], True
        for seed in seeds:
            try:
                rates.append(bench_sim(scene, count, steps, seed, warmup, precision) if mode == "sim"
                             else bench_rl(scene, count, steps, seed))
            except (MemoryError, RuntimeError) as exc:
                if "out of memory" not in str(exc).lower() and not isinstance(exc, MemoryError):
                    raise
                available = False
                break
        arr = np.asarray(rates) if available else np.full(1, np.nan)
        rep.rows.append(BenchRow(count, n_tets, mode, "b200", float(arr.mean()), float(arr.std()), available))
    return rep


def build_parser():
    ap = argparse.ArgumentParser(prog="paper_2503_18616_b200.cli",
                                 description="B200 tissue-reach env: benchmarks, PPO training, evaluation")
    sub = ap.add_subparsers(dest="command", required=True)
    common = argparse.ArgumentParser(add_help=False)
    common.add_argument("--scene", help="scene file path")
    common.add_argument("--tets", type=int, choices=sorted(SLAB_PRESETS), help="generate a slab preset")
    common.add_argument("--seed", type=int, default=0)
    common.add_argument("--backend", default="auto", help="accepted for compatibility: the engine is 'b200'")
    common.add_argument("--threads", type=int, default=None, help="accepted for compatibility")
    common.add_argument("--set", dest="set_pairs", action="append", metavar="KEY=VALUE",
                        help="override a scene setting (or ppo.NAME); repeatable")
    common.add_argument("--precision", choices=("fp32", "fp64"), default="fp32")
    b = sub.add_parser("bench", parents=[common], help="measure env-steps/second")
    b.add_argument("--mode", choices=("sim", "rl"), default="sim")
    b.add_argument("--num-envs", default="1")
    b.add_argument("--steps", type=int, default=2000)
    b.add_argument("--runs", type=int, default=5)
    b.add_argument("--warmup", type=int, default=100)
    b.add_argument("--csv")
    t = sub.add_parser("train", parents=[common], help="train the reach-task policy (PPO on the GPU)")
    t.add_argument("--num-envs", type=int, default=8)
    t.add_argument("--steps", type=int, default=None, help="total env steps (default: the PPO config's)")
    t.add_argument("--out", required=True, help="output directory")
    t.add_argument("--quiet", action="store_true")
    e = sub.add_parser("eval", parents=[common], help="evaluate a trained policy")
    e.add_argument("--checkpoint", required=True)
    e.add_argument("--episodes", type=int, default=100)
    e.add_argument("--num-envs", type=int, default=8)
    m = sub.add_parser("make-scene", help="generate a slab scene")
    m.add_argument("--tets", type=int, default=1170, choices=sorted(SLAB_PRESETS))
    m.add_argument("--out", required=True)
    m.add_argument("--pin", default="y0", choices=("x0", "x1", "y0", "y1"))
    m.add_argument("--spacing", type=float, default=0.0075)
    return ap


def _resolve_scene(args):
    if args.scene:
        return args.scene
    if args.tets:
        return make_slab_scene(os.path.join(tempfile.gettempdir(), "ffsrl_b200_scenes"), tets=args.tets)
    from .mesh import default_scene_path
    return default_scene_path()


def _check_backend(args):
    if args.backend not in (None, "auto", "b200", "cuda"):
        raise ValidationError(f"unknown backend {args.backend!r}; this engine is 'b200' only")


def main(argv=None):
    ap = build_parser()
    args = ap.parse_args(argv)
    try:
        if args.command == "make-scene":
            print(make_slab_scene(args.out, tets=args.tets, spacing=args.spacing, pin=args.pin))
            return 0
        _check_backend(args)
        path = _resolve_scene(args)
        if args.command == "train":
            return run_training(path, args.out, num_envs=args.num_envs, seed=args.seed, steps=args.steps,
                                set_pairs=args.set_pairs, verbose=not args.quiet, precision=args.precision)
        if args.command == "eval":
            run_eval(args.checkpoint, path, episodes=args.episodes, num_envs=args.num_envs, seed=args.seed,
                     set_pairs=args.set_pairs, precision=args.precision)
            return 0
        counts = [int(t) for t in str(args.num_envs).split(",") if t]
        if not counts or min(counts) < 1:
            raise ValidationError("--num-envs needs positive integers")
        scene = load_scene_with_overrides(path, args.set_pairs) if args.set_pairs else path
        rep = run_benchmark(args.mode, counts, scene, args.steps, [args.seed + k for k in range(args.runs)],
                            warmup=args.warmup, precision=args.precision)
        print(rep.pretty())
        if args.csv:
            rep.to_csv(args.csv)
            print(f"wrote {args.csv}")
        return 0
    except (ParseError, ValidationError, CheckpointError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2
    except SimulationDiverged as exc:
        print(f"simulation diverged: {exc}", file=sys.stderr)
        return 3


if __name__ == "__main__":
    sys.exit(main())
