"""Benchmark front end with the reference's report format (reference
cli.py:22-128, 222-321 for the CSV columns and the `bench` protocol).

    python -m paper_2503_18616_b200.cli bench --num-envs 1,64,4096 [--tets 9729] [--csv out.csv]
    python -m paper_2503_18616_b200.cli bench --mode rl --num-envs 4096
    python -m paper_2503_18616_b200.cli make-scene --tets 52359 --out scenes/

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

from .errors import ParseError, ValidationError
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
    n_tets = len(load_scene(scene)[0].tets)
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
                                 description="B200 tissue-reach env: benchmarks and scene generation")
    sub = ap.add_subparsers(dest="command", required=True)
    b = sub.add_parser("bench", help="measure env-steps/second")
    b.add_argument("--scene")
    b.add_argument("--tets", type=int, choices=sorted(SLAB_PRESETS))
    b.add_argument("--mode", choices=("sim", "rl"), default="sim")
    b.add_argument("--num-envs", default="1")
    b.add_argument("--steps", type=int, default=2000)
    b.add_argument("--runs", type=int, default=5)
    b.add_argument("--warmup", type=int, default=100)
    b.add_argument("--seed", type=int, default=0)
    b.add_argument("--precision", choices=("fp32", "fp64"), default="fp32")
    b.add_argument("--csv")
    m = sub.add_parser("make-scene", help="generate a slab scene")
    m.add_argument("--tets", type=int, default=1170, choices=sorted(SLAB_PRESETS))
    m.add_argument("--out", required=True)
    m.add_argument("--pin", default="y0", choices=("x0", "x1", "y0", "y1"))
    m.add_argument("--spacing", type=float, default=0.0075)
    return ap


def main(argv=None):
    ap = build_parser()
    args = ap.parse_args(argv)
    try:
        if args.command == "make-scene":
            print(make_slab_scene(args.out, tets=args.tets, spacing=args.spacing, pin=args.pin))
            return 0
        scene = args.scene
        if not scene and args.tets:
            scene = make_slab_scene(os.path.join(tempfile.gettempdir(), "ffsrl_b200_scenes"), tets=args.tets)
        if not scene:
            from .mesh import default_scene_path
            scene = default_scene_path()
        counts = [int(t) for t in str(args.num_envs).split(",") if t]
        if not counts or min(counts) < 1:
            raise ValidationError("--num-envs needs positive integers")
        rep = run_benchmark(args.mode, counts, scene, args.steps, [args.seed + k for k in range(args.runs)],
                            warmup=args.warmup, precision=args.precision)
        print(rep.pretty())
        if args.csv:
            rep.to_csv(args.csv)
            print(f"wrote {args.csv}")
        return 0
    except (ParseError, ValidationError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
