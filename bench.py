"""Benchmark: env-steps/s of the batched tissue-reach env step on B200.

    python bench.py [--gpus N --steps K --warmup W] [--impl b200|reference] [--config 3|1|2|5]
    python -m torch.distributed.run --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 \\
        --master-port P bench.py --gpus N --steps K --warmup W

``--gpus N`` (N > 1) without a torchrun environment re-launches this script
as N ranks under ``torch.distributed.run`` (one process per GPU, NCCL); under
torchrun the world size must equal ``--gpus``.  ``TS_BENCH_DIST=gloo`` puts
several ranks on one GPU (a test mode: NCCL needs one GPU per rank).

Workloads (BASELINE.json configs; the default is config 3, the metric's own):
  3  4096 envs per GPU, reach_1170, tets + distance + grasp + contact, 10 substeps
  1  1 env (latency-bound: one CTA, or --cluster K CTAs of a thread-block cluster)
  2  1024 envs, distance constraints only (tets emptied as the reference's tests do)
  5  16384 envs per GPU (the scaling sweep's per-GPU shard; --envs up to 65536)

A "step" is one EnvBatch.step over all envs of a GPU: tool command, grasp,
10 substeps of the distance + tet-volume solver, capsule contact, reward /
done / auto-reset -- the per-env command kernel (one thread per env), the
fused sm_100a step kernel (one CTA, or one cluster, per env) and the per-env
epilogue kernel, preceded by the on-device uniform(-1,1) action draw; the
launches are captured once in a CUDA graph and replayed.  Envs shard across
GPUs with no data-path collective ("scaling": "weak"); the global env id
indexes the action stream so a shard reproduces the single-GPU envs.

value  : device-timed throughput (inputs resident in HBM): CUDA events around
         each graph replay on the replaying stream, L2 flushed between timed
         steps (256 MiB write, untimed), max over ranks.
e2e    : the same metric through the public API with the reference's host
         semantics (EnvBatch.step_numpy: numpy actions drawn on the host inside
         the timed loop, in through pinned memory; numpy float64 obs / reward /
         terminated / truncated / info out through one D2H copy of the packed
         output block), max over ranks.
roofline: the binding roofline of this kernel is on-chip shared memory
         (SURVEY.md §8(d)); achieved = algorithmic bytes per env-step
         (substeps x (128 V + 88 E + 176 T) + 48 V + 64; 4,191,120 B for config 3)
         x envs per launch / the fused step kernel's own time (CUDA events the
         library records around that kernel on its stream, in a second timed
         loop of plain launches), peak = shared-memory bandwidth measured on
         this GPU by ts_smem_probe.  The HBM view is reported beside it
         (roofline_hbm, peak from MEASURED_PEAKS.json).  traffic = DRAM bytes
         per launch from the committed ncu --set full capture of this kernel.
cpu_baseline: the unmodified reference (oracle/_ref, compiled backend,
         deterministic mode, 16 OpenMP threads) timed on this host on a bounded
         sample of the same workload.
extras : (default run) short device-timed lines of the other configs -- 1, 2
         and 5, config 3 in the fp64 validation build -- each with its own CPU
         sample, and the config-4 PPO run to the reward-80 threshold.  With
         N > 1 ranks: config 5 and the PPO run with its NCCL gradient all-reduce.
--impl reference: that reference on the same config as a full bench line.
"""

from __future__ import annotations

import argparse
import ctypes
import dataclasses
import json
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

UNIT = "env-steps/s"
REF_THREADS = 16
SCENE = os.path.join(ROOT, "paper_2503_18616_b200", "scenes", "reach_1170.scene")
NCU_SUMMARY = os.path.join(ROOT, "profiles", "ncu_summary.json")

WORKLOADS = {
    "3": dict(envs=4096, distance_only=False,
              metric="env-steps/sec (XPBD tissue reach, 4096 envs)",
              workload="config 3: 4096-env tissue reach, tet-volume + distance constraints, grasp + capsule "
                       "contact, 10 substeps, auto-reset"),
    "1": dict(envs=1, distance_only=False,
              metric="env-steps/sec (XPBD tissue reach, 1 env)",
              workload="config 1: single-env tissue reach (reach_1170), full physics, random actions"),
    "2": dict(envs=1024, distance_only=True,
              metric="env-steps/sec (XPBD tissue reach, 1024 envs, distance constraints only)",
              workload="config 2: 1024-env tissue reach, distance constraints only (tets emptied), random "
                       "actions"),
    "5": dict(envs=16384, distance_only=False,
              metric="env-steps/sec (XPBD tissue reach, 16384 envs per GPU)",
              workload="config 5: 16384 envs per GPU shard, full physics"),
}


def alg_bytes(V, E, T, substeps=10):
    """per substep 128 V + 88 E + 176 T bytes of canonical fp32 data flow,
    plus 48 V of HBM state in/out and 64 B of I/O per env-step."""
    return substeps * (128 * V + 88 * E + 176 * T) + 48 * V + 64


def hbm_bytes(V):
    return 48 * V + 64


def env_info():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def check_world(world: int, gpus: int):
    """The rank count torchrun gave us must be the one the driver asked for."""
    if world != gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={world} but --gpus {gpus}; launch N ranks for --gpus N")


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def launch_ranks(gpus: int, argv) -> int:
    """--gpus N > 1 outside torchrun: run this script as N ranks under torch.distributed.run
    (one process per GPU, rendezvous on 127.0.0.1).  Rank 0 prints the JSON line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__), *argv]
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", "1")
    return subprocess.call(cmd, env=env)


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            return json.load(fh), "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


def distance_only(scene):
    """The scene with its tets emptied for the solver (edges / faces keep the full topology), as the
    reference's tests isolate distance constraints (pkg/tests/test_tool.py:198-204)."""
    mesh, rest, cfg = scene
    mesh = dataclasses.replace(mesh, tets=np.zeros((0, 4), np.int32))
    rest = dataclasses.replace(rest, rest_volume=np.zeros(0))
    return mesh, rest, cfg


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        time.sleep(0.25)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = max(mx, float(parts[2]))
            except ValueError:
                continue
            for name, flag in zip(names, parts[5:9]):
                if flag.lower() == "active":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU reference (unmodified tissuesim from oracle/_ref; the oracle port if absent)
# ---------------------------------------------------------------------------

def _cpu_flags():
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("flags"):
                    return set(ln.split(":", 1)[1].split())
    except OSError:
        pass
    return set()


def reference_dir():
    """oracle/_ref (the reference's own -march=native build) when this host's CPU has every
    instruction-set flag of the build host, else the portable x86-64-v3 copy.  -> (dir, march)."""
    ref = os.path.join(ROOT, "oracle", "_ref")
    flags_file = os.path.join(ref, "build_cpu_flags.txt")
    march = "native"
    if os.path.exists(os.path.join(ref, "build_march.txt")):
        with open(os.path.join(ref, "build_march.txt")) as fh:
            march = fh.read().strip()
    if os.path.exists(flags_file):
        with open(flags_file) as fh:
            need = set(fh.read().split())
        if not need <= _cpu_flags() and os.path.isdir(os.path.join(ref, "portable")):
            return os.path.join(ref, "portable"), "x86-64-v3"
    return ref, march


def reference_env(num_envs, seed=0, dist_only=False, threads=REF_THREADS):
    ref_dir, march = reference_dir()
    try:
        sys.path.insert(0, ref_dir)
        from tissuesim import backends
        from tissuesim.env import EnvBatch as RefEnv
        from tissuesim.mesh import load_scene as ref_load
        if not backends.HAVE_COMPILED:
            raise ImportError("compiled backend missing")
        scene = ref_load(SCENE)
        if dist_only:
            scene = distance_only(scene)
        env = RefEnv(scene, num_envs=num_envs, seed=seed, backend="compiled", mode="deterministic",
                     threads=threads)
        return env, "reference", threads, march
    except Exception:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import oracle as O
        from paper_2503_18616_b200.mesh import load_scene
        scene = load_scene(SCENE)
        if dist_only:
            scene = distance_only(scene)
        env = O.OracleEnv(O.scene_from_loaded(*scene), num_envs)
        return env, "port", 1, None


def time_reference(num_envs, steps, warmup, seed=0, dist_only=False, min_seconds=0.0, max_steps=None):
    """Env-steps/s of the reference on this host (the cli.py:70-81 protocol: actions drawn with
    numpy inside the timed loop): `steps` timed batches, or -- with min_seconds -- as many as it
    takes to reach that much CPU time (at most max_steps)."""
    threads = min(REF_THREADS, max(1, num_envs))
    env, kind, cores, march = reference_env(num_envs, seed, dist_only, threads)
    env.reset(seed=seed) if kind == "reference" else env.reset()
    rng = np.random.default_rng(seed)
    for _ in range(warmup):
        env.step(rng.uniform(-1.0, 1.0, (num_envs, 3)))
    t0 = time.perf_counter()
    done = 0
    while done < steps or (min_seconds and time.perf_counter() - t0 < min_seconds
                           and (max_steps is None or done < max_steps)):
        env.step(rng.uniform(-1.0, 1.0, (num_envs, 3)))
        done += 1
    el = time.perf_counter() - t0
    return dict(value=num_envs * done / el, seconds=el, kind=kind, cores=cores, steps=done, march=march)


def cpu_baseline(n, dist_only, min_seconds, min_steps=1):
    r = time_reference(n, min_steps, 1, dist_only=dist_only, min_seconds=min_seconds, max_steps=200000)
    build = f"-march={r['march']}" if r["march"] else "oracle port"
    return {"value": r["value"], "unit": UNIT, "cores": r["cores"], "kind": r["kind"],
            "sample": f"{r['steps']} env steps x {n} envs after 1 warm-up step ({r['seconds']:.1f} s), "
                      f"reach_1170{' distance-only' if dist_only else ''}, compiled backend ({build}), "
                      f"deterministic mode, {r['cores']} OpenMP threads on {os.cpu_count()} host cores"}


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

class Ctx:
    """Rank layout and the process group (one process per GPU)."""

    def __init__(self, gpus):
        import torch
        import torch.distributed as dist
        self.rank, self.world, local = env_info()
        check_world(self.world, gpus)
        self.backend = os.environ.get("TS_BENCH_DIST", "nccl")
        ndev = torch.cuda.device_count()
        if self.backend == "gloo":
            local = local % max(1, ndev)
        elif self.world > 1 and ndev < self.world:
            raise SystemExit(f"bench.py: --gpus {gpus} needs {gpus} GPUs, found {ndev}")
        if self.world > 1:
            if self.backend == "nccl":
                dist.init_process_group("nccl", device_id=torch.device("cuda", local))
            else:
                dist.init_process_group(self.backend)
        self.local = local
        torch.cuda.set_device(local)
        self.dev = torch.device("cuda", local)
        self.rdev = self.dev if self.backend == "nccl" else torch.device("cpu")   # timing reductions

    def barrier(self):
        if self.world > 1:
            import torch.distributed as dist
            dist.barrier()

    def max(self, *vals):
        """Max over ranks of per-rank values (the job is as slow as its slowest rank)."""
        import torch
        import torch.distributed as dist
        t = torch.tensor(vals, dtype=torch.float64, device=self.rdev)
        if self.world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return [float(x) for x in t.cpu()]

    def close(self):
        if self.world > 1:
            import torch.distributed as dist
            dist.barrier()
            dist.destroy_process_group()


def load_workload(wl):
    from paper_2503_18616_b200.mesh import load_scene
    scene = load_scene(SCENE)
    if wl["distance_only"]:
        scene = distance_only(scene)
    return scene


def measure(ctx, wl, n, steps, warmup, precision="fp32", cluster=0, e2e=True, flush_l2=True):
    """Device-timed (CUDA-graph replays) and kernel-timed (library events) runs of one workload on
    this rank's GPU, plus the end-to-end host-API run.  Times are maxed over ranks."""
    import torch
    from paper_2503_18616_b200 import EnvBatch, _native as N
    from paper_2503_18616_b200.shard import weak_range

    lib = N.load()
    dev = ctx.dev
    first_env, _ = weak_range(n, ctx.rank)
    scene = load_workload(wl)
    layout = {"cluster_size": cluster} if cluster else None
    env = EnvBatch(scene, num_envs=n, device=dev, precision=precision, layout=layout)
    env.reset(seed=0)
    acts = torch.empty((n, 3), dtype=torch.float64, device=dev)
    counter = torch.zeros(1, dtype=torch.int64, device=dev)
    stream_ptr = lambda: ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)  # noqa: E731
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)   # > 126 MB L2

    def draw():   # uniform(-1, 1) actions; the counter advances on the device (graph replays)
        N.check(lib.ts_uniform_actions_dev(N.ptr(acts), n, first_env, 12345, N.ptr(counter), stream_ptr()),
                "ts_uniform_actions_dev")

    # our kernels per step (action draw + command + step + epilogue), counted by the library on an
    # eager step; the graph replays below launch exactly these
    n0 = lib.ts_launch_count()
    draw()
    env.step(acts, validate=False)
    per_step_launches = lib.ts_launch_count() - n0
    # ---- device-timed: the graph-captured step (W warm-up steps run inside capture_step) ------
    replay = env.capture_step(acts, pre=draw, warmup=warmup)
    for _ in range(2):
        replay()
    torch.cuda.synchronize(dev)
    stream = torch.cuda.current_stream(dev)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    handle = env.sim.scene.handle
    ctx.barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(ctx.local) as clocks:
        # ~5 ms of GPU work ahead of the timed launches (untimed: the first event follows it), so a
        # host stall (the clock sampler thread, the GIL) never leaves the GPU idle inside a bracket
        torch.cuda._sleep(10_000_000)
        for i in range(steps):
            if flush_l2:
                flush.fill_(i & 0xFF)                   # evict the state from L2 (untimed)
            starts[i].record(stream)
            replay()
            ends[i].record(stream)
        torch.cuda.synchronize(dev)
        # ---- the fused step kernel alone (roofline denominator): plain launches, library events
        N.check(lib.ts_kernel_timing(handle, 1, steps), "ts_kernel_timing")
        torch.cuda._sleep(10_000_000)   # see above: the host queues ahead of the GPU
        for i in range(steps):
            if flush_l2:
                flush.fill_(i & 0xFF)
            draw()
            env.step(acts, validate=False)
        torch.cuda.synchronize(dev)
    sk_ms, sk_n = ctypes.c_double(0.0), ctypes.c_int64(0)
    N.check(lib.ts_kernel_time(handle, ctypes.byref(sk_ms), ctypes.byref(sk_n)), "ts_kernel_time")
    N.check(lib.ts_kernel_timing(handle, 0, 0), "ts_kernel_timing")
    assert sk_n.value == steps, (sk_n.value, steps)
    total_ms = float(np.sum([s.elapsed_time(e) for s, e in zip(starts, ends)]))
    ctx.barrier()
    total_ms, kern_total_ms = ctx.max(total_ms, sk_ms.value)
    out = {"n": n, "steps": steps, "ms_per_step": total_ms / steps, "kernel_ms": kern_total_ms / steps,
           "value": ctx.world * n * steps / (total_ms * 1e-3), "launches": per_step_launches * steps,
           "clocks": clocks.summary(), "kernel": lib.ts_step_kernel_name(handle).decode(),
           "info": dict(env.sim.scene.info), "mesh": scene[0], "substeps": scene[2].substeps}
    if out["info"]["cluster_size"] > 1:
        out["kernel"] += f" x{out['info']['cluster_size']} CTAs per env"
    del flush
    if not e2e:
        return out
    # ---- end to end through the public API with host buffers (reference semantics) ----------
    rng = np.random.default_rng(1000 + ctx.rank)
    act = np.empty((n, 3))

    def draw_host():
        # rng.uniform(-1, 1, (n, 3)) drawn into one buffer: -1 + 2 u, the same values (numpy's
        # uniform is low + (high - low) u) without a fresh array per step
        rng.random(out=act)
        np.multiply(act, 2.0, out=act)
        np.subtract(act, 1.0, out=act)
        return act

    for _ in range(min(2, warmup)):
        env.step_numpy(draw_host())
    ctx.barrier()
    torch.cuda.synchronize(dev)
    d2h0 = env.numpy_d2h_bytes
    t0 = time.perf_counter()
    for _ in range(steps):
        # the cli.py:70-81 protocol: numpy actions drawn inside the timed loop; numpy out
        o, r, te, tr, _ = env.step_numpy(draw_host())
    torch.cuda.synchronize(dev)
    (e2e_s,) = ctx.max(time.perf_counter() - t0)
    out["e2e"] = {"value": ctx.world * n * steps / e2e_s, "unit": UNIT, "h2d_bytes_per_step": n * 3 * 8,
                  "d2h_bytes_per_step": (env.numpy_d2h_bytes - d2h0) / steps, "obs_dtype": str(o.dtype),
                  "d2h_note": "output block every step; final observations (n x 6 f64) only on steps with a "
                              "done row"}
    return out


def roofline(m, smem_gbs, traffic=None):
    mesh = m["mesh"]
    V, E, T = mesh.vertex_count, len(mesh.edges), len(mesh.tets)
    alg = alg_bytes(V, E, T, m["substeps"])
    achieved = alg * m["n"] / (m["kernel_ms"] * 1e-3) / 1e9
    return {"bound": "smem", "achieved": achieved, "peak": smem_gbs, "unit": "GB/s", "frac": achieved / smem_gbs,
            "traffic": traffic, "peak_source": "ts_smem_probe on this GPU (conflict-free LDS.128, all SMs)",
            "algorithmic_bytes_per_env_step": alg, "kernel": m["kernel"], "kernel_ms": m["kernel_ms"],
            "envs_per_launch": m["n"]}


def ncu_traffic(kernel):
    """DRAM bytes per launch of `kernel` from the committed ncu --set full capture (or None)."""
    if not os.path.exists(NCU_SUMMARY):
        return None, None
    with open(NCU_SUMMARY) as fh:
        s = json.load(fh)
    if s.get("kernel") and s["kernel"] not in kernel:
        return None, None
    return s.get("dram_bytes_per_launch"), s.get("source")


def extra_line(ctx, key, n, steps, warmup, smem_gbs, precision="fp32", cpu_seconds=3.0, cpu=True):
    wl = WORKLOADS[key]
    m = measure(ctx, wl, n, steps, warmup, precision=precision)
    rec = {"metric": wl["metric"], "workload": wl["workload"], "envs_per_gpu": n, "precision": precision,
           "value": m["value"], "unit": UNIT, "ms_per_step": m["ms_per_step"], "steps": steps,
           "e2e": m["e2e"], "gpu_launches": m["launches"], "roofline": roofline(m, smem_gbs),
           "clocks": m["clocks"]}
    if cpu and ctx.world == 1:
        rec["cpu_baseline"] = cpu_baseline(n, wl["distance_only"], cpu_seconds)
    return rec


def ppo_record(ctx, envs=4096, max_updates=120, window=100):
    """Config 4 (and, with N ranks, config 5's NCCL gradient all-reduce): on-GPU PPO to the
    reference's stop rule (trailing-`window`-episode mean reward > 80 held for stop_patience
    updates, ppo.py:405-413); wall clock to the crossing, then a greedy evaluation."""
    import torch
    from paper_2503_18616_b200 import EnvBatch
    from paper_2503_18616_b200.ppo import PPOConfig, evaluate, train
    env = EnvBatch(load_workload(WORKLOADS["3"]), num_envs=envs, seed=ctx.rank, device=ctx.dev)
    cfg = PPOConfig.for_num_envs(envs, stop_at_reward=80.0, stop_window=window, seed=0)
    cfg.total_steps = max_updates * cfg.steps_before_update
    torch.cuda.synchronize(ctx.dev)
    ctx.barrier()
    t0 = time.perf_counter()
    stats = train(env, cfg)
    torch.cuda.synchronize(ctx.dev)
    (wall,) = ctx.max(time.perf_counter() - t0)
    ev = evaluate(env, stats.model, episodes=500, seed=123)
    return {"metric": f"wall-clock to trailing-{window}-episode mean reward > 80 "
                      f"(held {cfg.stop_patience} updates; on-GPU PPO, tissue reach)",
            "reward_crossed_at_env_steps": stats.reward_crossed_at,
            "reward_crossed_wall_s": stats.reward_crossed_wall, "wall_s": wall, "updates": len(stats.rows),
            "n_gpus": ctx.world, "envs_per_gpu": envs, "stop_window": window,
            "gradient_allreduce": (f"{ctx.backend} all_reduce of one flat fp32 buffer per minibatch"
                                   if ctx.world > 1 else "none (1 rank)"),
            "config": {k: getattr(cfg, k) for k in (
                "steps_before_update", "minibatch_size", "epochs", "learning_rate", "clip_range", "gamma",
                "gae_lambda", "log_std_final", "log_std_anneal_frac", "total_steps", "stop_patience")},
            "final_mean_reward": stats.rows[-1]["mean_ep_reward"] if stats.rows else None,
            "eval_greedy_500_episodes": ev,
            "reference_cpu": "P8: reward > 80 at 269,312 env steps, 148 s wall on 8 envs (SURVEY.md §6(B))"}


def run_gpu(args, wl):
    from paper_2503_18616_b200 import _native as N

    ctx = Ctx(args.gpus)
    lib = N.load()
    n = args.envs or wl["envs"]
    m = measure(ctx, wl, n, args.steps, args.warmup, precision=args.precision, cluster=args.cluster)
    smem_gbs = ctypes.c_double(0.0)
    N.check(lib.ts_smem_probe(ctx.local, 20000, ctypes.byref(smem_gbs)), "ts_smem_probe")
    peaks, peak_src = measured_peaks()
    traffic, traffic_src = ncu_traffic(m["kernel"]) if (args.config == "3" and not args.envs
                                                        and not args.cluster) else (None, None)
    mesh = m["mesh"]
    V, E, T = mesh.vertex_count, len(mesh.edges), len(mesh.tets)
    hbm_achieved = hbm_bytes(V) * n / (m["kernel_ms"] * 1e-3) / 1e9
    line = {
        "metric": wl["metric"], "value": m["value"], "unit": UNIT, "n_gpus": ctx.world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": m["ms_per_step"], "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32" if args.precision == "fp32" else "f64",
        "data": "synthetic (uniform(-1,1) actions drawn on device; scene reach_1170 from the in-tree preset)",
        "config": {"workload": wl["workload"], "scene": f"reach_1170 (V={V} E={E} T={T} F={len(mesh.surface_faces)})",
                   "envs_per_gpu": n, "global_envs": ctx.world * n, "precision": args.precision,
                   "ctas_per_env": m["info"]["cluster_size"], "cuda_graph": True,
                   "parallelism": f"env-sharded x{ctx.world} (no collective), {ctx.backend}",
                   "l2": "flushed between timed steps (256 MiB write, untimed)"},
        "e2e": m["e2e"],
        "gpu_launches": int(m["launches"]),
        "roofline": roofline(m, smem_gbs.value, traffic),
        "roofline_hbm": {"bound": "hbm", "achieved": hbm_achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                         "frac": hbm_achieved / peaks["hbm_gbs"], "peak_source": peak_src,
                         "algorithmic_bytes_per_env_step": hbm_bytes(V)},
        "clocks": m["clocks"],
    }
    if traffic_src:
        line["roofline"]["traffic_source"] = traffic_src
    if ctx.world == 1 and not args.no_cpu_baseline:
        # a bounded sample: at least --cpu-steps batches and at least 12 s of CPU work (~10-30 s)
        line["cpu_baseline"] = cpu_baseline(n, wl["distance_only"], 12.0, args.cpu_steps)
    if not args.no_extras and args.config == "3" and not args.envs and not args.cluster:
        ex = {}
        t_ex = time.perf_counter()
        if ctx.world == 1:
            ex["config1"] = extra_line(ctx, "1", 1, 200, args.warmup, smem_gbs.value, cpu_seconds=3.0)
            ex["config2"] = extra_line(ctx, "2", 1024, 20, args.warmup, smem_gbs.value, cpu_seconds=3.0)
            ex["config3_fp64"] = extra_line(ctx, "3", n, 10, args.warmup, smem_gbs.value, precision="fp64",
                                            cpu=False)
            ex["config3_fp64"]["note"] = ("fp64 validation build (bitwise vs the reference with pose "
                                          "injection): the equal-precision comparison with the CPU arm")
        ex["config5"] = extra_line(ctx, "5", 16384, 10, args.warmup, smem_gbs.value, cpu_seconds=3.0)
        ex["config4_ppo"] = ppo_record(ctx)
        ex["extras_wall_s"] = time.perf_counter() - t_ex
        line["extras"] = ex
    if ctx.rank == 0:
        print(json.dumps(line, default=str), flush=True)
    ctx.close()


def run_dry(args, wl):
    """--dry-run: the launch / rank / shard plumbing without a GPU (gloo) -- rank 0 prints the layout."""
    import torch.distributed as dist
    from paper_2503_18616_b200.shard import job_time, weak_range
    rank, world, _ = env_info()
    check_world(world, args.gpus)
    if world > 1:
        dist.init_process_group("gloo")
    n = args.envs or wl["envs"]
    shard = weak_range(n, rank)
    shards = [None] * world
    if world > 1:
        dist.all_gather_object(shards, shard)
    else:
        shards = [shard]
    t = job_time(0.001 * (rank + 1))
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "shards": shards, "job_time": t,
                          "metric": wl["metric"]}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_reference(args, wl):
    rank, world, local = env_info()
    if rank != 0:
        return
    n = args.envs or wl["envs"]
    threads = min(REF_THREADS, max(1, n))
    env, kind, cores, march = reference_env(n, 0, wl["distance_only"], threads)
    env.reset(seed=0) if kind == "reference" else env.reset()
    rng = np.random.default_rng(0)
    for _ in range(args.warmup):
        env.step(rng.uniform(-1.0, 1.0, (n, 3)))
    t0 = time.perf_counter()
    for _ in range(args.steps):
        env.step(rng.uniform(-1.0, 1.0, (n, 3)))
    el = time.perf_counter() - t0
    val = n * args.steps / el
    line = {
        "impl": "reference", "metric": wl["metric"], "value": val, "unit": UNIT, "n_gpus": max(world, args.gpus),
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": el * 1e3 / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (numpy uniform(-1,1) actions)",
        "config": {"workload": wl["workload"] + " (reference CPU implementation)", "envs": n,
                   "parallelism": f"{cores} OpenMP threads, -march={march}"},
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": kind,
                         "sample": f"{args.steps} env steps x {n} envs after {args.warmup} warm-up steps"},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("b200", "reference"), default="b200")
    ap.add_argument("--config", choices=sorted(WORKLOADS), default="3")
    ap.add_argument("--envs", type=int, default=0, help="envs per GPU (0: the config's)")
    ap.add_argument("--cluster", type=int, default=0, help="CTAs per env (0: automatic)")
    ap.add_argument("--precision", choices=("fp32", "fp64"), default="fp32")
    ap.add_argument("--cpu-steps", type=int, default=2, help="minimum timed CPU-baseline batches (and >= 12 s)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the other configs and the PPO run")
    ap.add_argument("--dry-run", action="store_true", help="rank / shard plumbing only (no GPU; gloo)")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    wl = WORKLOADS[args.config]
    if args.impl == "reference":
        run_reference(args, wl)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(launch_ranks(args.gpus, sys.argv[1:]))
    if args.dry_run:
        run_dry(args, wl)
    else:
        run_gpu(args, wl)


if __name__ == "__main__":
    main()
