"""Benchmark: env-steps/s of the batched tissue-reach env step on B200.

    python bench.py [--gpus N --steps K --warmup W] [--impl b200|reference] [--config 3|1|2|5]
    python -m torch.distributed.run --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 \\
        --master-port P bench.py --gpus N --steps K --warmup W

Workloads (BASELINE.json configs; the default is config 3, the metric's own):
  3  4096 envs per GPU, reach_1170, tets + distance + grasp + contact, 10 substeps
  1  1 env (latency-bound: one CTA, or --cluster K CTAs of a thread-block cluster)
  2  1024 envs, distance constraints only (tets emptied as the reference's tests do)
  5  16384 envs per GPU (the scaling sweep's per-GPU shard; --envs up to 65536)

A "step" is one EnvBatch.step over all envs of a GPU: tool command, grasp,
10 substeps of the distance + tet-volume solver, capsule contact, reward /
done / auto-reset -- the per-env command kernel (one thread per env), the
fused sm_100a step kernel (one CTA, or one cluster, per env) and the per-env
epilogue kernel, preceded by the on-device uniform(-1,1) action draw; the five
launches are captured once in a CUDA graph and replayed.  Envs shard across
GPUs with no data-path collective ("scaling": "weak"); the global env id
indexes the action stream so a shard reproduces the single-GPU envs.

value  : device-timed throughput (inputs resident in HBM): CUDA events around
         each graph replay on the replaying stream, L2 flushed between timed
         steps (256 MiB write, untimed), max over ranks.
e2e    : the same metric through the public API with the reference's host
         semantics (EnvBatch.step_numpy: numpy actions in through pinned memory,
         numpy obs / reward / terminated / truncated / info out through one D2H
         copy of the packed output block) inside the timed region.
roofline: the binding roofline of this kernel is on-chip shared memory
         (SURVEY.md §8(d)); achieved = algorithmic bytes per env-step
         (substeps x (128 V + 88 E + 176 T) + 48 V + 64; 4,191,120 B for config 3)
         x envs per launch / the fused step kernel's own time (CUDA events the
         library records around that kernel on its stream, in a second timed
         loop of plain launches), peak = shared-memory bandwidth measured on
         this GPU by ts_smem_probe.  The HBM view is reported beside it
         (roofline_hbm, peak from MEASURED_PEAKS.json).
cpu_baseline: the unmodified reference (oracle/_ref, compiled backend,
         deterministic mode, 16 OpenMP threads) timed on this host on a bounded
         sample of the same workload.
--impl reference: that reference on the same config as a full bench line.
"""

from __future__ import annotations

import argparse
import ctypes
import dataclasses
import json
import os
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

def reference_env(num_envs, seed=0, dist_only=False, threads=REF_THREADS):
    ref_dir = os.path.join(ROOT, "oracle", "_ref")
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
        return env, "reference", threads
    except Exception:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import oracle as O
        from paper_2503_18616_b200.mesh import load_scene
        scene = load_scene(SCENE)
        if dist_only:
            scene = distance_only(scene)
        env = O.OracleEnv(O.scene_from_loaded(*scene), num_envs)
        return env, "port", 1


def time_reference(num_envs, steps, warmup, seed=0, dist_only=False, min_seconds=0.0, max_steps=None):
    """Env-steps/s of the reference on this host: `steps` timed batches, or -- with min_seconds --
    as many as it takes to reach that much CPU time (at most max_steps).  Returns the steps run."""
    threads = min(REF_THREADS, max(1, num_envs))
    env, kind, cores = reference_env(num_envs, seed, dist_only, threads)
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
    return num_envs * done / el, el, kind, cores, done


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

def run_gpu(args, wl):
    import torch
    import torch.distributed as dist

    rank, world, local = env_info()
    # TS_BENCH_DIST=gloo: a test mode that runs several ranks on one GPU (NCCL needs one GPU per rank)
    backend = os.environ.get("TS_BENCH_DIST", "nccl")
    local = local % max(1, torch.cuda.device_count()) if backend == "gloo" else local
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    rdev = dev if backend == "nccl" else torch.device("cpu")   # where the timing reductions run

    from paper_2503_18616_b200 import EnvBatch, _native as N
    from paper_2503_18616_b200.mesh import load_scene

    lib = N.load()
    n = args.envs or wl["envs"]
    first_env = rank * n
    scene = load_scene(SCENE)
    if wl["distance_only"]:
        scene = distance_only(scene)
    mesh = scene[0]
    V, E, T = mesh.vertex_count, len(mesh.edges), len(mesh.tets)
    layout = {"cluster_size": args.cluster} if args.cluster else None
    env = EnvBatch(scene, num_envs=n, device=dev, precision=args.precision, layout=layout)
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
    replay = env.capture_step(acts, pre=draw, warmup=args.warmup)
    for _ in range(2):
        replay()
    torch.cuda.synchronize(dev)
    stream = torch.cuda.current_stream(dev)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    handle = env.sim.scene.handle
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(local) as clocks:
        for i in range(args.steps):
            flush.fill_(i & 0xFF)                       # evict the state from L2 (untimed)
            starts[i].record(stream)
            replay()
            ends[i].record(stream)
        torch.cuda.synchronize(dev)
        # ---- the fused step kernel alone (roofline denominator): plain launches, library events
        N.check(lib.ts_kernel_timing(handle, 1, args.steps), "ts_kernel_timing")
        for i in range(args.steps):
            flush.fill_(i & 0xFF)
            draw()
            env.step(acts, validate=False)
        torch.cuda.synchronize(dev)
    sk_ms, sk_n = ctypes.c_double(0.0), ctypes.c_int64(0)
    N.check(lib.ts_kernel_time(handle, ctypes.byref(sk_ms), ctypes.byref(sk_n)), "ts_kernel_time")
    N.check(lib.ts_kernel_timing(handle, 0, 0), "ts_kernel_timing")
    assert sk_n.value == args.steps, (sk_n.value, args.steps)
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    total_ms = float(np.sum(step_ms))
    t = torch.tensor([total_ms, sk_ms.value], dtype=torch.float64, device=rdev)
    if world > 1:
        dist.barrier()
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms, kern_total_ms = float(t[0]), float(t[1])
    value = world * n * args.steps / (total_ms * 1e-3)
    kern_avg_ms = kern_total_ms / args.steps
    # our kernels inside the timed graph replays
    launches = per_step_launches * args.steps

    # ---- end to end through the public API with host buffers -------------
    rng = np.random.default_rng(1000 + rank)
    host_actions = [rng.uniform(-1.0, 1.0, (n, 3)) for _ in range(args.steps)]
    for i in range(min(2, args.warmup)):
        env.step_numpy(host_actions[i])
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    d2h = env._layout[1]            # the packed output block: obs, reward, flags, info arrays
    for i in range(args.steps):
        o, r, te, tr, _ = env.step_numpy(host_actions[i])   # numpy in / numpy out, reference semantics
    torch.cuda.synchronize(dev)
    e2e_s = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=rdev)
    if world > 1:
        dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
    e2e_value = world * n * args.steps / float(e2e_s[0])

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    info = env.sim.scene.info
    peaks, peak_src = measured_peaks()
    smem_gbs = ctypes.c_double(0.0)
    N.check(lib.ts_smem_probe(local, 20000, ctypes.byref(smem_gbs)), "ts_smem_probe")
    alg = alg_bytes(V, E, T, scene[2].substeps)
    achieved = alg * n / (kern_avg_ms * 1e-3) / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(prof) and args.config == "3" and not args.envs and not args.cluster:
        with open(prof) as fh:
            traffic = json.load(fh).get("dram_bytes_per_launch")
    hbm_achieved = hbm_bytes(V) * n / (kern_avg_ms * 1e-3) / 1e9
    kname = lib.ts_step_kernel_name(handle).decode()   # the instantiation the program selects
    if info["cluster_size"] > 1:
        kname += f" x{info['cluster_size']} CTAs per env"

    line = {
        "metric": wl["metric"], "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32" if args.precision == "fp32" else "f64",
        "data": "synthetic (uniform(-1,1) actions drawn on device; scene reach_1170 from the in-tree preset)",
        "config": {"workload": wl["workload"], "scene": f"reach_1170 (V={V} E={E} T={T} F={len(mesh.surface_faces)})",
                   "envs_per_gpu": n, "global_envs": world * n, "precision": args.precision,
                   "ctas_per_env": info["cluster_size"], "cuda_graph": True,
                   "parallelism": f"env-sharded x{world} (no collective)",
                   "l2": "flushed between timed steps (256 MiB write, untimed)"},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": n * 3 * 8, "d2h_bytes_per_step": d2h},
        "gpu_launches": int(launches),
        "roofline": {"bound": "smem", "achieved": achieved, "peak": smem_gbs.value, "unit": "GB/s",
                     "frac": achieved / smem_gbs.value, "traffic": traffic,
                     "peak_source": "ts_smem_probe on this GPU (conflict-free LDS.128, all SMs)",
                     "algorithmic_bytes_per_env_step": alg, "kernel": kname,
                     "kernel_ms": kern_avg_ms, "envs_per_launch": n},
        "roofline_hbm": {"bound": "hbm", "achieved": hbm_achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                         "frac": hbm_achieved / peaks["hbm_gbs"], "peak_source": peak_src,
                         "algorithmic_bytes_per_env_step": hbm_bytes(V)},
        "clocks": clocks.summary(),
    }
    if world == 1 and not args.no_cpu_baseline:
        # a bounded sample: at least --cpu-steps batches and at least 12 s of CPU work (~10-30 s)
        val, el, kind, cores, cpu_steps = time_reference(n, args.cpu_steps, 1, dist_only=wl["distance_only"],
                                                         min_seconds=12.0, max_steps=200000)
        line["cpu_baseline"] = {"value": val, "unit": UNIT, "cores": cores, "kind": kind,
                                "sample": f"{cpu_steps} env steps x {n} envs after 1 warm-up step "
                                          f"({el:.1f} s), reach_1170{' distance-only' if wl['distance_only'] else ''}, "
                                          f"compiled backend, deterministic mode, {cores} OpenMP threads on "
                                          f"{os.cpu_count()} host cores"}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_reference(args, wl):
    rank, world, local = env_info()
    if rank != 0:
        return
    n = args.envs or wl["envs"]
    threads = min(REF_THREADS, max(1, n))
    env, kind, cores = reference_env(n, 0, wl["distance_only"], threads)
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
        "impl": "reference", "metric": wl["metric"], "value": val, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": el * 1e3 / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (numpy uniform(-1,1) actions)",
        "config": {"workload": wl["workload"] + " (reference CPU implementation)", "envs": n,
                   "parallelism": f"{cores} OpenMP threads"},
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
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    wl = WORKLOADS[args.config]
    if args.impl == "reference":
        run_reference(args, wl)
    else:
        run_gpu(args, wl)


if __name__ == "__main__":
    main()
