"""Turn one GPU round's raw outputs (gpurun_out/) into the tracked evidence under profiles/<tag>/.

    python tools/summarize_profiles.py <tag> [--kernel step_kernel]

Reads gpurun_out/launches_<tag>.csv (ncu gpu__time_duration launch list),
gpurun_out/prof_step_<tag>.ncu-rep (one `ncu --set full` capture of the step
kernel), bench_<tag>.json / bench_ref_<tag>.json, and writes:
  profiles/<tag>/launches.txt        per-kernel launch count, mean time, share of the step
  profiles/<tag>/ncu_full.txt        the counters the roofline / occupancy / stall story uses
  profiles/<tag>/ncu_source.txt      hottest source lines and SASS opcodes (from --page source)
  profiles/<tag>/bench.json          the bench lines of the same round
  profiles/ncu_summary.json          dram bytes per launch etc. (bench.py reads `traffic` from it)
"""

from __future__ import annotations

import collections
import contextlib
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__cycles_elapsed.avg", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__shared_mem_per_block_allocated", "launch__block_size",
    "launch__grid_size", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "launch__occupancy_limit_warps", "launch__waves_per_multiprocessor",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "l1tex__t_sector_pipe_lsu_mem_global_op_ld_hit_rate.pct", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
    "l1tex__t_sectors_pipe_lsu_mem_local_op_st.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
]
STALLS = ["barrier", "wait", "not_selected", "short_scoreboard", "long_scoreboard", "selected",
          "branch_resolving", "mio_throttle", "no_instruction", "dispatch_stall", "math_pipe_throttle", "lg_throttle"]


def launches(tag):
    path = os.path.join(OUT, f"launches_{tag}.csv")
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    per = collections.defaultdict(list)
    for r in rows[start + 1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            name = d["Kernel Name"]
            name = name.split("(")[0] if not name.startswith("void at::") else name[:60]
            if "spin_kernel" in name:   # bench.py's untimed torch.cuda._sleep ahead of its timed loops
                continue
            per[name].append(float(d["Metric Value"].replace(",", "")))
    return per


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (u, v) for h, u, v in zip(hdr, units, vals)}


def num(x):
    try:
        return float(str(x).replace(",", ""))
    except (TypeError, ValueError):
        return float("nan")


def main(tag, kernel="step_kernel"):
    dst = os.path.join(ROOT, "profiles", tag)
    os.makedirs(dst, exist_ok=True)
    summary = {"round_tag": tag}

    # ---- launch list ------------------------------------------------------
    per = launches(tag)
    tot = sum(sum(v) for v in per.values())
    lines = [f"ncu --metrics gpu__time_duration.sum --clock-control none (bench.py --steps 4 --warmup 3): "
             f"cold-cache serialised launch times; compare SHARES, not absolutes",
             f"{'launches':>8s} {'mean us':>10s} {'share':>6s}  kernel"]
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"{len(v):8d} {sum(v) / len(v) / 1e3:10.1f} {100 * sum(v) / tot:5.1f}%  {k}")
    step = [v for k, v in per.items() if kernel in k]
    if step:
        times = step[0]
        no_probe = sum(sum(v) for k, v in per.items() if "smem_probe" not in k and "Fill" not in k
                       and "elementwise" not in k)
        share = sum(times) / no_probe
        lines.append(f"\n{kernel}: {len(times)} launches, mean {sum(times) / len(times) / 1e3:.1f} us; "
                     f"share of the env-step's own launches (step + action generator + reset) {100 * share:.1f}%")
        summary["launch_list_step_us"] = sum(times) / len(times) / 1e3
        summary["launch_list_step_share"] = share
    open(os.path.join(dst, "launches.txt"), "w").write("\n".join(lines) + "\n")

    # ---- full capture -----------------------------------------------------
    rep = os.path.join(OUT, f"prof_step_{tag}.ncu-rep")
    if os.path.exists(rep):
        m = raw_metrics(rep)
        out = [f"ncu --set full --clock-control none --import-source on -k regex:{kernel} -s 3 -c 1 "
               f"python tools/profile_step.py   (4096 envs, fp32, reach_1170)", ""]
        for k in KEYS:
            if k in m:
                out.append(f"{k:85s} {m[k][0]:>14s} {m[k][1]}")
        out.append("")
        out.append("warp stall reasons (smsp__average_warps_issue_stalled_<r>_per_issue_active):")
        for s in STALLS:
            k = f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"
            if k in m:
                out.append(f"  {s:20s} {m[k][1]}")
        open(os.path.join(dst, "ncu_full.txt"), "w").write("\n".join(out) + "\n")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd = num(m["dram__bytes_read.sum"][1]) * scale.get(m["dram__bytes_read.sum"][0], 1)
        wr = num(m["dram__bytes_write.sum"][1]) * scale.get(m["dram__bytes_write.sum"][0], 1)
        summary.update({
            "dram_bytes_per_launch": rd + wr, "dram_read_bytes": rd, "dram_write_bytes": wr,
            "ncu_kernel_us": num(m["gpu__time_duration.sum"][1]),
            "smem_wavefronts": num(m["l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"][1]),
            "smem_pipe_pct_of_peak": num(m["l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"][1]),
            "warps_active_pct": num(m["sm__warps_active.avg.pct_of_peak_sustained_active"][1]),
            "issue_active_pct": num(m["smsp__issue_active.avg.pct_of_peak_sustained_active"][1]),
            "registers_per_thread": num(m["launch__registers_per_thread"][1]),
        })
        buf = io.StringIO()
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        import ncu_lines
        import ncu_sass_summary
        with contextlib.redirect_stdout(buf):
            print("== hottest CUDA source lines (share of executed instructions / stall samples / smem wavefronts)")
            ncu_lines.main(rep, 30)
            print("\n== SASS opcode mix, stall reasons, shared-memory wavefront efficiency")
            ncu_sass_summary.main(rep, 20)
        open(os.path.join(dst, "ncu_source.txt"), "w").write(buf.getvalue())

    # ---- bench lines ------------------------------------------------------
    bl = {}
    for name in (f"bench_{tag}.json", f"bench_ref_{tag}.json"):
        p = os.path.join(OUT, name)
        if os.path.exists(p):
            for ln in open(p):
                ln = ln.strip()
                if ln.startswith("{"):
                    bl[name] = json.loads(ln)
    if bl:
        json.dump(bl, open(os.path.join(dst, "bench.json"), "w"), indent=1)
    json.dump(summary, open(os.path.join(ROOT, "profiles", "ncu_summary.json"), "w"), indent=1)
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], *(sys.argv[2:3]))
