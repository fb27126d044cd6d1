"""Summarise an ncu source page (--page source --csv --print-source=sass): hot opcodes, stall reasons,
shared-memory wavefront efficiency.  Usage: python tools/ncu_sass_summary.py report.ncu-rep"""
import collections
import csv
import io
import subprocess
import sys


def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True).stdout
    lines = out.splitlines()
    start = next(i for i, ln in enumerate(lines) if ln.startswith('"Address"'))
    return list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))


def num(x):
    try:
        return float(x)
    except (TypeError, ValueError):
        return 0.0


def main(rep, top=25):
    rows = load(rep)
    by_op = collections.Counter()
    samples_op = collections.Counter()
    stalls = collections.Counter()
    smem_wf = smem_ideal = 0.0
    total_inst = 0.0
    for r in rows:
        op = r["Source"].strip().split()[0] if r["Source"].strip() else "?"
        if op.startswith("@"):
            op = r["Source"].strip().split()[1]
        op = op.split(".")[0]
        inst = num(r["Instructions Executed"])
        by_op[op] += inst
        total_inst += inst
        samples_op[op] += num(r["Warp Stall Sampling (All Samples)"])
        for k, v in r.items():
            if k.startswith("stall_") and "Not Issued" not in k:
                stalls[k] += num(v)
        smem_wf += num(r.get("L1 Wavefronts Shared"))
        smem_ideal += num(r.get("L1 Wavefronts Shared Ideal"))
    print(f"total warp instructions {total_inst:.4g}")
    print("top opcodes by executed instructions:")
    for op, n in by_op.most_common(top):
        print(f"  {op:10s} {n:12.4g}  {100 * n / total_inst:5.1f}%   stall samples {samples_op[op]:.0f}")
    tot_st = sum(stalls.values())
    print("stall reasons (all samples):")
    for k, v in stalls.most_common(12):
        print(f"  {k:28s} {100 * v / tot_st:5.1f}%")
    if smem_ideal:
        print(f"shared wavefronts {smem_wf:.4g} ideal {smem_ideal:.4g}  efficiency {smem_ideal / smem_wf:.3f}")
    # hottest individual instructions
    hot = sorted(rows, key=lambda r: -num(r["Warp Stall Sampling (All Samples)"]))[:top]
    print("hottest instructions (stall samples):")
    for r in hot:
        print(f"  {r['Address'][-5:]} {num(r['Warp Stall Sampling (All Samples)']):7.0f} {r['Source'].strip()[:70]}")


if __name__ == "__main__":
    main(sys.argv[1])
