"""Per-CUDA-source-line totals from an ncu report (instructions executed, stall samples, smem wavefronts).
Usage: python tools/ncu_lines.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys


def num(x):
    try:
        return float(x)
    except (TypeError, ValueError):
        return 0.0


def parse(rep):
    """[(file:line, source text, instructions, stall samples, smem wavefronts)] per CUDA source line."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                         capture_output=True, text=True).stdout
    lines = out.splitlines()
    start = next(i for i, ln in enumerate(lines) if ln.startswith('"Line No"'))
    rdr = csv.reader(io.StringIO("\n".join(lines[start:])))
    hdr = next(rdr)
    col = {h: i for i, h in enumerate(hdr)}
    # the second "Source" column is the SASS text; metrics follow
    i_inst = hdr.index("Instructions Executed")
    i_samp = hdr.index("Warp Stall Sampling (All Samples)")
    i_wf = hdr.index("L1 Wavefronts Shared") if "L1 Wavefronts Shared" in col else None
    rows = []
    cur = None
    fname = ""
    for r in rdr:
        if not r:
            continue
        if r[0] in ("File Path", "Function Name", "Line No"):
            if r[0] == "File Path":
                fname = r[1].split("/")[-1][:10]
            continue
        if r[0]:
            cur = [f"{fname}:{r[0]}", r[1][:90], 0.0, 0.0, 0.0]
            rows.append(cur)
        else:
            if cur is None:
                continue
            cur[2] += num(r[i_inst])
            cur[3] += num(r[i_samp])
            if i_wf is not None:
                cur[4] += num(r[i_wf])
    return rows


def phases(rep, ranges, fname=""):
    """Instruction / stall shares of named [first, last) line ranges of one source file."""
    rows = parse(rep)
    tot_i = sum(r[2] for r in rows)
    tot_s = sum(r[3] for r in rows)
    out = []
    for name, a, b in ranges:
        sel = [r for r in rows if r[0].split(":")[0] == fname and a <= int(r[0].split(":")[1]) < b]
        out.append((name, 100 * sum(r[2] for r in sel) / tot_i, 100 * sum(r[3] for r in sel) / tot_s))
    return out


def main(rep, top=40):
    rows = parse(rep)
    tot_i = sum(r[2] for r in rows)
    tot_s = sum(r[3] for r in rows)
    print(f"total inst {tot_i:.4g}  samples {tot_s:.4g}")
    for r in sorted(rows, key=lambda r: -r[3])[:top]:
        print(f"{r[0]:>16s} inst {100 * r[2] / tot_i:5.1f}%  stalls {100 * r[3] / tot_s:5.1f}%  wf {r[4]:9.3g}  {r[1]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
