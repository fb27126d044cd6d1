"""Shared-memory wavefront model of one substep of a compiled fp32 fast program (no GPU needed).

Replays the fast step kernel's shared-memory accesses per warp instruction straight from the
program blob -- phase-1 tet loads / predicated slot stores / dictionary loads, the owner edge
gather, the phase-2 slot sums and the position write-back -- and counts wavefronts the way the
hardware serves a 32-bit warp access: per bank, the number of DISTINCT word addresses (equal
addresses broadcast), the warp access costs the maximum over banks.  Prints ideal (one wavefront
per 32-bit access) vs modelled wavefronts per env-substep by category, so compiler changes can be
judged here before spending GPU time; ncu's l1tex__data_bank_conflicts counters are the check.

    python tools/bank_model.py [--block 320]
"""

from __future__ import annotations

import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

from program_interp import Program  # noqa: E402


def wavefronts(addrs):
    """Wavefronts of one warp-wide 32-bit access at byte addresses `addrs` (active lanes only)."""
    if len(addrs) == 0:
        return 0
    words = np.unique(np.asarray(addrs, np.int64) // 4)
    return int(np.bincount(words % 32, minlength=32).max())


def model(prog: Program):
    H = prog.h
    assert H["real_bytes"] == 4 and H["boff"] and H["narrow"] and H["n_chunks"] == 1, "fast fp32 programs only"
    B, Vf, Vstore = H["B"], H["Vf"], H["Vstore"]
    NW = B // 32
    out = {k: [0, 0] for k in ("tet_load", "tet_store", "tet_rv", "edge_load", "edge_rl", "p2_slot", "p2_write")}

    def acc(cat, addrs):
        out[cat][0] += 1 if len(addrs) else 0
        out[cat][1] += wavefronts(addrs)

    ws = prog.sec("WSPLIT", np.int32, NW + 1)
    ch = prog.chunks[0]
    tb = int(ch[4])
    tc = prog.sec("TET_C", np.uint32, 4 * (H["n_tet_items"] + B)).reshape(-1, 4)
    TAB = 1280
    # addresses relative to smem_base (TS_SMEM_HEAD); the tables sit below it, bank offsets alike
    HEAD = 1792
    for w in range(NW):
        wb, we = int(ws[w]), int(ws[w + 1])
        for j0 in range(wb, we, 32):
            items = [i for i in range(j0, min(j0 + 32, we))]
            q = tc[tb + np.asarray(items)]
            pos = [(q[:, 0] & 0x3FFF), (q[:, 0] >> 16) & 0x3FFF, (q[:, 1] & 0x3FFF), (q[:, 1] >> 16) & 0x3FFF]
            slots = [q[:, 2] & 0xFFFF, q[:, 2] >> 16, q[:, 3] & 0xFFFF, q[:, 3] >> 16]
            for r in range(4):
                for c in range(3):
                    acc("tet_load", HEAD + pos[r].astype(np.int64) + 4 * c)
            ri = ((q[:, 0] >> 14) & 3) | ((q[:, 0] >> 28) & 12) | ((q[:, 1] >> 10) & 48) | ((q[:, 1] >> 24) & 192)
            acc("tet_rv", TAB + 4 * 64 + 4 * ri.astype(np.int64))
            for r in range(4):
                live = slots[r] != 0xFFFF
                for c in range(3):
                    acc("tet_store", HEAD + slots[r][live].astype(np.int64) + 4 * c)
    # owner edge gather (phase 1) and phase-2 slot sums, per warp
    ev = prog.evalence
    val = prog.valence[0]
    reg = prog.region[0]
    raw = prog.sec("EINC", np.uint32, int(prog.eregion[-1] + 32 * ev[32 * (NW - 1):32 * NW].max() + 32))
    for w in range(NW):
        ps = [p for p in range(32 * w, 32 * w + 32) if p < Vf]
        if not ps:
            continue
        for k in range(int(max(ev[p] for p in ps))):
            act = [p for p in ps if k < ev[p]]
            rec = raw[prog.eregion[w] + 32 * k + np.asarray(act) % 32]
            nb = (rec & 0xFFFF).astype(np.int64)
            for c in range(3):
                acc("edge_load", HEAD + nb + 4 * c)
            acc("edge_rl", TAB + (rec >> 16).astype(np.int64))     # {rest, coef} pair (one 64-bit load)
        pitch = H.get("slot_pitch", 32) or 32
        for k in range(int(max(val[p] for p in ps))):
            act = np.asarray([p for p in ps if k < val[p]])
            base = 12 * (Vstore + reg[w] + pitch * k + act % 32)
            for c in range(3):
                acc("p2_slot", HEAD + base + 4 * c)
        for c in range(3):
            acc("p2_write", HEAD + 12 * np.asarray(ps) + 4 * c)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--block", type=int, default=0)
    args = ap.parse_args()
    from paper_2503_18616_b200 import scene as S
    from paper_2503_18616_b200.mesh import default_scene_path, load_scene
    mesh, rest, cfg = load_scene(default_scene_path())
    arr = S.SceneArrays.from_loaded(mesh, rest, cfg)
    kw = {"block_threads": args.block} if args.block else {}
    blob, info = S.compile_program(arr, precision="fp32", **kw)
    prog = Program(np.frombuffer(bytes(blob), np.uint8).copy())
    out = model(prog)
    ti = tm = 0
    for k, (ideal, real) in out.items():
        ti += ideal
        tm += real
        print(f"{k:10s} ideal {ideal:6d}  modelled {real:6d}  x{real / max(ideal, 1):.2f}")
    print(f"{'total':10s} ideal {ti:6d}  modelled {tm:6d}  x{tm / max(ti, 1):.2f}  (per env-substep); "
          f"compiler residual {info['bank_conflicts_p1']}")


if __name__ == "__main__":
    main()


def edge_bounds(prog: Program):
    """Per warp: rounds kmax, the largest bank load of the warp's neighbour multiset (all / free
    neighbours only), the modelled cost (sum over rounds of the max bank multiplicity)."""
    H = prog.h
    B, Vf = H["B"], H["Vf"]
    ev = prog.evalence
    rows = []
    for w in range(B // 32):
        ps = [p for p in range(32 * w, 32 * w + 32) if p < Vf]
        if not ps:
            continue
        nbs = [prog.edge_records(p)[0] for p in ps]
        allb = np.bincount(np.concatenate(nbs) % 32, minlength=32)
        freeb = np.bincount(np.concatenate([n[n < H["Vf_pad"]] for n in nbs]) % 32, minlength=32)
        kmax = max(len(n) for n in nbs)
        cost = 0
        for k in range(kmax):
            a = [n[k] for n in nbs if k < len(n)]
            cost += wavefronts(12 * np.asarray(a))
        rows.append((w, kmax, int(allb.max()), int(freeb.max()), cost))
    return rows
