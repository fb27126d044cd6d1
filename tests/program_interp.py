"""CPU interpreter of a compiled scene program (test infrastructure).

Executes the kernel's substep data flow -- phase 1 (constraint corrections
into slots) and phase 2 (owner gathers its slots in slot order) -- in numpy
float64 straight from the program blob the sm_100a kernel consumes.  Because
the arithmetic is plain IEEE fp64, the result must be bitwise equal to the
oracle's (and so the reference's) substeps iff the compiler's slot layout,
per-vertex order, counts and chunking are right.  This pins the scene
compiler without a GPU.
"""

from __future__ import annotations

import numpy as np

SECTIONS = ["CHUNK", "EDGE_IDX", "EDGE_PAR", "TET_IDX", "TET_SLOT", "TET_RV", "ATT_IDX", "ATT_SLOT",
            "ATT_PAR", "ATT_ANCHOR", "REGION", "VALENCE", "STATIC_CNT", "S2O", "O2S", "W", "FACES",
            "FACES_ORIG", "REST", "GSPLIT", "EDGE_C", "TET_C", "EINC", "EREGION", "EVAL", "FACE_GID",
            "SEND_OFF", "SEND", "FACE_OWN", "WSPLIT", "RLTAB", "RVTAB"]
HDR_FIELDS = ["magic", "version", "real_bytes", "n_sections", "V", "Vf", "Vf_pad", "Vstore", "F", "B",
              "VPT", "G", "n_chunks", "grasp_chunk", "slot_capacity", "n_att", "n_edge_items",
              "n_tet_items", "n_att_items", "bank_conflicts", "n_slots_total", "compact", "edge_gather",
              "einc_bytes", "Vown", "cluster_k", "cluster_rank", "boff", "rvdict", "narrow", "n_rltab", "n_rvtab"]


class Program:
    def __init__(self, blob: np.ndarray):
        b = blob.view(np.uint8)
        ints = b[:4 * len(HDR_FIELDS)].view(np.int32)
        self.h = dict(zip(HDR_FIELDS, (int(v) for v in ints)))
        assert self.h["magic"] == 0x54534231
        o = 4 * len(HDR_FIELDS)
        self.w_free = float(b[o:o + 8].view(np.float64)[0])
        self.off = b[o + 8:o + 8 + 8 * len(SECTIONS)].view(np.int64)
        self.b = b
        if self.h["compact"]:
            nE, nT = self.h["n_edge_items"], self.h["n_tet_items"]
            self.edge_c = self.sec("EDGE_C", np.uint32, 4 * nE).reshape(nE, 4)
            self.tet_c = self.sec("TET_C", np.uint32, 4 * nT).reshape(nT, 4)
        rt = np.float64 if self.h["real_bytes"] == 8 else np.float32
        H = self.h
        nE, nT, nA = H["n_edge_items"], H["n_tet_items"], H["n_att_items"]
        C, G, Vfp = H["n_chunks"], H["G"], H["Vf_pad"]
        # TsChunk: edge_begin, edge_count, att_begin, att_count, tet_begin, tet_count, slot_count,
        #          region_off, val_off, conflicts, pad, pad
        self.chunks = self.sec("CHUNK", np.int32, C * 12).reshape(C, 12)
        self.edge_idx = self.sec("EDGE_IDX", np.int32, 4 * nE).reshape(nE, 4)
        self.edge_par = self.sec("EDGE_PAR", rt, 4 * nE).reshape(nE, 4).astype(np.float64)
        self.tet_idx = self.sec("TET_IDX", np.int32, 4 * nT).reshape(nT, 4)
        self.tet_slot = self.sec("TET_SLOT", np.int32, 4 * nT).reshape(nT, 4)
        self.tet_rv = self.sec("TET_RV", rt, nT).astype(np.float64)
        self.att_idx = self.sec("ATT_IDX", np.int32, 4 * nA).reshape(nA, 4)
        self.att_slot = self.sec("ATT_SLOT", np.int32, 4 * nA).reshape(nA, 4)
        self.att_par = self.sec("ATT_PAR", rt, 4 * nA).reshape(nA, 4).astype(np.float64)
        self.att_anchor = self.sec("ATT_ANCHOR", rt, 4 * nA).reshape(nA, 4).astype(np.float64)
        self.region = self.sec("REGION", np.int32, C * G).reshape(C, G) if C * G else np.zeros((C, G), np.int32)
        self.valence = self.sec("VALENCE", np.int32, C * Vfp).reshape(C, Vfp) if C * Vfp else np.zeros((C, Vfp), np.int32)
        self.static_cnt = self.sec("STATIC_CNT", np.int32, Vfp)
        self.s2o = self.sec("S2O", np.int32, H["Vstore"])
        self.o2s = self.sec("O2S", np.int32, H["V"])
        self.w = self.sec("W", rt, H["Vstore"]).astype(np.float64)
        self.faces = self.sec("FACES", np.int32, 3 * H["F"]).reshape(-1, 3)
        self.gsplit = self.sec("GSPLIT", np.int32, Vfp)
        if H["edge_gather"]:
            G = H["G"]
            self.eregion = self.sec("EREGION", np.int32, G)
            self.evalence = self.sec("EVAL", np.int32, Vfp)
            eb = H["einc_bytes"]
            n = int(self.eregion[-1] + 32 * self.evalence[32 * (G - 1):32 * G].max()) if G else 0
            raw = self.sec("EINC", np.uint8, max(n, 1) * eb).reshape(-1, eb)
            word = raw[:, 0:4].copy().view(np.uint32)[:, 0]
            self.e_null = np.zeros(len(word), bool)
            if eb == 4:           # {offset | 8 pair index << 16}; pairs {rest, -k_s w_p / (w_p + w_q)}
                tab = self.sec("RLTAB", np.float32, 2 * H["n_rltab"]).reshape(-1, 2).astype(np.float64)
                idx = (word >> 16) >> 3      # the pair's byte offset in the table, 8 B per pair
                self.e_rest = tab[idx, 0]
                self.e_pair_coef = tab[idx, 1]
                self.e_coef = None
                # pair 0 = {0, 0}: a null record (a gap of the conflict-free rounds), whose term is 0
                self.e_null = idx == 0
                word = word & 0xFFFF
            self.e_nbr = (word & 0x7FFFFFFF).astype(np.int32)
            if H["boff"]:
                assert np.all(self.e_nbr % 12 == 0)
                self.e_nbr //= 12                               # fp32 records hold byte offsets
            self.e_nbr_pinned = (word >> 31).astype(bool)       # bit 31: neighbour pinned (w = 0)
            if eb == 4:
                pass
            elif eb == 8:
                self.e_rest = raw[:, 4:8].copy().view(np.float32)[:, 0].astype(np.float64)
                self.e_coef = None
            elif H["real_bytes"] == 8:
                self.e_rest = raw[:, 8:16].copy().view(np.float64)[:, 0]
                self.e_coef = None
            else:
                self.e_coef = raw[:, 4:8].copy().view(np.float32)[:, 0].astype(np.float64)
                self.e_rest = raw[:, 8:12].copy().view(np.float32)[:, 0].astype(np.float64)

    def edge_records(self, p):
        """(neighbour storage positions, rest lengths) of free position p, in gather order (null
        records skipped)."""
        k = np.arange(int(self.evalence[p]))
        r = self.eregion[p // 32] + 32 * k + p % 32
        if hasattr(self, "e_null"):
            r = r[~self.e_null[r]]
        return self.e_nbr[r], self.e_rest[r]

    def edge_nulls(self, p):
        """Null records of free position p that read p's own position: dx = 0, so the kernel counts
        each as a degenerate edge (the compiler adds them to static_cnt).  Nulls reading a pinned
        position are not degenerate and not counted."""
        if not hasattr(self, "e_null"):
            return 0
        k = np.arange(int(self.evalence[p]))
        r = self.eregion[p // 32] + 32 * k + p % 32
        return int((self.e_null[r] & (self.e_nbr[r] == p)).sum())

    def edge_null_count(self, p):
        """All null records of free position p."""
        if not hasattr(self, "e_null"):
            return 0
        k = np.arange(int(self.evalence[p]))
        return int(self.e_null[self.eregion[p // 32] + 32 * k + p % 32].sum())

    def sec(self, name, dtype, count):
        o = int(self.off[SECTIONS.index(name)])
        nbytes = count * np.dtype(dtype).itemsize
        return self.b[o:o + nbytes].view(dtype).copy()


class PartRun:
    """Section C of step_kernel.cuh for one program (or one cluster part) in fp64."""

    def __init__(self, prog: Program, x, v, grasp_vertex, drag, g, h, damping, ks, kv):
        self.prog, self.g, self.h, self.ks, self.kv = prog, np.asarray(g, np.float64), h, ks, kv
        self.drag = np.asarray(drag, np.float64)
        H = prog.h
        self.Vf = Vf = H["Vf"]
        s2o = prog.s2o
        self.valid = s2o >= 0
        self.xs = np.zeros((H["Vstore"], 3))
        self.xs[self.valid] = x[s2o[self.valid]]
        self.vf = v[s2o[:Vf]].copy()
        self.damp = 1.0 if damping == 0.0 else max(0.0, 1.0 - damping * h)
        o = prog.o2s[grasp_vertex] if grasp_vertex >= 0 else -1
        self.gvs = o

    def predict(self):
        self.vf += self.h * self.g[None, :]
        self.xs[:self.Vf] = self.xs[:self.Vf] + self.h * self.vf

    def accumulate(self):
        """Corrections of one substep from the current snapshot: (acc, count adjustment)."""
        prog, xs, Vf, ks, kv = self.prog, self.xs, self.Vf, self.ks, self.kv
        H = prog.h
        gvs, drag = self.gvs, self.drag
        scap = H["slot_capacity"]
        lane = np.arange(Vf) % 32
        grp = np.arange(Vf) // 32
        acc = np.zeros((Vf, 3))
        cnt_adj = np.zeros(Vf, np.int64)
        def owner_edges():
            # owner-gathered distance constraints (step_kernel.cuh owner_edges, fp64 form)
            for p in range(Vf):
                nb, rl = prog.edge_records(p)
                cnt_adj[p] -= prog.edge_nulls(p)
                if len(nb) == 0:
                    continue
                d = xs[p][None, :] - xs[nb]
                dist = np.sqrt((d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1]) + d[:, 2] * d[:, 2])
                m = 0.5 + np.copysign(0.5, dist - 1e-12)
                wp = prog.w[p]
                scale = m * ks * (dist - rl) / (dist * (wp + prog.w[nb]) + (1.0 - m))
                corr = -(wp * scale)[:, None] * d
                for k in range(len(nb)):          # sequential: the reference's summation order
                    acc[p] += corr[k]
                cnt_adj[p] -= int(np.sum(m == 0))

        def add_grasp():
            if 0 <= gvs < Vf:
                d = np.asarray(drag, np.float64) - xs[gvs]
                dist = np.sqrt((d[0] * d[0] + d[1] * d[1]) + d[2] * d[2])
                if not (dist <= 1e-12):
                    acc[gvs] += d
                    cnt_adj[gvs] += 1

        for c in range(H["n_chunks"]):
            eb, ec, ab, ac, tb, tc = (int(v) for v in prog.chunks[c, :6])
            slots = np.full((scap, 3), np.nan)
            deg = np.zeros(H["Vf_pad"], np.int64)
            if ac:
                raise NotImplementedError("attachment chunks are exercised on the GPU tests")
            if ec:
                idx = prog.edge_idx[eb:eb + ec]
                par = prog.edge_par[eb:eb + ec]
                d = xs[idx[:, 0]] - xs[idx[:, 1]]
                dist = np.sqrt((d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1]) + d[:, 2] * d[:, 2])
                m = 0.5 + np.copysign(0.5, dist - 1e-12)
                scale = m * ks * (dist - par[:, 0]) / (dist * par[:, 3] + (1.0 - m))
                ca = -par[:, 1] * scale
                cb = par[:, 2] * scale
                for col, coef, pos in ((2, ca, 0), (3, cb, 1)):
                    sl = idx[:, col]          # -1: pinned endpoint, no slot
                    keep = sl >= 0
                    slots[sl[keep]] = (coef[:, None] * d)[keep]
                    free = idx[:, pos] < H["Vf_pad"]
                    np.add.at(deg, idx[free & (m == 0), pos], 1)
            if tc:
                live = (prog.tet_slot[tb:tb + tc] >= 0).any(axis=1)   # idle lanes of the bank schedule
                idx = prog.tet_idx[tb:tb + tc][live]
                sl = prog.tet_slot[tb:tb + tc][live]
                rv = prog.tet_rv[tb:tb + tc][live]
                pa = xs[idx[:, 0]]
                ba, ca_, da = xs[idx[:, 1]] - pa, xs[idx[:, 2]] - pa, xs[idx[:, 3]] - pa

                def cr(u, w):
                    return np.stack([u[:, 1] * w[:, 2] - u[:, 2] * w[:, 1], u[:, 2] * w[:, 0] - u[:, 0] * w[:, 2],
                                     u[:, 0] * w[:, 1] - u[:, 1] * w[:, 0]], axis=1)
                gb, gc, gd = cr(ca_, da) / 6.0, cr(da, ba) / 6.0, cr(ba, ca_) / 6.0
                ga = -((gb + gc) + gd)
                cval = ((gd[:, 0] * da[:, 0] + gd[:, 1] * da[:, 1]) + gd[:, 2] * da[:, 2]) - rv
                den = np.zeros(len(idx))
                for gg in (ga, gb, gc, gd):
                    for k in range(3):
                        den = den + gg[:, k] * gg[:, k]
                m = 0.5 + np.copysign(0.5, den - 1e-18)
                scv = -m * kv * cval / (den + (1.0 - m))
                for r, gg in enumerate((ga, gb, gc, gd)):
                    keep = sl[:, r] >= 0                           # -1: pinned corner, no slot
                    slots[sl[keep, r]] = (scv[:, None] * gg)[keep]
                    free = idx[:, r] < H["Vf_pad"]
                    np.add.at(deg, idx[free & (m == 0), r], 1)
            # phase 2: slots in order, the grasp spliced after the edge slots of the grasp chunk
            if H["edge_gather"] and c == 0:
                owner_edges()
            base = prog.region[c, grp] + lane
            val = prog.valence[c, :Vf]
            pre = prog.gsplit[:Vf] if c == H["grasp_chunk"] else val
            for k in range(int(pre.max()) if len(pre) else 0):
                live = pre > k
                acc[live] += slots[base[live] + 32 * k]
            if c == H["grasp_chunk"]:
                add_grasp()
                for k in range(int(val.max()) if len(val) else 0):
                    live = (val > k) & (k >= pre)
                    acc[live] += slots[base[live] + 32 * k]
            cnt_adj -= deg[:Vf]
        if H["grasp_chunk"] == H["n_chunks"]:
            if H["edge_gather"] and H["n_chunks"] == 0:
                owner_edges()
            add_grasp()
        return acc, cnt_adj

    def apply(self, acc, cnt_adj, last):
        prog, Vf, h = self.prog, self.Vf, self.h
        n = (prog.static_cnt[:Vf] + cnt_adj).astype(np.float64)
        m = 0.5 + np.copysign(0.5, n - 0.5)
        inv = m / (n + (1.0 - m))
        e = acc * inv[:, None]
        self.xs[:Vf] = self.xs[:Vf] + e
        self.vf = self.vf + e / h
        if self.damp != 1.0:
            self.vf = self.vf * self.damp
        if not last:
            self.vf = self.vf + h * self.g[None, :]
            self.xs[:Vf] = self.xs[:Vf] + h * self.vf

    def write_back(self, x, v):
        prog, Vf = self.prog, self.Vf
        s2o = prog.s2o
        own = np.zeros(len(s2o), bool)
        own[:prog.h["Vown"]] = True
        sel = self.valid & own
        x[s2o[sel]] = self.xs[sel]
        v[s2o[:Vf]] = self.vf
        pinned = s2o[Vf:prog.h["Vown"]]
        v[pinned[pinned >= 0]] = 0.0


def run_substeps(prog: Program, x, v, grasp_vertex, drag, g, h, substeps, damping, ks, kv):
    """One env: x, v (V,3) float64 in place. Mirrors step_kernel.cuh section C."""
    run = PartRun(prog, x, v, grasp_vertex, drag, g, h, damping, ks, kv)
    run.predict()
    for s in range(substeps):
        acc, cnt = run.accumulate()
        run.apply(acc, cnt, s + 1 == substeps)
    run.write_back(x, v)


def cluster_parts(blob: np.ndarray):
    """The part programs of a cluster program (TsClusterHeader + K part blobs)."""
    b = blob.view(np.uint8)
    magic, K = (int(q) for q in b[:8].view(np.int32))
    assert magic == 0x54534331, hex(magic)
    off = b[16:16 + 8 * 16].view(np.int64)
    size = b[16 + 8 * 16:16 + 16 * 16].view(np.int64)
    return [Program(b[int(off[r]):int(off[r]) + int(size[r])].copy()) for r in range(K)]


def run_substeps_cluster(parts, x, v, grasp_vertex, drag, g, h, substeps, damping, ks, kv):
    """The cluster kernel's data flow on CPU: every part computes its owned vertices from its
    local snapshot, then the owners refresh every halo copy (the DSMEM sends)."""
    runs = [PartRun(p, x, v, grasp_vertex, drag, g, h, damping, ks, kv) for p in parts]
    owner = {}
    for r, p in enumerate(parts):
        for q in range(p.h["Vf"]):
            owner[int(p.s2o[q])] = (r, q)

    def refresh():
        for r, p in enumerate(parts):
            for q in range(p.h["Vown"], p.h["Vstore"]):
                o = int(p.s2o[q])
                if o >= 0 and o in owner:
                    rr, qq = owner[o]
                    runs[r].xs[q] = runs[rr].xs[qq]
    for run in runs:
        run.predict()
    refresh()
    for s in range(substeps):
        upd = [run.accumulate() for run in runs]
        for run, (acc, cnt) in zip(runs, upd):
            run.apply(acc, cnt, s + 1 == substeps)
        refresh()
    for run in runs:
        run.write_back(x, v)
