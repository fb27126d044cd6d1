"""The scene compiler's program (what the sm_100a kernel executes), pinned on CPU.

* Interpreting the compiled program in fp64 must reproduce the oracle's
  substeps bitwise -- for the benchmark scene, a small slab, several chunk
  budgets and with/without the bank-aware schedule.  This proves the slot
  layout encodes the reference's per-vertex accumulation order
  (_kernels.pyx:260-352) independently of the GPU.
* Structural invariants: every (constraint, free endpoint) incidence has
  exactly one slot, slots are unique, warp-interleaved and in constraint order.
* The bank-aware schedule is a permutation of the constraint items and
  reduces phase-1 shared-memory conflicts.
"""

import os
import sys

import numpy as np
import pytest

import oracle as O
import program_interp as PI
from conftest import ROOT, build_slab_scene
from paper_2503_18616_b200 import scene as S


def _arrays(scene):
    return S.SceneArrays.from_loaded(*scene)


def _oracle_substeps(mesh, rest, cfg, x, v, gv, drag, att=None):
    xa, va = x[None].copy(), v[None].copy()
    a = att or dict(att_vertex=np.zeros(0), att_faces=np.zeros((0, 3)), att_is_face=np.zeros(0),
                    att_anchor=np.zeros((0, 3)), att_rest=np.zeros(0), att_k=np.zeros(0))
    O.run_substeps(xa, va, rest.inverse_mass, mesh.edges, rest.rest_length, cfg.k_s, mesh.tets, rest.rest_volume,
                   cfg.k_v, a["att_vertex"], a["att_faces"], a["att_is_face"], a["att_anchor"], a["att_rest"],
                   a["att_k"], np.array([gv]), drag[None], cfg.gravity, cfg.dt / cfg.substeps, cfg.substeps,
                   cfg.damping)
    return xa[0], va[0]


@pytest.mark.parametrize("opts", [dict(edge_gather=True), dict(edge_gather=True, max_chunk_slots=1024),
                                  dict(edge_gather=True, max_chunk_slots=200),
                                  dict(edge_gather=True, schedule_banks=False),
                                  dict(edge_gather=True, block_threads=64), dict(),
                                  dict(edge_gather=False), dict(edge_gather=False, max_chunk_slots=1024),
                                  dict(edge_gather=False, block_threads=64)])
def test_program_reproduces_oracle_bitwise(reach_scene, opts):
    mesh, rest, cfg = reach_scene
    blob, info = S.compile_program(_arrays(reach_scene), precision="fp64", **opts)
    prog = PI.Program(blob)
    rng = np.random.default_rng(1)
    free = np.flatnonzero(rest.inverse_mass > 0)
    x0 = mesh.positions_rest + rng.normal(0, 5e-4, mesh.positions_rest.shape) * (rest.inverse_mass > 0)[:, None]
    v0 = rng.normal(0, 1e-2, x0.shape) * (rest.inverse_mass > 0)[:, None]
    for gv in (-1, int(free[11]), int(free[-1])):
        drag = x0[free[11]] + np.array([0.001, 0.002, -0.0005])
        xa, va = _oracle_substeps(mesh, rest, cfg, x0, v0, gv, drag)
        xb, vb = x0.copy(), v0.copy()
        PI.run_substeps(prog, xb, vb, gv, drag, cfg.gravity, cfg.dt / cfg.substeps, cfg.substeps, cfg.damping,
                        cfg.k_s, cfg.k_v)
        assert np.array_equal(xa, xb) and np.array_equal(va, vb), (opts, gv)


@pytest.mark.parametrize("gather", [True, False])
def test_program_degenerate_constraints_counted_like_reference(gather):
    """Coincident edge endpoints and collapsed tets drop out of the counts (m = 0 guards)."""
    mesh, rest, cfg = build_slab_scene(3, 2, 2)
    blob, _ = S.compile_program(_arrays((mesh, rest, cfg)), precision="fp64", max_chunk_slots=64,
                                edge_gather=gather)
    prog = PI.Program(blob)
    x0 = mesh.positions_rest.copy()
    e = mesh.edges[5]
    x0[e[1]] = x0[e[0]]          # coincident edge
    t = mesh.tets[7]
    x0[t[3]] = x0[t[0]]          # collapsed tet shares that corner
    v0 = np.zeros_like(x0)
    xa, va = _oracle_substeps(mesh, rest, cfg, x0, v0, -1, np.zeros(3))
    xb, vb = x0.copy(), v0.copy()
    PI.run_substeps(prog, xb, vb, -1, np.zeros(3), cfg.gravity, cfg.dt / cfg.substeps, cfg.substeps, cfg.damping,
                    cfg.k_s, cfg.k_v)
    assert np.array_equal(xa, xb) and np.array_equal(va, vb)


def _edge_incidence(mesh, w):
    inc = np.zeros(mesh.vertex_count, int)
    for a, b in mesh.edges:
        if w[a] + w[b] > 0:
            inc[a] += w[a] > 0
            inc[b] += w[b] > 0
    return inc


@pytest.mark.parametrize("gather", [True, False])
def test_slot_structure(reach_scene, gather):
    mesh, rest, cfg = reach_scene
    blob, info = S.compile_program(_arrays(reach_scene), precision="fp32", edge_gather=gather)
    p = PI.Program(blob)
    H = p.h
    Vf = H["Vf"]
    w = rest.inverse_mass
    assert H["edge_gather"] == info["edge_gather"] == int(gather)
    # storage order: free first (sorted by gather cost, descending), then pinned
    assert np.all(w[p.s2o[:Vf]] > 0) and np.all(w[p.s2o[H["Vf_pad"]:][p.s2o[H["Vf_pad"]:] >= 0]] == 0)
    own = p.s2o[:H["Vown"]]
    assert np.array_equal(np.sort(own[own >= 0]), np.arange(mesh.vertex_count))
    # after Vown (fp32 gather programs): extra shared copies of the pinned vertices only, each pinned
    # vertex the same number of times, every copy of a vertex in a different bank
    copies = p.s2o[H["Vown"]:]
    pinned = np.flatnonzero(w == 0)
    if gather:
        assert len(copies) > 0 and np.all(w[copies[copies >= 0]] == 0)
        reps = np.bincount(copies[copies >= 0], minlength=mesh.vertex_count)[pinned]
        assert np.all(reps == reps[0]) and reps[0] >= 1
        for v in pinned:
            assert len(set(np.flatnonzero(p.s2o == v) % 32)) == reps[0] + 1
    else:
        assert np.all(copies < 0)
    # warps own vertices of similar cost: the groups of 32 are the cost-sorted order
    # (lanes inside a group may be permuted by the bank refinement); an owner-gathered edge
    # weighs three slots
    nulls = np.array([p.edge_nulls(q) for q in range(H["Vf_pad"])]) if gather else np.zeros(H["Vf_pad"], int)
    alln = np.array([p.edge_null_count(q) for q in range(H["Vf_pad"])]) if gather else np.zeros(H["Vf_pad"], int)
    sc = p.static_cnt[:Vf] - nulls[:Vf] + (2 * (p.evalence[:Vf] - alln[:Vf]) if gather else 0)
    ref = np.sort(sc)[::-1]
    for g in range(0, Vf, 32):
        assert sorted(sc[g:g + 32]) == sorted(ref[g:g + 32])
    expected = 0
    for kind, items, roles in ((0, p.edge_idx, 2), (2, p.tet_idx, 4)):
        slots = (p.edge_idx[:, 2:4] if kind == 0 else p.tet_slot)
        used = []
        for c in range(H["n_chunks"]):
            b, n, padded = p.chunks[c, 2 * kind], p.chunks[c, 2 * kind + 1], p.chunks[c, 6]
            if n == 0:
                continue
            sl = slots[b:b + n]
            idx = items[b:b + n, :roles]
            if kind == 2:                       # idle lanes of the bank schedule (all four slots -1)
                keep = (sl >= 0).any(axis=1)
                assert np.all(sl[~keep] == -1)
                sl, idx = sl[keep], idx[keep]
            real = sl >= 0
            assert np.all(real == (idx < H["Vf_pad"]))     # real slots exactly for free endpoints
            assert np.all(sl[real] < padded)                # pinned endpoints: no slot (-1)
            s = sl[real]
            assert len(np.unique(s)) == len(s)
            # slot k of lane l sits at region + 32k + l: bank = owner lane
            assert np.all(sl[real] % 32 == idx[real] % 32)
            used.append(len(s))
        expected += sum(used)
    n_inc = info["n_edge_incidences"] if gather else 0
    assert expected == info["n_slots_total"] == p.static_cnt.sum() - n_inc - nulls.sum()
    # per-vertex incidence count equals the reference's count of live constraints touching it
    inc = _edge_incidence(mesh, w)
    if gather:
        assert np.array_equal(p.evalence[:Vf] - alln[:Vf], inc[p.s2o[:Vf]]) and n_inc == inc.sum()
    for t in mesh.tets:
        inc[t] += w[t] > 0
    # static counts: live incidences, plus the null records of the gather rounds (each counted
    # degenerate every substep, so the applied count is unchanged)
    assert np.array_equal(p.static_cnt[:Vf] - nulls[:Vf], inc[p.s2o[:Vf]])


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_edge_gather_records(reach_scene, precision):
    """Owner-gathered edges: every free vertex lists exactly its live incident edges, in edge-index
    order (the reference's accumulation order), warp-interleaved, with the right rest lengths."""
    mesh, rest, cfg = reach_scene
    blob, info = S.compile_program(_arrays(reach_scene), precision=precision, edge_gather=True)
    p = PI.Program(blob)
    w = rest.inverse_mass
    assert p.h["einc_bytes"] == (4 if precision == "fp32" else 16)      # fp32: dictionary-coded rest lengths
    assert info["n_edge_items"] == 0            # no phase-1 edge items, no edge slots
    rt = np.float32 if precision == "fp32" else np.float64
    for pos in range(p.h["Vf"]):
        v = p.s2o[pos]
        nb, rl = p.edge_records(pos)
        want = [e for e, (a, b) in enumerate(mesh.edges) if (a == v or b == v) and w[a] + w[b] > 0]
        other = [int(b if a == v else a) for a, b in mesh.edges[want]]
        want_rl = rest.rest_length[want].astype(rt).astype(np.float64)
        if precision == "fp64":      # the reference's summation order: edge index
            assert np.array_equal(p.s2o[nb], other)
            assert np.array_equal(rl, want_rl)
        else:                        # fp32: same incidences, bank-scheduled order
            got = sorted(zip(p.s2o[nb].tolist(), rl.tolist()))
            assert got == sorted(zip(other, want_rl.tolist()))


def test_schedule_is_permutation_and_reduces_conflicts(reach_scene):
    arr = _arrays(reach_scene)
    b1, i1 = S.compile_program(arr, precision="fp32", schedule_banks=True, edge_gather=False)
    b0, i0 = S.compile_program(arr, precision="fp32", schedule_banks=False, edge_gather=False)
    p1, p0 = PI.Program(b1), PI.Program(b0)

    def constraints(p, idx, roles):
        vf = p.h["Vf_pad"]
        out = []
        live = (p.tet_slot >= 0).any(axis=1) if roles == 4 else np.ones(len(idx), bool)
        for row in idx[live][:, :roles]:
            if np.all(row >= vf):          # padding lane (pinned-only dummy edge)
                continue
            out.append(tuple(sorted(int(p.s2o[q]) for q in row)))
        return sorted(out)
    for idx1, idx0, roles in ((p1.edge_idx, p0.edge_idx, 2), (p1.tet_idx, p0.tet_idx, 4)):
        assert constraints(p1, idx1, roles) == constraints(p0, idx0, roles)
    assert i1["bank_conflicts_p1"] < i0["bank_conflicts_p1"]
    # the edge lists are conflict-free by construction (bipartite edge colouring)
    ex = 0
    for b in range(0, len(p1.edge_idx), 32):
        for r in range(2):
            ex += np.bincount(p1.edge_idx[b:b + 32, r] % 32, minlength=32).max() - 1
    assert ex == 0


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_compact_streams_encode_the_full_program(reach_scene, precision):
    """The 16-bit item streams the kernel reads for uniform-mass scenes carry exactly the full program:
    same positions and slots, same rest lengths, and edge weights recoverable from the pinned flags."""
    mesh, rest, cfg = reach_scene
    blob, info = S.compile_program(_arrays(reach_scene), precision=precision, edge_gather=False)
    p = PI.Program(blob)
    assert info["compact"] == 1 and p.h["compact"] == 1
    lo, hi = p.edge_c[:, 0] & 0xFFFF, p.edge_c[:, 0] >> 16
    assert np.array_equal(lo, p.edge_idx[:, 0]) and np.array_equal(hi, p.edge_idx[:, 1])
    for col, half in ((2, p.edge_c[:, 1] & 0xFFFF), (3, p.edge_c[:, 1] >> 16)):
        dec = half.astype(np.int64)
        dec[dec == 0xFFFF] = -1                                  # pinned endpoint: no slot
        assert np.array_equal(dec, p.edge_idx[:, col])
    if precision == "fp64":
        rl = p.edge_c[:, 2:4].copy().view(np.float64)[:, 0]
        vfp = p.h["Vf_pad"]
        wa = np.where(p.edge_idx[:, 0] < vfp, p.w_free, 0.0)
        wb = np.where(p.edge_idx[:, 1] < vfp, p.w_free, 0.0)
        live = (p.edge_idx[:, 0] < vfp) | (p.edge_idx[:, 1] < vfp)   # skip padding lanes
        assert np.array_equal(wa[live], p.edge_par[live, 1]) and np.array_equal(wb[live], p.edge_par[live, 2])
        assert np.array_equal((wa + wb)[live], p.edge_par[live, 3])
    else:
        rl = p.edge_c[:, 2].copy().view(np.float32).astype(np.float64)
    assert np.array_equal(rl, p.edge_par[:, 0])
    live = (p.tet_slot >= 0).any(axis=1)
    tc = p.tet_c[: len(p.tet_slot)]
    assert np.all(tc[~live, 2] == 0xFFFFFFFF) and np.all(tc[~live, 3] == 0xFFFFFFFF)   # idle lanes
    for k in range(4):
        assert np.array_equal(((tc[:, k // 2] >> (16 * (k % 2))) & 0xFFFF)[live], p.tet_idx[live, k])
        sl = ((tc[:, 2 + k // 2] >> (16 * (k % 2))) & 0xFFFF).astype(np.int64)
        sl[sl == 0xFFFF] = -1                                   # pinned corner: no slot
        assert np.array_equal(sl[live], p.tet_slot[live, k])


def test_nonuniform_mass_uses_full_streams(small_scene):
    mesh, rest, cfg = small_scene
    arr = _arrays(small_scene)
    arr.inverse_mass = arr.inverse_mass.copy()
    free = np.flatnonzero(arr.inverse_mass > 0)
    arr.inverse_mass[free[0]] *= 2.0
    _, info = S.compile_program(arr, precision="fp32")
    assert info["compact"] == 0


def test_compile_errors():
    mesh, rest, cfg = build_slab_scene()
    arr = _arrays((mesh, rest, cfg))
    arr.edges = arr.edges.copy()
    arr.edges[0, 0] = 10_000
    with pytest.raises(Exception, match="out of range"):
        S.compile_program(arr)


# ---------------------------------------------------------------------------
# cluster programs (large-mesh mode: one thread-block cluster of K CTAs per env)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("k", [2, 4, 16])
def test_cluster_program_reproduces_oracle_bitwise(reach_scene, k):
    """K parts, each owning a block of vertices and reading a halo refreshed by the owners every
    substep, reproduce the reference's substeps bit for bit (fp64 program, CPU interpreter)."""
    mesh, rest, cfg = reach_scene
    blob, info = S.compile_program(_arrays(reach_scene), precision="fp64", cluster_size=k)
    assert info["cluster_size"] == k
    parts = PI.cluster_parts(blob)
    assert len(parts) == k
    rng = np.random.default_rng(3)
    free = np.flatnonzero(rest.inverse_mass > 0)
    x0 = mesh.positions_rest + rng.normal(0, 5e-4, mesh.positions_rest.shape) * (rest.inverse_mass > 0)[:, None]
    v0 = rng.normal(0, 1e-2, x0.shape) * (rest.inverse_mass > 0)[:, None]
    for gv in (-1, int(free[17])):
        drag = x0[free[17]] + np.array([0.001, -0.002, 0.0005])
        xa, va = _oracle_substeps(mesh, rest, cfg, x0, v0, gv, drag)
        xb, vb = x0.copy(), v0.copy()
        PI.run_substeps_cluster(parts, xb, vb, gv, drag, cfg.gravity, cfg.dt / cfg.substeps, cfg.substeps,
                                cfg.damping, cfg.k_s, cfg.k_v)
        assert np.array_equal(xa, xb) and np.array_equal(va, vb), (k, gv)


def test_cluster_parts_partition_and_halo_sends(reach_scene):
    """Every vertex is owned by exactly one part; every halo copy is fed by exactly one send of its
    owner; every surface face is handled by exactly one part that holds its three vertices."""
    mesh, rest, cfg = reach_scene
    k = 4
    blob, info = S.compile_program(_arrays(reach_scene), precision="fp32", cluster_size=k)
    parts = PI.cluster_parts(blob)
    V = mesh.vertex_count
    owners = np.zeros(V, int)
    loc = []
    for r, p in enumerate(parts):
        H = p.h
        assert H["cluster_k"] == k and H["cluster_rank"] == r
        own = p.s2o[:H["Vown"]]
        owners[own[own >= 0]] += 1
        loc.append({int(o): q for q, o in enumerate(p.s2o) if o >= 0})
    assert np.all(owners == 1)
    # sends: (rank, pos) pairs of owned free vertex q must be exactly its halo copies elsewhere
    for r, p in enumerate(parts):
        H = p.h
        off = p.sec("SEND_OFF", np.int32, H["Vf_pad"] + 1)
        snd = p.sec("SEND", np.int32, int(off[-1]))
        for q in range(H["Vf"]):
            o = int(p.s2o[q])
            got = sorted((int(s) >> 20, int(s) & 0xFFFFF) for s in snd[off[q]:off[q + 1]])
            want = sorted((rr, loc[rr][o]) for rr in range(k) if rr != r and o in loc[rr])
            assert got == want
    # faces: a partition of the surface, ascending global ids per part, vertices local
    gids = []
    for r, p in enumerate(parts):
        g = p.sec("FACE_GID", np.int32, p.h["F"])
        assert np.all(np.diff(g) > 0)
        gids.extend(g.tolist())
        for i, f in enumerate(g):
            assert all(int(vv) in loc[r] for vv in mesh.surface_faces[f])
    assert sorted(gids) == list(range(len(mesh.surface_faces)))
    # equal shared-memory layout across ranks (DSMEM addresses coincide)
    assert len({(p.h["Vstore"], p.h["slot_capacity"], p.h["B"]) for p in parts}) == 1


def test_large_presets_compile_to_clusters():
    """Table II-right meshes: the 52359-tet slab does not fit one CTA, and compiles to a cluster."""
    import tempfile
    from paper_2503_18616_b200.mesh import load_scene, make_slab_scene
    d = tempfile.mkdtemp()
    sc = load_scene(make_slab_scene(d, tets=52359))
    blob, info = S.compile_program(_arrays(sc), precision="fp32")
    assert 2 <= info["cluster_size"] <= 16
    assert info["n_free"] == int((sc[1].inverse_mass > 0).sum())
    with pytest.raises(Exception, match="too large|shared memory"):
        S.compile_program(_arrays(sc), precision="fp32", cluster_size=1)


def test_dictionary_coded_streams(reach_scene):
    """fp32 byte-offset programs of a structured slab: rest lengths and 6 V0 take two fp32 values
    each, so the edge records shrink to 4 bytes and the tet stream carries a 6 V0 index in the
    spare top bits of its position offsets -- decoding them gives back exactly the full arrays."""
    blob, info = S.compile_program(_arrays(reach_scene), precision="fp32")
    p = PI.Program(blob)
    assert p.h["einc_bytes"] == 4 and p.h["rvdict"] == 1
    live = (p.tet_slot >= 0).any(axis=1)
    n_rv = len(np.unique(p.tet_rv[live].astype(np.float32)))
    rvtab = p.sec("RVTAB", np.float32, n_rv)
    q = p.tet_c[: len(p.tet_rv)]
    ri = ((q[:, 0] >> 14) & 3) | ((q[:, 0] >> 28) & 12) | ((q[:, 1] >> 10) & 48) | ((q[:, 1] >> 24) & 192)
    assert np.array_equal(rvtab[ri[live]].astype(np.float64), p.tet_rv[live])
    offs = np.stack([q[:, 0] & 0x3FFF, (q[:, 0] >> 16) & 0x3FFF, q[:, 1] & 0x3FFF, (q[:, 1] >> 16) & 0x3FFF], 1)
    assert np.array_equal(offs[live], 12 * p.tet_idx[live])
    # narrow layout: positions first, slot fields are byte offsets from the same base (+ 12 Vstore)
    assert p.h["narrow"] == 1
    sl = np.stack([q[:, 2] & 0xFFFF, q[:, 2] >> 16, q[:, 3] & 0xFFFF, q[:, 3] >> 16], 1).astype(np.int64)
    want = np.where(p.tet_slot >= 0, 12 * (p.h["Vstore"] + p.tet_slot), 0xFFFF)
    assert np.array_equal(sl[live], want[live])


def test_latency_cluster_policy():
    """layout=None: clusters only for meshes past ~768 vertices and only while envs x CTAs fit the SMs
    (measured crossover, profiles/r01r/mesh_scaling.json)."""
    from paper_2503_18616_b200.solver import latency_cluster_size as k
    assert k(392, 1, 148) == 0 and k(504, 1, 148) == 0        # one CTA beats any cluster
    assert k(845, 1, 148) == 4 and k(2527, 1, 148) == 8 and k(12180, 1, 148) == 16
    assert k(12180, 16, 148) == 8 and k(12180, 4096, 148) == 0   # throughput: the compiler's smallest fit
    assert k(2527, 74, 148) == 2 and k(2527, 75, 148) == 0


def test_latency_block_policy():
    """Small fp32 batches (<= one env per SM) get ~1.3 threads per free vertex; large batches, fp64
    and already-wide meshes keep the compiler's default."""
    from paper_2503_18616_b200.solver import latency_block_threads as b
    assert b(294, 1, 148, "fp32") == 384 and b(294, 148, 148, "fp32") == 384
    assert b(294, 149, 148, "fp32") == 0 and b(294, 1, 148, "fp64") == 0
    assert b(500, 1, 148, "fp32") == 0           # 512 cap: no wider than the default 512


def test_fast_program_is_bank_conflict_free(reach_scene):
    """The fp32 production program (pinned copies, packed tet batches, coloured gather rounds,
    DESIGN.md §2.5): replaying its shared-memory accesses per warp instruction
    (tools/bank_model.py) every phase-1 / phase-2 access is served in its ideal number of
    wavefronts -- the compiler's conflict-free construction, checked on the blob the kernel reads."""
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import bank_model
    blob, info = S.compile_program(_arrays(reach_scene), precision="fp32")
    assert info["bank_conflicts_p1"] == 0
    out = bank_model.model(PI.Program(blob))
    for cat, (ideal, modelled) in out.items():
        assert modelled == ideal, (cat, ideal, modelled)
    # every tet appears exactly once, and the rest volume carries the sign of its (permuted) corner
    # order: at rest the stored 6 V0 equals the signed 6 V of the corners in program order
    mesh, rest, _ = reach_scene
    p = PI.Program(blob)
    live = (p.tet_slot >= 0).any(axis=1)
    idx, rv = p.tet_idx[live], p.tet_rv[live]
    verts = p.s2o[idx]                                      # storage (or pinned-copy) position -> vertex
    assert sorted(map(tuple, np.sort(verts, axis=1))) == sorted(map(tuple, np.sort(mesh.tets, axis=1)))
    X = mesh.positions_rest
    a, b, c, d = (X[verts[:, k]] for k in range(4))
    six_v = np.einsum("ij,ij->i", np.cross(b - a, c - a), d - a)
    assert np.allclose(rv, six_v, rtol=1e-5, atol=1e-12)
    # the kernel reads 6 V0 through the dictionary index in the stream's spare bits
    tab = p.sec("RVTAB", np.float32, p.h["n_rvtab"]).astype(np.float64)
    q = p.tet_c[live]
    ri = ((q[:, 0] >> 14) & 3) | ((q[:, 0] >> 28) & 12) | ((q[:, 1] >> 10) & 48) | ((q[:, 1] >> 24) & 192)
    assert np.array_equal(tab[ri], rv)


@pytest.mark.parametrize("layout", [{}, {"precision": "fp64"}, {"cluster_size": 2}])
def test_compiler_is_deterministic(layout):
    """The same scene and options compile to the same bytes every time (the searches use fixed
    seeds) -- the program cache and every parity claim on a cached program rely on it."""
    arrays = _arrays(build_slab_scene(nx=5, ny=3, nz=2))
    o = S.layout_opts(**layout)
    b1, i1 = S._compile_raw(arrays, o)
    b2, i2 = S._compile_raw(arrays, o)
    assert np.array_equal(b1, b2) and bytes(i1) == bytes(i2)
