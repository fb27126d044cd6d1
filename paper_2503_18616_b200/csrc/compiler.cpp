// compiler.cpp -- host scene compiler: scene arrays -> TsProgram blob.
//
// This is the B200 replacement of Simulation.__init__'s array packing
// (solver.py:280-305) plus the reference's implicit "summation order"
// contract (_kernels.pyx:260-352): it lays constraints out so the sm_100a
// kernel can run them as a deterministic gather with no atomics on floats,
// in exactly the reference's per-vertex accumulation order.
//
//  * vertex storage order: free vertices sorted by incidence count so warps
//    are load balanced in the per-vertex gather; pinned vertices last;
//  * constraint chunks: contiguous constraint-index ranges of one kind
//    (edges, attachments, tets) sized to a shared-memory slot budget;
//  * slots: one per (constraint, free endpoint), laid out warp-interleaved
//    (slot k of lane l at region + 32k + l) so the owner warp's reads are
//    bank-conflict free and coalesced;
//  * phase-1 schedule: items reordered into 32-wide batches whose lanes hit
//    distinct banks for every role (the role of a graph colouring: a batch
//    is a colour class of the "same bank" conflict graph); results do not
//    depend on this order, only shared-memory wavefronts do.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/tissuesim_b200.h"
#include "program.h"

namespace ts {

namespace {

struct Item {
    int kind;          // TsChunkKind
    int index;         // constraint index in its kind
    int nroles;
    int pos[4];        // storage positions of the roles
    int slot[4];       // slot id inside the chunk (-1 pinned endpoint)
};

inline int roundup(int x, int m) { return (x + m - 1) / m * m; }

template <typename T>
void put(std::vector<uint8_t> &blob, int64_t off, const std::vector<T> &v) {
    if (!v.empty()) std::memcpy(blob.data() + off, v.data(), v.size() * sizeof(T));
}

// Swap-based local search over a schedule: lanes are grouped into sub-batches
// of `bank_mod` items (a warp for 32-bit data, a half-warp for 64-bit); the
// cost of a sub-batch is, per role, (max items on one bank - 1) = the extra
// shared-memory wavefronts that role's loads and stores pay.  Deterministic
// (fixed-seed xorshift), first-improvement, sideways moves allowed.
void local_search(std::vector<Item> &s, int bank_mod) {
    const int n = (int)s.size();
    const int nsb = (n + bank_mod - 1) / bank_mod;
    const int R4 = 4;
    std::vector<int> cnt((size_t)nsb * R4 * bank_mod, 0);
    auto C = [&](int sb, int r, int b) -> int & { return cnt[((size_t)sb * R4 + r) * bank_mod + b]; };
    for (int i = 0; i < n; ++i)
        for (int r = 0; r < s[i].nroles; ++r) C(i / bank_mod, r, s[i].pos[r] % bank_mod)++;
    auto sb_cost = [&](int sb) {
        int c = 0;
        for (int r = 0; r < R4; ++r) {
            int m = 0;
            for (int b = 0; b < bank_mod; ++b) m = std::max(m, C(sb, r, b));
            if (m > 1) c += m - 1;
        }
        return c;
    };
    std::vector<int> cost(nsb);
    int total = 0;
    for (int sb = 0; sb < nsb; ++sb) { cost[sb] = sb_cost(sb); total += cost[sb]; }
    uint64_t rng = 0x9E3779B97F4A7C15ull;
    auto next = [&]() { rng ^= rng << 13; rng ^= rng >> 7; rng ^= rng << 17; return rng; };
    const long iters = std::min<long>(400000L, 200L * n);
    for (long it = 0; it < iters && total > 0; ++it) {
        // pick a position in a costly sub-batch and a random partner elsewhere
        int i = (int)(next() % n), j = (int)(next() % n);
        int si = i / bank_mod, sj = j / bank_mod;
        if (si == sj || (cost[si] == 0 && cost[sj] == 0)) continue;
        auto move = [&](int k, int from, int to) {
            for (int r = 0; r < s[k].nroles; ++r) { C(from, r, s[k].pos[r] % bank_mod)--; C(to, r, s[k].pos[r] % bank_mod)++; }
        };
        move(i, si, sj);
        move(j, sj, si);
        const int ci = sb_cost(si), cj = sb_cost(sj);
        const int delta = ci + cj - cost[si] - cost[sj];
        if (delta <= 0) {
            std::swap(s[i], s[j]);
            total += delta;
            cost[si] = ci; cost[sj] = cj;
        } else {
            move(i, sj, si);
            move(j, si, sj);
        }
    }
}

// Greedy bank-aware batching + local search.  Returns items in schedule
// order and the number of extra shared-memory wavefronts the residual
// conflicts cost per pass over the chunk.
std::vector<Item> schedule_items(std::vector<Item> items, int bank_mod, int batch, bool enable,
                                 int *extra_wavefronts) {
    *extra_wavefronts = 0;
    if (!enable || items.size() <= 1) {
        // conflicts of the identity order, for reporting
    }
    std::vector<Item> out;
    out.reserve(items.size());
    std::vector<char> taken(items.size(), 0);
    size_t first_free = 0;
    const size_t window = 8192;
    auto conflicts_of = [&](const std::vector<int> &idx) {
        int extra = 0;
        if (idx.empty()) return 0;
        int nroles = 0;
        for (int i : idx) nroles = std::max(nroles, items[i].nroles);
        for (int r = 0; r < nroles; ++r) {
            // lanes are split into sub-batches of `bank_mod` (half-warps for 64-bit)
            for (size_t b0 = 0; b0 < idx.size(); b0 += bank_mod) {
                std::vector<int> cnt(bank_mod, 0);
                int worst = 0;
                for (size_t k = b0; k < std::min(idx.size(), b0 + bank_mod); ++k) {
                    const Item &it = items[idx[k]];
                    if (r >= it.nroles) continue;
                    int c = ++cnt[it.pos[r] % bank_mod];
                    worst = std::max(worst, c);
                }
                if (worst > 1) extra += worst - 1;
            }
        }
        return extra;
    };
    size_t done = 0;
    while (done < items.size()) {
        std::vector<int> pick;
        std::vector<uint64_t> used(4, 0);  // per role, bank bitmask (bank_mod <= 32)
        while (first_free < items.size() && taken[first_free]) ++first_free;
        if (enable) {
            size_t scanned = 0;
            for (size_t i = first_free; i < items.size() && (int)pick.size() < batch && scanned < window; ++i) {
                if (taken[i]) continue;
                ++scanned;
                const Item &it = items[i];
                // the sub-batch (half-warp for 64-bit data) this item would land in
                uint64_t ok = 1;
                for (int r = 0; r < it.nroles && ok; ++r)
                    if (used[r] >> (it.pos[r] % bank_mod) & 1ull) ok = 0;
                if (!ok) continue;
                pick.push_back((int)i);
                taken[i] = 1;
                for (int r = 0; r < it.nroles; ++r) used[r] |= 1ull << (it.pos[r] % bank_mod);
                if ((int)pick.size() % bank_mod == 0) std::fill(used.begin(), used.end(), 0);
            }
        }
        // fill the rest of the batch in index order
        for (size_t i = first_free; i < items.size() && (int)pick.size() < batch; ++i) {
            if (taken[i]) continue;
            pick.push_back((int)i);
            taken[i] = 1;
        }
        for (int i : pick) out.push_back(items[i]);
        done += pick.size();
    }
    if (enable && out.size() > (size_t)bank_mod) local_search(out, bank_mod);
    for (size_t b0 = 0; b0 < out.size(); b0 += batch) {
        std::vector<int> idx;
        for (size_t k = b0; k < std::min(out.size(), b0 + batch); ++k) idx.push_back((int)k);
        items.swap(out);
        *extra_wavefronts += conflicts_of(idx);
        items.swap(out);
    }
    return out;
}

template <typename Real>
struct Real4T { Real x, y, z, w; };

}  // namespace

int compile_program(const ts_scene_desc &d, const ts_layout_opts &o, std::vector<uint8_t> &blob,
                    ts_layout_info &info, std::string &err) {
    const int V = d.n_vert, E = d.n_edge, T = d.n_tet, F = d.n_face, A = d.n_att;
    const int prec = o.precision;
    if (prec != TS_F32 && prec != TS_F64) { err = "precision must be TS_F32 or TS_F64"; return TS_ERR_INVALID; }
    const int R = prec == TS_F64 ? 8 : 4;
    if (V < 0 || E < 0 || T < 0 || F < 0 || A < 0) { err = "negative counts"; return TS_ERR_INVALID; }
    if (V > 0 && (!d.positions_rest || !d.inverse_mass)) { err = "missing vertex arrays"; return TS_ERR_INVALID; }
    auto bad_vid = [&](int v) { return v < 0 || v >= V; };
    for (int i = 0; i < 2 * E; ++i) if (bad_vid(d.edges[i])) { err = "edge vertex index out of range"; return TS_ERR_INVALID; }
    for (int i = 0; i < 4 * T; ++i) if (bad_vid(d.tets[i])) { err = "tet vertex index out of range"; return TS_ERR_INVALID; }
    for (int i = 0; i < 3 * F; ++i) if (bad_vid(d.faces[i])) { err = "face vertex index out of range"; return TS_ERR_INVALID; }
    for (int i = 0; i < A; ++i) {
        if (bad_vid(d.att_vertex[i])) { err = "attachment vertex out of range"; return TS_ERR_INVALID; }
        if (d.att_is_face[i])
            for (int k = 0; k < 3; ++k) if (bad_vid(d.att_faces[3 * i + k])) { err = "attachment face vertex out of range"; return TS_ERR_INVALID; }
    }
    const double *w = d.inverse_mass;
    auto is_free = [&](int v) { return w[v] > 0.0; };

    // ---- live constraints and per-vertex incidence counts ---------------
    std::vector<int> inc(V, 0);
    std::vector<char> edge_live(E), att_live(A), tet_live(T);
    for (int e = 0; e < E; ++e) {
        int a = d.edges[2 * e], b = d.edges[2 * e + 1];
        edge_live[e] = (w[a] + w[b]) > 0.0;  // _kernels.pyx:111 skips wsum <= 0
        if (edge_live[e]) { inc[a] += is_free(a); inc[b] += is_free(b); }
    }
    std::vector<double> att_wv(A), att_wc(A);
    for (int i = 0; i < A; ++i) {
        int v = d.att_vertex[i];
        const int *f = d.att_faces + 3 * i;
        att_wv[i] = w[v];
        att_wc[i] = d.att_is_face[i] ? (w[f[0]] + w[f[1]] + w[f[2]]) / 3.0 : 0.0;
        att_live[i] = (att_wv[i] + att_wc[i]) > 0.0;  // _kernels.pyx:309
        if (!att_live[i]) continue;
        inc[v] += is_free(v);
        if (d.att_is_face[i]) for (int k = 0; k < 3; ++k) inc[f[k]] += is_free(f[k]);
    }
    for (int t = 0; t < T; ++t) {
        const int *q = d.tets + 4 * t;
        bool any = false;
        for (int k = 0; k < 4; ++k) any |= is_free(q[k]);
        tet_live[t] = any;  // all-pinned tets only touch pinned accumulators
        if (any) for (int k = 0; k < 4; ++k) inc[q[k]] += is_free(q[k]);
    }

    // ---- storage order -------------------------------------------------
    std::vector<int> free_v, pinned_v;
    for (int v = 0; v < V; ++v) (is_free(v) ? free_v : pinned_v).push_back(v);
    std::stable_sort(free_v.begin(), free_v.end(), [&](int a, int b) { return inc[a] > inc[b]; });
    const int Vf = (int)free_v.size();
    const int Vf_pad = roundup(Vf, 32);
    const int Vstore = Vf_pad + roundup((int)pinned_v.size(), 32);
    std::vector<int> s2o(Vstore, -1), o2s(V, -1);
    for (int i = 0; i < Vf; ++i) { s2o[i] = free_v[i]; o2s[free_v[i]] = i; }
    for (size_t i = 0; i < pinned_v.size(); ++i) { s2o[Vf_pad + i] = pinned_v[i]; o2s[pinned_v[i]] = Vf_pad + (int)i; }

    // fp32: one thread per free vertex (3 CTAs/SM fit); fp64 runs 1 CTA/SM (shared memory), so it
    // takes 1.5x the threads to widen phase 1 (measured on B200: 3.81 vs 4.30 ms at 4096 envs)
    int B = o.block_threads > 0 ? o.block_threads
                                : std::min(512, std::max(64, R == 8 ? roundup(Vf_pad * 3 / 2, 32) : Vf_pad));
    if (B % 32 != 0 || B < 32 || B > 512) { err = "block_threads must be a multiple of 32 in [32, 512]"; return TS_ERR_INVALID; }
    const int VPT = std::max(1, (Vf_pad + B - 1) / B);
    if (VPT > 8) { err = "mesh too large for one CTA per environment (more than 8 vertices per thread)"; return TS_ERR_UNSUPPORTED; }
    const int G = Vf_pad / 32;

    // ---- items per kind (constraint index order) -----------------------
    auto P = [&](int v) { return o2s[v]; };
    std::vector<Item> kinds[3];
    for (int e = 0; e < E; ++e) if (edge_live[e]) {
        Item it{}; it.kind = TS_CHUNK_EDGE; it.index = e; it.nroles = 2;
        it.pos[0] = P(d.edges[2 * e]); it.pos[1] = P(d.edges[2 * e + 1]);
        kinds[0].push_back(it);
    }
    for (int i = 0; i < A; ++i) if (att_live[i]) {
        Item it{}; it.kind = TS_CHUNK_ATT; it.index = i;
        it.pos[0] = P(d.att_vertex[i]);
        if (d.att_is_face[i]) { it.nroles = 4; for (int k = 0; k < 3; ++k) it.pos[1 + k] = P(d.att_faces[3 * i + k]); }
        else it.nroles = 1;
        kinds[1].push_back(it);
    }
    for (int t = 0; t < T; ++t) if (tet_live[t]) {
        Item it{}; it.kind = TS_CHUNK_TET; it.index = t; it.nroles = 4;
        for (int k = 0; k < 4; ++k) it.pos[k] = P(d.tets[4 * t + k]);
        kinds[2].push_back(it);
    }

    // ---- chunking by slot budget ---------------------------------------
    // The reference's per-vertex accumulation order is the constraint sequence
    // [live edges..., grasp, live attachments..., live tets...].  Chunks are
    // contiguous ranges of that sequence (kinds may mix); the grasp is spliced
    // into the chunk where the edges end, after each vertex's edge slots.
    std::vector<Item> seq;
    for (int k = 0; k < 3; ++k) seq.insert(seq.end(), kinds[k].begin(), kinds[k].end());
    const int budget = o.max_chunk_slots > 0 ? o.max_chunk_slots : (1 << 30);
    struct ChunkBuild { std::vector<Item> items; std::vector<int> val; std::vector<int> kmax; int padded; };
    std::vector<ChunkBuild> chunks;
    {
        size_t i = 0;
        while (i < seq.size()) {
            ChunkBuild c;
            c.val.assign(Vf_pad, 0); c.kmax.assign(G, 0); c.padded = 0;
            while (i < seq.size()) {
                const Item &it = seq[i];
                // default layout: a new chunk at every kind change (measured fastest on B200 for
                // reach_1170: 2 chunks at 3 CTAs/SM beat 1 mixed chunk at 2 CTAs/SM)
                if (o.max_chunk_slots == 0 && !c.items.empty() && c.items.back().kind != it.kind) break;
                int grow = 0;
                std::vector<int> touched_g;
                for (int r = 0; r < it.nroles; ++r) if (it.pos[r] < Vf_pad) c.val[it.pos[r]]++;
                for (int r = 0; r < it.nroles; ++r) {
                    const int p = it.pos[r];
                    if (p >= Vf_pad) continue;
                    const int g = p / 32;
                    if (c.val[p] > c.kmax[g]) { grow += 32 * (c.val[p] - c.kmax[g]); c.kmax[g] = c.val[p]; touched_g.push_back(g); }
                }
                if (!c.items.empty() && c.padded + grow > budget) {
                    for (int r = 0; r < it.nroles; ++r) if (it.pos[r] < Vf_pad) c.val[it.pos[r]]--;
                    for (int g : touched_g) {
                        int mx = 0; for (int q = 32 * g; q < 32 * g + 32; ++q) mx = std::max(mx, c.val[q]);
                        c.kmax[g] = mx;
                    }
                    break;
                }
                c.padded += grow;
                c.items.push_back(it);
                ++i;
            }
            chunks.push_back(std::move(c));
        }
    }
    const int n_chunks = (int)chunks.size();
    // grasp chunk: the chunk holding the first non-edge item (n_chunks if there is none)
    int grasp_chunk = n_chunks;
    {
        const size_t n_edges = kinds[0].size();
        if (n_edges < seq.size()) {
            size_t pos = 0;
            for (int c = 0; c < n_chunks; ++c) {
                if (n_edges < pos + chunks[c].items.size()) { grasp_chunk = c; break; }
                pos += chunks[c].items.size();
            }
        }
    }

    // ---- slot assignment (reference per-vertex order) -------------------
    std::vector<int32_t> region((size_t)n_chunks * G), valence((size_t)n_chunks * Vf_pad), static_cnt(Vf_pad, 0);
    std::vector<int32_t> gsplit(Vf_pad, 0);
    int slot_cap = 0, n_slots_total = 0;
    for (int c = 0; c < n_chunks; ++c) {
        ChunkBuild &cb = chunks[c];
        int base = 0;
        for (int g = 0; g < G; ++g) { region[(size_t)c * G + g] = base; base += 32 * cb.kmax[g]; }
        cb.padded = base;
        // 32 "trash" slots after the regions: edge / tet endpoints that are pinned store there
        // unconditionally (bank = p % 32, same as their position reads), nobody reads them back
        const int trash = base;
        slot_cap = std::max(slot_cap, base + 32);
        std::vector<int> k_next(Vf_pad, 0);
        for (Item &it : cb.items) {  // items are in sequence order here
            for (int r = 0; r < it.nroles; ++r) {
                int p = it.pos[r];
                if (p >= Vf_pad) { it.slot[r] = it.kind == TS_CHUNK_ATT ? -1 : trash + (p % 32); continue; }
                it.slot[r] = region[(size_t)c * G + p / 32] + 32 * k_next[p] + (p % 32);
                k_next[p]++;
                if (c == grasp_chunk && it.kind == TS_CHUNK_EDGE) gsplit[p] = k_next[p];
            }
        }
        for (int p = 0; p < Vf_pad; ++p) {
            valence[(size_t)c * Vf_pad + p] = k_next[p];
            static_cnt[p] += k_next[p];
            n_slots_total += k_next[p];
        }
    }
    // contact records reuse the slot buffer: 3F records x 7 reals <= 3 arrays x S reals
    slot_cap = std::max(slot_cap, 7 * F);
    slot_cap = roundup(std::max(slot_cap, 32), 32);

    // ---- phase-1 schedule (per chunk, per kind) ----------------------------
    const bool sched = o.schedule_banks >= 0;
    const int bank_mod = (R == 8) ? 16 : 32;
    int total_conf = 0;
    std::vector<TsChunk> chunk_rec(n_chunks);
    std::vector<Item> all_items[3];
    for (int c = 0; c < n_chunks; ++c) {
        ChunkBuild &cb = chunks[c];
        TsChunk &r = chunk_rec[c];
        std::memset(&r, 0, sizeof(r));
        int begin[3], count[3];
        for (int k = 0; k < 3; ++k) {
            const int kind = k == 0 ? TS_CHUNK_EDGE : (k == 1 ? TS_CHUNK_ATT : TS_CHUNK_TET);
            std::vector<Item> part;
            for (const Item &it : cb.items) if (it.kind == kind) part.push_back(it);
            int conf = 0;
            std::vector<Item> s = schedule_items(part, bank_mod, 32, sched && kind != TS_CHUNK_ATT, &conf);
            r.conflicts += conf;
            begin[k] = (int)all_items[k].size();
            count[k] = (int)s.size();
            all_items[k].insert(all_items[k].end(), s.begin(), s.end());
        }
        total_conf += r.conflicts;
        r.edge_begin = begin[0]; r.edge_count = count[0];
        r.att_begin = begin[1]; r.att_count = count[1];
        r.tet_begin = begin[2]; r.tet_count = count[2];
        r.slot_count = cb.padded;
        r.region_off = c * G;
        r.val_off = c * Vf_pad;
    }

    // ---- emit --------------------------------------------------------------
    const int nE = (int)all_items[0].size(), nA = (int)all_items[1].size(), nT = (int)all_items[2].size();
    std::vector<int32_t> edge_idx(4 * (size_t)nE), tet_idx(4 * (size_t)nT), tet_slot(4 * (size_t)nT);
    std::vector<int32_t> att_idx(4 * (size_t)nA), att_slot(4 * (size_t)nA);
    std::vector<double> edge_par(4 * (size_t)nE), tet_rv(nT), att_par(4 * (size_t)nA), att_anc(4 * (size_t)nA);
    for (int i = 0; i < nE; ++i) {
        const Item &it = all_items[0][i];
        int a = d.edges[2 * it.index], b = d.edges[2 * it.index + 1];
        edge_idx[4 * i + 0] = it.pos[0]; edge_idx[4 * i + 1] = it.pos[1];
        edge_idx[4 * i + 2] = it.slot[0]; edge_idx[4 * i + 3] = it.slot[1];
        edge_par[4 * i + 0] = d.rest_length[it.index];
        if (R == 8) {   // exact build: the reference's operands
            edge_par[4 * i + 1] = w[a]; edge_par[4 * i + 2] = w[b]; edge_par[4 * i + 3] = w[a] + w[b];
        } else {        // fp32 build: ca = -(ks wa / wsum)(1 - rl/dist), cb = (ks wb / wsum)(1 - rl/dist)
            const double wsum = w[a] + w[b];
            edge_par[4 * i + 1] = d.k_s * w[a] / wsum; edge_par[4 * i + 2] = d.k_s * w[b] / wsum;
            edge_par[4 * i + 3] = 0.0;
        }
    }
    for (int i = 0; i < nT; ++i) {
        const Item &it = all_items[2][i];
        for (int k = 0; k < 4; ++k) { tet_idx[4 * i + k] = it.pos[k]; tet_slot[4 * i + k] = it.slot[k]; }
        // fp32 build works with unscaled cross products G = 6 grad: it needs 6 V0
        tet_rv[i] = R == 8 ? d.rest_volume[it.index] : 6.0 * d.rest_volume[it.index];
    }
    for (int i = 0; i < nA; ++i) {
        const Item &it = all_items[1][i];
        int t = it.index;
        att_idx[4 * i + 0] = it.pos[0];
        att_slot[4 * i + 0] = it.slot[0];
        for (int k = 1; k < 4; ++k) {
            att_idx[4 * i + k] = it.nroles == 4 ? it.pos[k] : it.pos[0];
            att_slot[4 * i + k] = it.nroles == 4 ? it.slot[k] : -1;
        }
        att_par[4 * i + 0] = d.att_rest[t]; att_par[4 * i + 1] = d.att_k[t];
        att_par[4 * i + 2] = att_wv[t]; att_par[4 * i + 3] = att_wc[t];
        const double *an = d.att_anchor + 3 * t;
        att_anc[4 * i + 0] = d.att_is_face[t] ? 0.0 : an[0];
        att_anc[4 * i + 1] = d.att_is_face[t] ? 0.0 : an[1];
        att_anc[4 * i + 2] = d.att_is_face[t] ? 0.0 : an[2];
        att_anc[4 * i + 3] = d.att_is_face[t] ? 1.0 : 0.0;
    }
    std::vector<double> wst(Vstore, 0.0);
    for (int p = 0; p < Vstore; ++p) if (s2o[p] >= 0) wst[p] = w[s2o[p]];
    std::vector<int32_t> faces_s(3 * (size_t)F), faces_o(3 * (size_t)F);
    for (int i = 0; i < 3 * F; ++i) { faces_o[i] = d.faces[i]; faces_s[i] = o2s[d.faces[i]]; }
    std::vector<double> rest(3 * (size_t)V);
    for (int i = 0; i < 3 * V; ++i) rest[i] = d.positions_rest[i];

    // ---- compact 16-bit item streams ---------------------------------------
    // Every mesh built by load_scene has one inverse mass for all free vertices
    // (mesh.py:217: uniform mass), so an edge needs only its rest length: the
    // per-endpoint weights follow from which endpoints are pinned.
    double w_free = 0.0;
    bool uniform = true;
    for (int v = 0; v < V; ++v)
        if (is_free(v)) {
            if (w_free == 0.0) w_free = w[v];
            else if (w[v] != w_free) uniform = false;
        }
    const bool compact = o.compact >= 0 && uniform && Vstore <= 65535 && slot_cap <= 65535;
    std::vector<uint32_t> edge_c(compact ? 4 * (size_t)nE : 0), tet_c(compact ? 4 * (size_t)nT : 0);
    if (compact) {
        auto pk = [](int lo, int hi) { return (uint32_t)(lo & 0xffff) | ((uint32_t)(hi & 0xffff) << 16); };
        for (int i = 0; i < nE; ++i) {
            edge_c[4 * i + 0] = pk(edge_idx[4 * i + 0], edge_idx[4 * i + 1]);
            edge_c[4 * i + 1] = pk(edge_idx[4 * i + 2], edge_idx[4 * i + 3]);
            const double rl = edge_par[4 * i + 0];
            if (R == 8) { std::memcpy(&edge_c[4 * i + 2], &rl, 8); }
            else { const float f = (float)rl; std::memcpy(&edge_c[4 * i + 2], &f, 4); edge_c[4 * i + 3] = 0; }
        }
        for (int i = 0; i < nT; ++i) {
            tet_c[4 * i + 0] = pk(tet_idx[4 * i + 0], tet_idx[4 * i + 1]);
            tet_c[4 * i + 1] = pk(tet_idx[4 * i + 2], tet_idx[4 * i + 3]);
            tet_c[4 * i + 2] = pk(tet_slot[4 * i + 0], tet_slot[4 * i + 1]);
            tet_c[4 * i + 3] = pk(tet_slot[4 * i + 2], tet_slot[4 * i + 3]);
        }
    }

    // sizes (bytes) per section
    int64_t sz[TS_SEC_COUNT];
    sz[TS_SEC_CHUNK] = (int64_t)n_chunks * sizeof(TsChunk);
    sz[TS_SEC_EDGE_IDX] = 16LL * nE;
    sz[TS_SEC_EDGE_PAR] = 4LL * R * nE;
    sz[TS_SEC_TET_IDX] = 16LL * nT;
    sz[TS_SEC_TET_SLOT] = 16LL * nT;
    sz[TS_SEC_TET_RV] = (int64_t)R * nT;
    sz[TS_SEC_ATT_IDX] = 16LL * nA;
    sz[TS_SEC_ATT_SLOT] = 16LL * nA;
    sz[TS_SEC_ATT_PAR] = 4LL * R * nA;
    sz[TS_SEC_ATT_ANCHOR] = 4LL * R * nA;
    sz[TS_SEC_REGION] = 4LL * region.size();
    sz[TS_SEC_VALENCE] = 4LL * valence.size();
    sz[TS_SEC_STATIC_CNT] = 4LL * Vf_pad;
    sz[TS_SEC_S2O] = 4LL * Vstore;
    sz[TS_SEC_O2S] = 4LL * V;
    sz[TS_SEC_W] = (int64_t)R * Vstore;
    sz[TS_SEC_FACES] = 12LL * F;
    sz[TS_SEC_FACES_ORIG] = 12LL * F;
    sz[TS_SEC_REST] = 3LL * R * V;
    sz[TS_SEC_GSPLIT] = 4LL * Vf_pad;
    sz[TS_SEC_EDGE_C] = 4LL * edge_c.size();
    sz[TS_SEC_TET_C] = 4LL * tet_c.size();
    TsProgHeader hdr{};
    hdr.compact = compact ? 1 : 0;
    hdr.w_free = w_free;
    hdr.magic = TS_PROG_MAGIC; hdr.version = TS_PROG_VERSION; hdr.real_bytes = R; hdr.n_sections = TS_SEC_COUNT;
    hdr.V = V; hdr.Vf = Vf; hdr.Vf_pad = Vf_pad; hdr.Vstore = Vstore;
    hdr.F = F; hdr.B = B; hdr.VPT = VPT; hdr.G = G;
    hdr.n_chunks = n_chunks; hdr.grasp_chunk = grasp_chunk; hdr.slot_capacity = slot_cap; hdr.n_att = nA;
    hdr.n_edge_items = nE; hdr.n_tet_items = nT; hdr.n_att_items = nA; hdr.bank_conflicts = total_conf;
    hdr.n_slots_total = n_slots_total;
    int64_t off = roundup((int)sizeof(TsProgHeader), 256);
    for (int s = 0; s < TS_SEC_COUNT; ++s) { hdr.off[s] = off; off += ((sz[s] + 255) / 256) * 256; }
    hdr.total_bytes = off;
    blob.assign((size_t)off, 0);
    std::memcpy(blob.data(), &hdr, sizeof(hdr));
    put(blob, hdr.off[TS_SEC_CHUNK], chunk_rec);
    put(blob, hdr.off[TS_SEC_EDGE_IDX], edge_idx);
    put(blob, hdr.off[TS_SEC_TET_IDX], tet_idx);
    put(blob, hdr.off[TS_SEC_TET_SLOT], tet_slot);
    put(blob, hdr.off[TS_SEC_ATT_IDX], att_idx);
    put(blob, hdr.off[TS_SEC_ATT_SLOT], att_slot);
    put(blob, hdr.off[TS_SEC_REGION], region);
    put(blob, hdr.off[TS_SEC_VALENCE], valence);
    put(blob, hdr.off[TS_SEC_STATIC_CNT], static_cnt);
    put(blob, hdr.off[TS_SEC_S2O], s2o);
    put(blob, hdr.off[TS_SEC_O2S], o2s);
    put(blob, hdr.off[TS_SEC_FACES], faces_s);
    put(blob, hdr.off[TS_SEC_FACES_ORIG], faces_o);
    put(blob, hdr.off[TS_SEC_GSPLIT], gsplit);
    put(blob, hdr.off[TS_SEC_EDGE_C], edge_c);
    put(blob, hdr.off[TS_SEC_TET_C], tet_c);
    auto put_real = [&](int sec, const std::vector<double> &v) {
        if (R == 8) put(blob, hdr.off[sec], v);
        else { std::vector<float> f(v.begin(), v.end()); put(blob, hdr.off[sec], f); }
    };
    put_real(TS_SEC_EDGE_PAR, edge_par);
    put_real(TS_SEC_TET_RV, tet_rv);
    put_real(TS_SEC_ATT_PAR, att_par);
    put_real(TS_SEC_ATT_ANCHOR, att_anc);
    put_real(TS_SEC_W, wst);
    put_real(TS_SEC_REST, rest);

    std::memset(&info, 0, sizeof(info));
    info.precision = prec; info.block_threads = B; info.vertices_per_thread = VPT; info.n_chunks = n_chunks;
    info.n_free = Vf; info.n_store = Vstore; info.slot_capacity = slot_cap;
    info.n_edge_items = nE; info.n_tet_items = nT; info.n_att_items = nA; info.n_slots_total = n_slots_total;
    info.bank_conflicts_p1 = total_conf; info.program_bytes = off; info.compact = compact ? 1 : 0;
    return TS_OK;
}

}  // namespace ts
