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
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/tissuesim_b200.h"
#include "compiler.h"
#include "program.h"

namespace ts {

namespace {

struct Item {
    int kind;          // TsChunkKind
    int index;         // constraint index in its kind
    int nroles;
    int pos[4];        // storage positions of the roles
    int slot[4];       // slot id inside the chunk (-1 pinned endpoint)
    int vid[4];        // original vertex ids of the roles
    int chunk;
    int sign = 1;      // fp32 tets: -1 after an odd corner permutation (signed volume flips)
    int copy[4] = {0, 0, 0, 0};   // pinned corner: which shared-memory copy of the vertex it reads
    int idle_pos = 0;  // idle lane whose pos[] holds the four (pinned) positions it reads
};

// Pinned vertices never move, so fp32 fast programs keep several shared-memory copies of them
// (copy j of the pinned vertex at primary position p sits in bank (p + j * 32 / n_copies) mod 32):
// a pinned corner of a tet (or a pinned edge neighbour) reads whichever copy keeps its batch
// conflict-free.  Copy 0 is the primary (written back, divergence-checked); copies 1.. sit after
// Vown, where the kernel treats them like halo positions (loaded with the state, never written).
struct PinCopies {
    int n = 1, Vf_pad = 0, Vown = 0, Np_pad = 0;
    // copy j sits j * shift() banks from the primary: 9 (not 32 / n) so the bank sets of different
    // vertices overlap and a pinned corner's load can move between any two banks through chains
    int shift() const {
        if (const char *env = std::getenv("TS_PIN_SHIFT")) return std::atoi(env);
        return n > 1 ? 9 : 0;
    }
    bool pinned(int p) const { return p >= Vf_pad && p < Vown; }
    // storage position of copy j of the vertex whose primary position is p
    int pos(int p, int j) const {
        if (j == 0 || !pinned(p)) return p;
        return Vown + (j - 1) * Np_pad + (p - Vf_pad + j * shift()) % Np_pad;
    }
};

inline int roundup(int x, int m) { return (x + m - 1) / m * m; }

// effort of the bank-conflict searches (cluster parts compile K programs twice: a tenth)
thread_local double g_search_effort = 1.0;
// share of SA proposals that start from a conflicting sub-batch (TS_SA_FOCUS overrides)
thread_local double g_focus = 0.7;
// idle lanes allowed per 32-item tet batch (TS_TET_HOLES overrides; tuned on B200)
int g_tet_holes = 0;

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
    const long iters = (long)(g_search_effort * std::min<long>(400000L, 200L * n));
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
                                 int *extra_wavefronts, int max_holes = 0) {
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
        // lanes left without a conflict-free candidate: up to `max_holes` idle lanes (a dummy
        // item the kernel skips: it costs issue slots but no shared-memory wavefronts, and the
        // slack lets the banks of the remaining lanes stay distinct); the rest in index order
        int holes = 0;
        if (enable && done + pick.size() < items.size())
            holes = std::min(max_holes, batch - (int)pick.size());
        for (size_t i = first_free; i < items.size() && (int)pick.size() + holes < batch; ++i) {
            if (taken[i]) continue;
            pick.push_back((int)i);
            taken[i] = 1;
        }
        for (int i : pick) out.push_back(items[i]);
        for (int hcount = 0; hcount < holes && (int)pick.size() + hcount < batch; ++hcount) {
            Item dummy{};
            dummy.kind = items.empty() ? TS_CHUNK_TET : items[0].kind;
            dummy.index = -1;
            dummy.nroles = 0;
            out.push_back(dummy);
        }
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

// Extra shared-memory wavefronts of a scheduled item range (per role, per
// sub-batch of `bank_mod` lanes: max items on one bank - 1).
int batch_conflicts(const std::vector<Item> &items, int begin, int count, int bank_mod) {
    int extra = 0;
    for (int b0 = 0; b0 < count; b0 += bank_mod) {
        for (int r = 0; r < 4; ++r) {
            int cnt[32] = {0}, worst = 0;
            for (int k = b0; k < std::min(count, b0 + bank_mod); ++k) {
                const Item &it = items[begin + k];
                if (r < it.nroles) worst = std::max(worst, ++cnt[it.pos[r] % bank_mod]);
            }
            if (worst > 1) extra += worst - 1;
        }
    }
    return extra;
}

struct ListRef { std::vector<Item> *items; int begin, count; };

// Joint refinement of the phase-1 bank pattern by simulated annealing over
// three kinds of result-preserving moves:
//   * swap two items of one (chunk, kind) list          -> which lanes run together;
//   * swap the storage positions of two vertices of one warp group (or of the
//     pinned pool)                                        -> which bank a vertex lives in;
//     (a warp keeps the same vertices, so phase-2 balance and chunk padding are unchanged)
//   * swap an edge's endpoints (bit-exact in both builds: every product only
//     changes sign), or apply an orientation-preserving permutation to a tet's
//     corners (fp32 build only: it changes the fp64 expression trees).
// Deterministic (fixed-seed xorshift).  Slots are assigned afterwards from the
// final positions, so the per-vertex summation order is untouched.
void bank_refine(const std::vector<ListRef> &lists, std::vector<int> &o2s, std::vector<int> &s2o, int Vf,
                 int Vf_pad, int Vown, int bank_mod, bool permute_tets, int refine_iters,
                 const PinCopies &pc = PinCopies()) {
    struct Ref { int list, idx; };
    std::vector<Ref> items;                 // global item id -> (list, index)
    std::vector<int> sb_of, list_sb0;
    int nsb = 0;
    for (int l = 0; l < (int)lists.size(); ++l) {
        list_sb0.push_back(nsb);
        for (int i = 0; i < lists[l].count; ++i) { items.push_back({l, i}); sb_of.push_back(nsb + i / bank_mod); }
        nsb += (lists[l].count + bank_mod - 1) / bank_mod;
    }
    const int n = (int)items.size();
    if (n == 0) return;
    auto item = [&](int g) -> Item & { const Ref &r = items[g]; return (*lists[r.list].items)[lists[r.list].begin + r.idx]; };
    const int V = (int)o2s.size();
    std::vector<std::vector<std::pair<int, int>>> inc(V);
    for (int g = 0; g < n; ++g)
        for (int r = 0; r < item(g).nroles; ++r) inc[item(g).vid[r]].push_back({g, r});
    std::vector<int> cnt((size_t)nsb * 4 * bank_mod, 0), hist((size_t)nsb * 4 * 33, 0), mx((size_t)nsb * 4, 0);
    for (int q = 0; q < nsb * 4; ++q) hist[(size_t)q * 33] = bank_mod;
    auto add = [&](int sb, int r, int b, int delta) {
        const int q = sb * 4 + r;
        int &c = cnt[(size_t)q * bank_mod + b];
        hist[(size_t)q * 33 + c]--;
        c += delta;
        hist[(size_t)q * 33 + c]++;
        if (c > mx[q]) mx[q] = c;
        while (mx[q] > 0 && hist[(size_t)q * 33 + mx[q]] == 0) mx[q]--;
    };
    auto bank = [&](int v) { return o2s[v] % bank_mod; };
    // bank of role r of item x: its vertex's position, or the copy it reads (pinned corners)
    auto ibank = [&](const Item &x, int r) { return pc.pos(o2s[x.vid[r]], x.copy[r]) % bank_mod; };
    for (int g = 0; g < n; ++g)
        for (int r = 0; r < item(g).nroles; ++r) add(sb_of[g], r, ibank(item(g), r), +1);
    // objective: 4 x (extra wavefronts = max bank load - 1) + (items sharing a bank): the
    // second term is a smooth surrogate that lets the search cross the plateaus of the first
    auto sb_cost = [&](int sb) {
        int c = 0;
        for (int r = 0; r < 4; ++r) {
            const int q = sb * 4 + r;
            const int nz = bank_mod - hist[(size_t)q * 33];
            int items_in = 0;
            for (int k = 1; k <= mx[q]; ++k) items_in += k * hist[(size_t)q * 33 + k];
            c += 4 * std::max(0, mx[q] - 1) + (items_in - nz);
        }
        return c;
    };
    long total = 0;
    for (int sb = 0; sb < nsb; ++sb) total += sb_cost(sb);
    uint64_t rng = 0x2545F4914F6CDD1Dull;
    auto next = [&]() { rng ^= rng << 13; rng ^= rng >> 7; rng ^= rng << 17; return rng; };
    auto unif = [&]() { return (double)(next() >> 11) * (1.0 / 9007199254740992.0); };
    // pools a vertex may move in: its warp group (free), the owned pinned block, the halo block
    const int n_pinned = (int)std::count_if(s2o.begin() + Vf_pad, s2o.begin() + Vown, [](int v) { return v >= 0; });
    const int n_halo = (int)std::count_if(s2o.begin() + Vown, s2o.end(), [](int v) { return v >= 0; });
    std::vector<int> touched;
    auto collect = [&](int sb) { if (std::find(touched.begin(), touched.end(), sb) == touched.end()) touched.push_back(sb); };
    // thorough by default (measured on B200, reach_1170 fp32: 175 k iterations -> 140 residual
    // conflicts, 0.688 ms/step; 3 M -> 107, 0.674; 12 M -> 86, 0.670); programs are cached by
    // the Python layer, so the seconds are paid once per scene and library build
    long iters = refine_iters > 0 ? (long)refine_iters
               : refine_iters < 0 ? std::min<long>(600000L, 150L * n) : std::min<long>(4000000L, 3000L * n);
    iters = (long)(g_search_effort * iters);
    g_focus = 0.7;
    if (const char *env = std::getenv("TS_SA_FOCUS")) g_focus = std::atof(env);
    if (const char *env = std::getenv("TS_REFINE_ITERS")) iters = std::atol(env);
    const double T0 = 1.5, T1 = 0.05;
    // best state seen (the schedule lists, the vertex positions)
    long best = total;
    std::vector<std::vector<Item>> best_lists;
    std::vector<int> best_o2s = o2s, best_s2o = s2o;
    auto snapshot = [&]() {
        best_lists.clear();
        for (const ListRef &l : lists)
            best_lists.emplace_back(l.items->begin() + l.begin, l.items->begin() + l.begin + l.count);
        best_o2s = o2s; best_s2o = s2o;
    };
    snapshot();
    long last_snap = 0;
    for (long it = 0; it < iters && total > 0; ++it) {
        if (total < best && it - last_snap > 2000) { best = total; snapshot(); last_snap = it; }
        const double T = T0 * std::pow(T1 / T0, (double)it / iters);
        touched.clear();
        const int kind = (int)(next() % (pc.n > 1 ? 12 : 10));
        // --- propose ---------------------------------------------------------
        int g1 = -1, g2 = -1, u = -1, v = -1, perm = -1, rc = -1, old_copy = 0;
        // focus: most proposals start from an item of a sub-batch that still has a conflict
        auto pick = [&]() {
            int g = (int)(next() % n);
            if (unif() < g_focus)
                for (int tries = 0; tries < 8; ++tries) {
                    const int q = sb_of[g] * 4;
                    if (mx[q] > 1 || mx[q + 1] > 1 || mx[q + 2] > 1 || mx[q + 3] > 1) break;
                    g = (int)(next() % n);
                }
            return g;
        };
        if (kind < 5) {                                   // item swap inside a list
            g1 = pick();
            const Ref r1 = items[g1];
            const int cnt_l = lists[r1.list].count;
            const int j = (int)(next() % cnt_l);
            g2 = g1 - r1.idx + j;
            if (sb_of[g1] == sb_of[g2]) continue;
            collect(sb_of[g1]); collect(sb_of[g2]);
        } else if (kind < 8) {                            // vertex swap inside a warp group / the pinned pool
            const Item &src = item(pick());
            if (src.nroles == 0) continue;   // idle lane of a batch
            u = src.vid[next() % 2];
            const int pu = o2s[u];
            if (pu < 0) continue;
            int pv;
            if (pu < Vf_pad) {
                const int g = pu / 32;
                const int hi = std::min(Vf, 32 * g + 32);
                pv = 32 * g + (int)(next() % (hi - 32 * g));
            } else if (pu < Vown) {
                if (n_pinned < 2) continue;
                pv = Vf_pad + (int)(next() % n_pinned);
            } else {
                if (n_halo < 2) continue;
                pv = Vown + (int)(next() % n_halo);
            }
            v = s2o[pv];
            if (v < 0 || v == u || bank(u) == bank(v)) continue;
            for (auto &e : inc[u]) collect(sb_of[e.first]);
            for (auto &e : inc[v]) collect(sb_of[e.first]);
        } else if (kind >= 10) {                          // another copy for a pinned corner
            g1 = pick();
            Item &x = item(g1);
            if (x.nroles == 0) continue;
            const int r = (int)(next() % x.nroles);
            if (!pc.pinned(o2s[x.vid[r]])) continue;
            rc = r;
            old_copy = x.copy[r];
            collect(sb_of[g1]);
        } else {                                          // role permutation of one item
            g1 = (int)(next() % n);
            Item &x = item(g1);
            if (x.kind == TS_CHUNK_EDGE) perm = 0;
            else if (x.kind == TS_CHUNK_TET && permute_tets) perm = 1 + (int)(next() % 6);
            else continue;
            collect(sb_of[g1]);
        }
        long before = 0;
        for (int sb : touched) before += sb_cost(sb);
        // --- apply (as a reversible function) -----------------------------------
        auto remove_item = [&](int g) { Item &x = item(g); for (int r = 0; r < x.nroles; ++r) add(sb_of[g], r, ibank(x, r), -1); };
        auto insert_item = [&](int g) { Item &x = item(g); for (int r = 0; r < x.nroles; ++r) add(sb_of[g], r, ibank(x, r), +1); };
        auto permute = [&](Item &x, int p) {
            // edges: (a b) -> (b a); tets: the three double transpositions (orientation kept)
            if (p == 0) { std::swap(x.vid[0], x.vid[1]); std::swap(x.copy[0], x.copy[1]); }
            else {
                // tets (fp32 build): one transposition of two corners; the signed volume flips, so
                // the constraint is rewritten with -V0 (C' = -C, grad C' = -grad C: same correction)
                static const int tr[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
                std::swap(x.vid[tr[p - 1][0]], x.vid[tr[p - 1][1]]);
                std::swap(x.copy[tr[p - 1][0]], x.copy[tr[p - 1][1]]);
                x.sign = -x.sign;
            }
        };
        auto swap_vertices = [&]() {
            for (auto &e : inc[u]) add(sb_of[e.first], e.second, ibank(item(e.first), e.second), -1);
            for (auto &e : inc[v]) add(sb_of[e.first], e.second, ibank(item(e.first), e.second), -1);
            std::swap(o2s[u], o2s[v]);
            s2o[o2s[u]] = u; s2o[o2s[v]] = v;
            for (auto &e : inc[u]) add(sb_of[e.first], e.second, ibank(item(e.first), e.second), +1);
            for (auto &e : inc[v]) add(sb_of[e.first], e.second, ibank(item(e.first), e.second), +1);
        };
        auto recopy = [&](int c) {
            Item &x = item(g1);
            remove_item(g1);
            x.copy[rc] = c;
            insert_item(g1);
        };
        auto swap_items = [&]() {
            remove_item(g1); remove_item(g2);
            std::swap(item(g1), item(g2));
            insert_item(g1); insert_item(g2);
        };
        auto fix_inc_after_swap = [&]() {
            // after swapping item contents of g1 and g2, incidences (g1, r) <-> (g2, r)
            std::vector<int> vs;
            for (int g : {g1, g2}) for (int r = 0; r < item(g).nroles; ++r) vs.push_back(item(g).vid[r]);
            std::sort(vs.begin(), vs.end());
            vs.erase(std::unique(vs.begin(), vs.end()), vs.end());
            for (int w : vs)
                for (auto &e : inc[w]) {
                    if (e.first == g1) e.first = g2;
                    else if (e.first == g2) e.first = g1;
                }
        };
        auto permute_item = [&](int p) {
            Item &x = item(g1);
            remove_item(g1);
            // incidences carry the role index
            for (int r = 0; r < x.nroles; ++r)
                for (auto &e : inc[x.vid[r]]) if (e.first == g1 && e.second == r) e.second = -1 - r;
            permute(x, p);
            for (int r = 0; r < x.nroles; ++r)
                for (auto &e : inc[x.vid[r]]) if (e.first == g1 && e.second < 0) { e.second = r; break; }
            insert_item(g1);
        };
        if (g2 >= 0) { swap_items(); fix_inc_after_swap(); }
        else if (u >= 0) swap_vertices();
        else if (rc >= 0) recopy((old_copy + 1 + (int)(next() % (pc.n - 1))) % pc.n);
        else permute_item(perm);
        long after = 0;
        for (int sb : touched) after += sb_cost(sb);
        const long delta = after - before;
        if (delta <= 0 || unif() < std::exp(-(double)delta / T)) {
            total += delta;
            continue;
        }
        // --- revert ----------------------------------------------------------------
        if (g2 >= 0) { swap_items(); fix_inc_after_swap(); }
        else if (u >= 0) swap_vertices();
        else if (rc >= 0) recopy(old_copy);
        else {
            // inverse permutations: every move above is an involution
            permute_item(perm);
        }
    }
    if (std::getenv("TS_DEBUG_REFINE")) {
        long check = 0;
        for (int sb = 0; sb < nsb; ++sb) check += sb_cost(sb);
        std::fprintf(stderr, "bank_refine: tracked %ld recomputed %ld best %ld\n", total, check, best);
    }
    if (total > best) {   // restore the best state seen
        for (size_t l = 0; l < lists.size(); ++l)
            std::copy(best_lists[l].begin(), best_lists[l].end(), lists[l].items->begin() + lists[l].begin);
        o2s = best_o2s; s2o = best_s2o;
    }
}

// Conflict-free schedule of one edge list by bipartite edge colouring.
// Every edge is an arc between the bank of its role-a vertex and the bank of
// its role-b vertex; a warp batch (a half-warp for 64-bit data) is conflict-free
// iff its arcs form a matching of the bank x bank bipartite graph.  Endpoints are
// oriented to balance every bank's in/out degree (swapping roles is bit-exact),
// then Koenig's theorem gives a colouring with max-degree colours; each colour
// becomes one batch, padded with dummy edges between pinned vertices (they
// have no slots -- their stores are predicated off -- and touch no counter).  Returns false (list untouched)
// when there are no pinned vertices to build dummies from.
bool edge_coloring_schedule(std::vector<Item> &list, const std::vector<int> &o2s, const std::vector<int> &s2o,
                            int Vf_pad, int bank_mod) {
    const int n = (int)list.size();
    if (n < bank_mod) return false;
    std::vector<int> pinned_by_bank[32];
    for (int p = Vf_pad; p < (int)s2o.size(); ++p)
        if (s2o[p] >= 0) pinned_by_bank[p % bank_mod].push_back(s2o[p]);
    for (int b = 0; b < bank_mod; ++b)
        if (pinned_by_bank[b].size() < 2) return false;
    auto bank = [&](int v) { return o2s[v] % bank_mod; };
    // orientation: greedy, then improving flips
    std::vector<int> outd(bank_mod, 0), ind(bank_mod, 0);
    for (Item &e : list) {
        const int a = bank(e.vid[0]), b = bank(e.vid[1]);
        if (std::max(outd[b] + 1, ind[a] + 1) < std::max(outd[a] + 1, ind[b] + 1)) std::swap(e.vid[0], e.vid[1]);
        outd[bank(e.vid[0])]++; ind[bank(e.vid[1])]++;
    }
    for (int pass = 0; pass < 20; ++pass) {
        bool changed = false;
        for (Item &e : list) {
            const int a = bank(e.vid[0]), b = bank(e.vid[1]);
            if (a == b) continue;
            const int cur = std::max(std::max(outd[a], ind[b]), std::max(outd[b], ind[a]));
            const int alt = std::max(std::max(outd[a] - 1, ind[b] - 1), std::max(outd[b] + 1, ind[a] + 1));
            if (alt < cur) {
                outd[a]--; ind[b]--; outd[b]++; ind[a]++;
                std::swap(e.vid[0], e.vid[1]);
                changed = true;
            }
        }
        if (!changed) break;
    }
    int delta = 0;
    for (int b = 0; b < bank_mod; ++b) delta = std::max(delta, std::max(outd[b], ind[b]));
    const int C = std::max(delta, (n + bank_mod - 1) / bank_mod);
    // Koenig colouring: L[x][c] / R[y][c] = edge index using colour c at left bank x / right bank y
    std::vector<int> L((size_t)bank_mod * C, -1), R((size_t)bank_mod * C, -1), col(n, -1);
    auto Lc = [&](int x, int c) -> int & { return L[(size_t)x * C + c]; };
    auto Rc = [&](int y, int c) -> int & { return R[(size_t)y * C + c]; };
    for (int e = 0; e < n; ++e) {
        const int x = bank(list[e].vid[0]), y = bank(list[e].vid[1]);
        int a = 0; while (Lc(x, a) >= 0) ++a;
        int b = 0; while (Rc(y, b) >= 0) ++b;
        if (Rc(y, a) >= 0) {
            // flip the a/b alternating path that starts at right node y with colour a
            std::vector<int> path;
            int node = y; bool right = true; int c = a;
            while (true) {
                const int f = right ? Rc(node, c) : Lc(node, c);
                if (f < 0) break;
                path.push_back(f);
                node = right ? bank(list[f].vid[0]) : bank(list[f].vid[1]);
                right = !right;
                c = (c == a) ? b : a;
            }
            for (int f : path) {   // clear
                Lc(bank(list[f].vid[0]), col[f]) = -1; Rc(bank(list[f].vid[1]), col[f]) = -1;
            }
            for (int f : path) {   // swap a <-> b
                col[f] = (col[f] == a) ? b : a;
                Lc(bank(list[f].vid[0]), col[f]) = f; Rc(bank(list[f].vid[1]), col[f]) = f;
            }
        }
        col[e] = a;
        Lc(x, a) = e; Rc(y, a) = e;
    }
    // batches = colour classes, each padded to bank_mod lanes with dummies on unused banks
    std::vector<Item> out;
    out.reserve((size_t)C * bank_mod);
    for (int c = 0; c < C; ++c) {
        std::vector<int> members;
        std::vector<char> used_a(bank_mod, 0), used_b(bank_mod, 0);
        for (int x = 0; x < bank_mod; ++x) {
            const int e = Lc(x, c);
            if (e >= 0) { members.push_back(e); used_a[x] = 1; used_b[bank(list[e].vid[1])] = 1; }
        }
        if (members.empty()) continue;
        for (int e : members) out.push_back(list[e]);
        int fa = 0, fb = 0;
        for (int k = (int)members.size(); k < bank_mod; ++k) {
            while (used_a[fa]) ++fa;
            while (used_b[fb]) ++fb;
            used_a[fa] = used_b[fb] = 1;
            Item d{};
            d.kind = TS_CHUNK_EDGE; d.index = -1; d.nroles = 2; d.chunk = list[0].chunk;
            d.vid[0] = pinned_by_bank[fa][0];
            d.vid[1] = pinned_by_bank[fb][fa == fb ? 1 : 0];
            out.push_back(d);
        }
    }
    list.swap(out);
    return true;
}

template <typename Real>
struct Real4T { Real x, y, z, w; };

uint64_t xorshift(uint64_t &s) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return s; }
double unit(uint64_t &s) { return (double)(xorshift(s) >> 11) * (1.0 / 9007199254740992.0); }

// ---- fp32 gather programs: lanes for the owner edge gather ------------------------------------
// In round k of the owner gather the 32 lanes of warp w read their k-th neighbours; the round is
// conflict-free only if those sit in distinct banks, so the rounds a warp needs are at least the
// largest number of its neighbour reads that fall in one bank (its "bank load").  Free vertex
// banks are their lanes; lanes inside a warp group are free to permute (the group keeps its
// vertices, so phase-2 balance is unchanged).  Simulated annealing over lane swaps minimises, per
// warp, the bank load above the warp's longest list (the rounds it runs anyway), with a quadratic
// term that spreads the rest; pinned neighbours are left out (they read whichever copy fits).
// The tet corners' per-bank totals stay under the tet batches' capacity (penalty).
void balance_lanes(const std::vector<std::vector<int>> &nbrs, const std::vector<int> &tetval, std::vector<int> &o2s,
                   std::vector<int> &s2o, int Vf, int tet_cap_per_bank) {
    const int G = (Vf + 31) / 32;
    std::vector<int> kmax(G, 0);
    for (int p = 0; p < Vf; ++p) kmax[p / 32] = std::max(kmax[p / 32], (int)nbrs[s2o[p]].size());
    // rev[u]: free vertices that read u (u's bank lands in their warps' loads)
    const int V = (int)o2s.size();
    std::vector<std::vector<int>> rev(V);
    for (int p = 0; p < Vf; ++p)
        for (int u : nbrs[s2o[p]]) if (o2s[u] >= 0 && o2s[u] < Vf) rev[u].push_back(s2o[p]);
    std::vector<int> L((size_t)G * 32, 0), T(32, 0);
    auto warp = [&](int v) { return o2s[v] / 32; };
    auto bank = [&](int v) { return o2s[v] % 32; };
    for (int p = 0; p < Vf; ++p) {
        const int v = s2o[p];
        for (int u : nbrs[v]) if (o2s[u] >= 0 && o2s[u] < Vf) L[(size_t)warp(v) * 32 + bank(u)]++;
        T[p % 32] += tetval[v];
    }
    auto lcost = [&](int w, int l) { const int e = std::max(0, l - kmax[w]); return 64L * e + (long)l * l; };
    auto tcost = [&](int t) { return 256L * std::max(0, t - tet_cap_per_bank); };
    uint64_t rng = 0x9E3779B97F4A7C15ull;
    const long iters = std::min<long>(3000000L, 4000L * Vf);
    const double T0 = 8.0, T1 = 0.05;
    std::vector<std::pair<size_t, int>> delta;   // (L index, change)
    std::vector<size_t> cells;                   // touched cells (costs are evaluated on them)
    auto report = [&](const char *when) {
        if (!std::getenv("TS_DEBUG_REFINE")) return;
        for (int w = 0; w < G; ++w) {
            int mx = 0;
            for (int b = 0; b < 32; ++b) mx = std::max(mx, L[(size_t)w * 32 + b]);
            std::fprintf(stderr, "%s warp %d kmax %d free-neighbour bank load %d\n", when, w, kmax[w], mx);
        }
        int tm = 0; for (int b = 0; b < 32; ++b) tm = std::max(tm, T[b]);
        std::fprintf(stderr, "%s tet bank max %d (cap %d)\n", when, tm, tet_cap_per_bank);
    };
    report("before");
    for (long it = 0; it < iters; ++it) {
        const int pa = (int)(xorshift(rng) % Vf);
        const int g = pa / 32, hi = std::min(Vf, 32 * g + 32);
        const int pb = 32 * g + (int)(xorshift(rng) % (hi - 32 * g));
        if (pa == pb) continue;
        const int a = s2o[pa], b = s2o[pb];
        const int ba = pa % 32, bb = pb % 32;
        delta.clear();
        for (int v : rev[a]) { delta.push_back({(size_t)warp(v) * 32 + ba, -1}); delta.push_back({(size_t)warp(v) * 32 + bb, +1}); }
        for (int v : rev[b]) { delta.push_back({(size_t)warp(v) * 32 + bb, -1}); delta.push_back({(size_t)warp(v) * 32 + ba, +1}); }
        long before = tcost(T[ba]) + tcost(T[bb]), after;
        cells.clear();

        for (auto &d : delta) cells.push_back(d.first);
        std::sort(cells.begin(), cells.end());
        cells.erase(std::unique(cells.begin(), cells.end()), cells.end());
        for (size_t c : cells) before += lcost((int)(c / 32), L[c]);
        for (auto &d : delta) L[d.first] += d.second;
        T[ba] += tetval[b] - tetval[a]; T[bb] += tetval[a] - tetval[b];
        after = tcost(T[ba]) + tcost(T[bb]);
        for (size_t c : cells) after += lcost((int)(c / 32), L[c]);
        const double temp = T0 * std::pow(T1 / T0, (double)it / iters);
        if (after <= before || unit(rng) < std::exp(-(double)(after - before) / temp)) {
            std::swap(o2s[a], o2s[b]);
            s2o[pa] = b; s2o[pb] = a;
        } else {
            for (auto &d : delta) L[d.first] -= d.second;
            T[ba] -= tetval[b] - tetval[a]; T[bb] -= tetval[a] - tetval[b];
        }
    }
    report("after");
}

// ---- fp32 gather programs: conflict-free tet batches ------------------------------------------
// A batch of 32 tets is conflict-free when, for each role, its 32 corners sit in distinct banks.
// With free corner order (fp32: any permutation, the rest volume's sign follows the parity) that
// holds iff every bank carries at most 4 of the batch's 128 corners: the batch is then a bipartite
// multigraph (tets x banks) of maximum degree 4, which Koenig's theorem colours with 4 colours =
// roles.  So: (1) simulated annealing packs the tets into batches under a per-bank capacity of 4
// (moves: swap two tets, move a tet into a batch's spare lane, re-pick the copy a pinned corner
// reads); (2) each batch's roles come from an exact bipartite edge colouring; (3) spare lanes get
// idle items whose four role positions are pinned positions on banks the batch leaves unused.
// Returns the residual extra wavefronts per pass (0 when every batch fits).
int pack_tet_batches(std::vector<Item> &items, const std::vector<int> &o2s, const std::vector<int> &s2o,
                     const PinCopies &pc, int Vstore) {
    const int n = (int)items.size();
    if (n == 0) return 0;
    int extra_batches = 0;
    if (const char *env = std::getenv("TS_TET_EXTRA_BATCHES")) extra_batches = std::atoi(env);
    const int NB = (n + 31) / 32 + extra_batches;
    auto tok_bank = [&](const Item &x, int r) { return pc.pos(o2s[x.vid[r]], x.copy[r]) % 32; };
    std::vector<int> batch(n), size(NB, 0), cnt((size_t)NB * 32, 0);
    std::vector<std::vector<int>> members(NB);
    // greedy start: each tet into the batch (with room) where it adds the least excess
    for (int t = 0; t < n; ++t) {
        int best = -1, bexc = 1 << 30;
        for (int j = 0; j < NB; ++j) {
            if (size[j] >= 32) continue;
            int exc = 0;
            for (int r = 0; r < 4; ++r) exc += cnt[(size_t)j * 32 + tok_bank(items[t], r)] >= 4;
            if (exc < bexc) { bexc = exc; best = j; if (!exc) break; }
        }
        batch[t] = best; size[best]++;
        for (int r = 0; r < 4; ++r) cnt[(size_t)best * 32 + tok_bank(items[t], r)]++;
    }
    auto cell = [&](int j, int b) -> int & { return cnt[(size_t)j * 32 + b]; };
    long total = 0;
    for (int j = 0; j < NB; ++j) for (int b = 0; b < 32; ++b) total += std::max(0, cell(j, b) - 4);
    std::vector<std::vector<int>> pinned_roles(n);
    for (int t = 0; t < n; ++t)
        for (int r = 0; r < 4; ++r) if (pc.pinned(o2s[items[t].vid[r]])) pinned_roles[t].push_back(r);
    uint64_t rng = 0x2545F4914F6CDD1Dull;
    long iters = std::min<long>(12000000L, 3000L * n);   // reach_1170: ~3.5 M, a few seconds
    if (const char *env = std::getenv("TS_PACK_ITERS")) iters = std::atol(env);
    const double T0 = 3.0, T1 = 0.05;
    auto exc = [&](int v) { return std::max(0, v - 4); };
    // objective per (batch, bank) cell: the excess over 4 (extra wavefronts) plus a quadratic term
    // that keeps the search moving on the plateaus of the excess
    auto cc = [&](int v) { return 16L * exc(v) + (long)v * v; };
    long obj = 0;
    for (int j = 0; j < NB; ++j) for (int b = 0; b < 32; ++b) obj += cc(cell(j, b));
    const long total0 = total;
    long n_acc = 0, n_it = 0;
    auto bad_item = [&](int t) {
        for (int r = 0; r < 4; ++r) if (cell(batch[t], tok_bank(items[t], r)) > 4) return true;
        return false;
    };
    // annealing passes (the later ones reheated less) until the packing is conflict-free
    for (int pass = 0; pass < 4 && total > 0; ++pass)
    for (long it = 0; it < iters && total > 0; ++it) {
        const double temp = (T0 / (1 + pass)) * std::pow(T1 / (T0 / (1 + pass)), (double)it / iters);
        ++n_it;
        const int kind = (int)(xorshift(rng) % 8);
        int t = (int)(xorshift(rng) % n);
        for (int tries = 0; tries < 16 && !bad_item(t); ++tries) t = (int)(xorshift(rng) % n);   // focus
        long dobj = 0, dexc = 0;
        auto bump = [&](int j, int b, int sgn) {
            int &c = cell(j, b);
            dobj -= cc(c); dexc -= exc(c);
            c += sgn;
            dobj += cc(c); dexc += exc(c);
        };
        auto shift = [&](int x, int from, int to) {
            for (int r = 0; r < 4; ++r) { const int b = tok_bank(items[x], r); bump(from, b, -1); bump(to, b, +1); }
        };
        if (kind < 5) {                                   // swap two tets between batches / move to a spare lane
            const int u = (int)(xorshift(rng) % n);
            const int ja = batch[t], jb = batch[u];
            if (ja == jb) continue;
            const bool move = kind == 4 && size[jb] < 32;
            shift(t, ja, jb);
            if (!move) shift(u, jb, ja);
            if (dobj <= 0 || unit(rng) < std::exp(-(double)dobj / temp)) {
                total += dexc; obj += dobj; ++n_acc;
                batch[t] = jb;
                if (move) { size[ja]--; size[jb]++; }
                else batch[u] = ja;
            } else {
                if (!move) shift(u, ja, jb);
                shift(t, jb, ja);
            }
        } else {                                          // re-pick a pinned corner's copy
            if (pc.n < 2 || pinned_roles[t].empty()) continue;
            const int r = pinned_roles[t][xorshift(rng) % pinned_roles[t].size()];
            const int j = batch[t];
            const int c0 = items[t].copy[r];
            const int b0 = tok_bank(items[t], r);
            items[t].copy[r] = (c0 + 1 + (int)(xorshift(rng) % (pc.n - 1))) % pc.n;
            const int b1 = tok_bank(items[t], r);
            bump(j, b0, -1); bump(j, b1, +1);
            if (dobj <= 0 || unit(rng) < std::exp(-(double)dobj / temp)) {
                total += dexc; obj += dobj;
            } else {
                bump(j, b1, -1); bump(j, b0, +1);
                items[t].copy[r] = c0;
            }
        }
    }
    if (std::getenv("TS_DEBUG_REFINE")) {
        long chk = 0;
        for (int j = 0; j < NB; ++j) for (int b = 0; b < 32; ++b) chk += std::max(0, cell(j, b) - 4);
        std::fprintf(stderr, "pack: %d tets, %d batches, excess %ld -> %ld (check %ld), %ld iterations, %ld swaps accepted\n",
                     n, NB, total0, total, chk, n_it, n_acc);
    }
    // pinned storage positions by bank (for the idle lanes)
    std::vector<int> pin_by_bank(32, -1);
    for (int p = pc.Vf_pad; p < Vstore; ++p)
        if (s2o[p] >= 0 && pin_by_bank[p % 32] < 0) pin_by_bank[p % 32] = p;
    // per batch: roles by bipartite edge colouring (tets x banks, 4 colours)
    std::vector<Item> out;
    out.reserve((size_t)NB * 32);
    for (int j = 0; j < NB; ++j) members[j].clear();
    for (int t = 0; t < n; ++t) members[batch[t]].push_back(t);
    int residual = 0;
    for (int j = 0; j < NB; ++j) {
        const std::vector<int> &mb = members[j];
        const int m = (int)mb.size();
        // colour[i][k]: role of corner k of member i; at_t[i][c] / at_b[b][c]: corner holding colour c
        const int NC = std::max(4, [&] { int mx = 0; for (int b = 0; b < 32; ++b) mx = std::max(mx, cell(j, b)); return mx; }());
        std::vector<int> col((size_t)m * 4, -1), at_t((size_t)m * NC, -1), at_b((size_t)32 * NC, -1);
        auto bk = [&](int i, int k) { return tok_bank(items[mb[i]], k); };
        for (int i = 0; i < m; ++i)
            for (int k = 0; k < 4; ++k) {
                const int b = bk(i, k);
                int ca = -1, cb = -1;
                for (int c = 0; c < NC && ca < 0; ++c) if (at_t[(size_t)i * NC + c] < 0) ca = c;
                for (int c = 0; c < NC && cb < 0; ++c) if (at_b[(size_t)b * NC + c] < 0) cb = c;
                if (at_b[(size_t)b * NC + ca] >= 0) {
                    // flip the (ca, cb) alternating path that starts at bank b
                    std::vector<int> path;   // corners (i * 4 + k) along the path
                    int node = b, side = 1, c_want = ca;
                    while (true) {
                        const int e = side ? at_b[(size_t)node * NC + c_want] : at_t[(size_t)node * NC + c_want];
                        if (e < 0) break;
                        path.push_back(e);
                        node = side ? e / 4 : bk(e / 4, e % 4);
                        side ^= 1;
                        c_want = c_want == ca ? cb : ca;
                    }
                    for (int e : path) {   // clear, then recolour swapped
                        at_t[(size_t)(e / 4) * NC + col[e]] = -1;
                        at_b[(size_t)bk(e / 4, e % 4) * NC + col[e]] = -1;
                    }
                    for (int e : path) {
                        col[e] = col[e] == ca ? cb : ca;
                        at_t[(size_t)(e / 4) * NC + col[e]] = e;
                        at_b[(size_t)bk(e / 4, e % 4) * NC + col[e]] = e;
                    }
                }
                col[(size_t)i * 4 + k] = ca;
                at_t[(size_t)i * NC + ca] = i * 4 + k;
                at_b[(size_t)b * NC + ca] = i * 4 + k;
            }
        // members: corners with colour >= 4 (over-full banks only) go to the free role of their tet
        std::vector<std::vector<char>> used(4, std::vector<char>(32, 0));
        for (int i = 0; i < m; ++i) {
            Item x = items[mb[i]];
            int role_of[4], taken = 0;
            for (int k = 0; k < 4; ++k) { role_of[k] = col[(size_t)i * 4 + k] < 4 ? col[(size_t)i * 4 + k] : -1; if (role_of[k] >= 0) taken |= 1 << role_of[k]; }
            for (int k = 0; k < 4; ++k)
                if (role_of[k] < 0) { int r = 0; while (taken >> r & 1) ++r; role_of[k] = r; taken |= 1 << r; }
            Item y = x;
            int perm[4];
            for (int k = 0; k < 4; ++k) { y.vid[role_of[k]] = x.vid[k]; y.copy[role_of[k]] = x.copy[k]; perm[k] = role_of[k]; }
            int inv = 0;
            for (int a = 0; a < 4; ++a) for (int b2 = a + 1; b2 < 4; ++b2) inv += perm[a] > perm[b2];
            if (inv & 1) y.sign = -y.sign;
            for (int r = 0; r < 4; ++r) used[r][tok_bank(y, r)]++;
            out.push_back(y);
        }
        for (int r = 0; r < 4; ++r) for (int b = 0; b < 32; ++b) residual += std::max(0, (int)used[r][b] - 1);
        // idle lanes: one position per role on a bank that role leaves unused (all idle lanes of the
        // batch read the same four addresses: a broadcast)
        if (m < 32) {
            Item dmy{};
            dmy.kind = TS_CHUNK_TET; dmy.index = -1; dmy.nroles = 0; dmy.idle_pos = 1;
            for (int r = 0; r < 4; ++r) {
                int p = pc.Vf_pad;
                for (int b = 0; b < 32; ++b) if (!used[r][b] && pin_by_bank[b] >= 0) { p = pin_by_bank[b]; break; }
                dmy.pos[r] = p;
            }
            for (int i = m; i < 32; ++i) out.push_back(dmy);
        }
    }
    items.swap(out);
    return residual;
}

// Owner-gather rounds of fp32 4-byte programs with pinned copies: conflict-free by bipartite edge
// colouring (lanes x banks).  A pinned neighbour reads the copy on the least-loaded bank, then
// Koenig's theorem colours each warp's reads with K colours = rounds, K = max(longest list, largest
// bank load) -- no round has two reads on one bank.  A lane's gaps become -1 (null records).
// other(p, e): storage position of edge e's endpoint that is not p.
template <typename Other>
void colour_gather_rounds(std::vector<std::vector<int>> &lists, std::vector<std::vector<int>> &ecopy, int G, int Vf,
                          const PinCopies &pc, Other other) {
    for (int g = 0; g < G; ++g) {
        const int p0 = 32 * g, p1 = std::min(Vf, 32 * g + 32);
        if (p1 <= p0) continue;
        struct Tok { int p, e, copy, bank; };
        std::vector<Tok> toks;
        std::vector<int> deg(32, 0), lane_deg(32, 0), pinned_tok;
        for (int p = p0; p < p1; ++p)
            for (int e : lists[p]) {
                const int q = other(p, e);
                lane_deg[p % 32]++;
                if (pc.pinned(q)) { pinned_tok.push_back((int)toks.size()); toks.push_back({p, e, 0, -1}); }
                else { toks.push_back({p, e, 0, q % 32}); deg[q % 32]++; }
            }
        for (int ti : pinned_tok) {   // least-loaded copy
            Tok &t = toks[ti];
            const int q = other(t.p, t.e);
            int bc = 0, bb = pc.pos(q, 0) % 32;
            for (int j = 1; j < pc.n; ++j) {
                const int b = pc.pos(q, j) % 32;
                if (deg[b] < deg[bb]) { bb = b; bc = j; }
            }
            t.copy = bc; t.bank = bb; deg[bb]++;
        }
        const int NC = std::max(*std::max_element(deg.begin(), deg.end()),
                                *std::max_element(lane_deg.begin(), lane_deg.end()));
        if (NC == 0) continue;
        std::vector<int> col(toks.size(), -1), at_l((size_t)32 * NC, -1), at_b((size_t)32 * NC, -1);
        for (int ti = 0; ti < (int)toks.size(); ++ti) {
            const int l = toks[ti].p % 32, b = toks[ti].bank;
            int ca = -1, cb = -1;
            for (int c = 0; c < NC && ca < 0; ++c) if (at_l[(size_t)l * NC + c] < 0) ca = c;
            for (int c = 0; c < NC && cb < 0; ++c) if (at_b[(size_t)b * NC + c] < 0) cb = c;
            if (at_b[(size_t)b * NC + ca] >= 0) {   // flip the (ca, cb) path from bank b
                std::vector<int> path;
                int node = b, side = 1, cw = ca;
                while (true) {
                    const int e = side ? at_b[(size_t)node * NC + cw] : at_l[(size_t)node * NC + cw];
                    if (e < 0) break;
                    path.push_back(e);
                    node = side ? toks[e].p % 32 : toks[e].bank;
                    side ^= 1;
                    cw = cw == ca ? cb : ca;
                }
                for (int e : path) { at_l[(size_t)(toks[e].p % 32) * NC + col[e]] = -1; at_b[(size_t)toks[e].bank * NC + col[e]] = -1; }
                for (int e : path) {
                    col[e] = col[e] == ca ? cb : ca;
                    at_l[(size_t)(toks[e].p % 32) * NC + col[e]] = e;
                    at_b[(size_t)toks[e].bank * NC + col[e]] = e;
                }
            }
            col[ti] = ca;
            at_l[(size_t)l * NC + ca] = ti;
            at_b[(size_t)b * NC + ca] = ti;
        }
        // rounds -> lists: up to the lane's last coloured round, gaps as nulls (-1)
        for (int p = p0; p < p1; ++p) {
            int last = -1;
            for (int c = 0; c < NC; ++c) if (at_l[(size_t)(p % 32) * NC + c] >= 0) last = c;
            std::vector<int> nl(last + 1, -1), nc(last + 1, 0);
            for (int c = 0; c <= last; ++c) {
                const int ti = at_l[(size_t)(p % 32) * NC + c];
                if (ti >= 0) { nl[c] = toks[ti].e; nc[c] = toks[ti].copy; }
            }
            lists[p] = nl;
            ecopy[p] = nc;
        }
}
}

// Owner-gather rounds of other fp32 programs: in round k the 32 lanes of a warp read their k-th
// neighbours; permute each lane's list (and re-pick pinned copies) so one round's neighbours sit in
// distinct banks as far as possible (deterministic local search, sum over rounds of the largest
// bank multiplicity).  The order of a vertex's edges is free in fp32 (fp64 keeps edge-index order).
template <typename Other, typename NbrPos>
void order_gather_rounds(std::vector<std::vector<int>> &lists, std::vector<std::vector<int>> &ecopy, int G,
                         const PinCopies &pc, Other other, NbrPos nbr_pos) {
    uint64_t rs = 0x2545F4914F6CDD1Dull;
    auto rnd = [&]() { rs ^= rs << 13; rs ^= rs >> 7; rs ^= rs << 17; return rs; };
    for (int g = 0; g < G; ++g) {
        int kmax = 0;
        for (int p = 32 * g; p < 32 * g + 32; ++p) kmax = std::max(kmax, (int)lists[p].size());
        if (kmax < 1) continue;
        std::vector<int> cnt((size_t)kmax * 32, 0);
        auto bank = [&](int p, int k) { return nbr_pos(p, k) % 32; };
        for (int p = 32 * g; p < 32 * g + 32; ++p)
            for (int k = 0; k < (int)lists[p].size(); ++k) cnt[(size_t)k * 32 + bank(p, k)]++;
        auto rmax = [&](int k) { int m = 0; for (int b = 0; b < 32; ++b) m = std::max(m, cnt[(size_t)k * 32 + b]); return m; };
        const long iters = 6000L * kmax;
        for (long it = 0; it < iters; ++it) {
            const int p = 32 * g + (int)(rnd() % 32);
            const int n = (int)lists[p].size();
            if (n < 1) continue;
            if (pc.n > 1 && (rnd() & 1)) {          // another copy of a pinned neighbour
                const int k = (int)(rnd() % n);
                if (!pc.pinned(other(p, lists[p][k]))) continue;
                const int b0 = bank(p, k), c0 = ecopy[p][k];
                const int before = rmax(k);
                ecopy[p][k] = (c0 + 1 + (int)(rnd() % (pc.n - 1))) % pc.n;
                const int b1 = bank(p, k);
                cnt[(size_t)k * 32 + b0]--; cnt[(size_t)k * 32 + b1]++;
                if (rmax(k) > before) {
                    cnt[(size_t)k * 32 + b1]--; cnt[(size_t)k * 32 + b0]++;
                    ecopy[p][k] = c0;
                }
                continue;
            }
            if (n < 2) continue;
            const int ka = (int)(rnd() % n), kb = (int)(rnd() % n);
            const int ba = bank(p, ka), bb = bank(p, kb);
            if (ka == kb || ba == bb) continue;
            const int before = rmax(ka) + rmax(kb);
            cnt[(size_t)ka * 32 + ba]--; cnt[(size_t)kb * 32 + ba]++;
            cnt[(size_t)kb * 32 + bb]--; cnt[(size_t)ka * 32 + bb]++;
            if (rmax(ka) + rmax(kb) <= before) {
                std::swap(lists[p][ka], lists[p][kb]);
                std::swap(ecopy[p][ka], ecopy[p][kb]);
            } else {
                cnt[(size_t)ka * 32 + ba]++; cnt[(size_t)kb * 32 + ba]--;
                cnt[(size_t)kb * 32 + bb]++; cnt[(size_t)ka * 32 + bb]--;
            }
        }
}
}

// Phase-1 work split (the WSPLIT section): each warp takes a contiguous range of 32-item tet batches
// of the chunk, sized so that its owner edge gather (chunk 0; the longest lane's incidences, CE
// each) plus its batches (CT each) is about the same for every warp.  int32 [n_chunks][B/32 + 1].
std::vector<int32_t> warp_split(const std::vector<TsChunk> &chunk_rec, const std::vector<int32_t> &evalence, bool eg,
                                int B, int VPT, int Vf) {
    const int NW = B / 32, n_chunks = (int)chunk_rec.size();
    std::vector<int32_t> wsplit((size_t)n_chunks * (NW + 1), 0);
    const double CE = 1.0;   // owner-gathered edge incidence vs one tet batch (tuned on B200, tools/sweep_ct.sh)
    double CT = 4.0;
    if (const char *env = std::getenv("TS_SPLIT_CT")) CT = std::atof(env);
    for (int c = 0; c < n_chunks; ++c) {
        const int nt = chunk_rec[c].tet_count;
        const int nb = (nt + 31) / 32;
        std::vector<double> ce(NW, 0.0);
        if (eg && c == 0)
            for (int w = 0; w < NW; ++w)
                for (int lane = 0; lane < 32; ++lane) {
                    int sum = 0;
                    for (int r = 0; r < VPT; ++r) {
                        const int p = r * B + 32 * w + lane;
                        if (p < Vf) sum += evalence[p];
                    }
                    ce[w] = std::max(ce[w], CE * sum);
                }
        // smallest level T with sum_w floor((T - ce_w) / CT) >= nb batches (32 items each)
        double lo = 0.0, hi = 1e9;
        auto fits = [&](double T) {
            long tot = 0;
            for (int w = 0; w < NW; ++w) tot += std::max(0L, (long)std::floor((T - ce[w]) / CT));
            return tot >= nb;
        };
        for (int it = 0; it < 100; ++it) { const double mid = 0.5 * (lo + hi); (fits(mid) ? hi : lo) = mid; }
        int left = nb, start = 0;
        for (int w = 0; w < NW; ++w) {
            int take = std::min(left, std::max(0, (int)std::floor((hi - ce[w]) / CT)));
            if (w == NW - 1) take = left;
            wsplit[(size_t)c * (NW + 1) + w] = std::min(start, nt);
            start += 32 * take;
            left -= take;
        }
        wsplit[(size_t)c * (NW + 1) + NW] = nt;
    }
    return wsplit;
}

// The owner-gathered distance constraints of a program (EINC / EREGION / EVAL / RLTAB sections).
struct GatherSpec {
    const ts_scene_desc *d;
    const std::vector<char> *edge_live;
    const std::vector<int> *o2s, *s2o;
    const PinCopies *pc;
    std::function<bool(int)> own_free, is_free;
    int Vf, Vf_pad, G, Vstore, R;
    bool boff, compact, packed, schedule;
};
struct GatherProgram {
    std::vector<float> pair_tab;              // 4-byte records: {rest length, coefficient} pairs
    std::vector<int32_t> eregion, evalence;   // [G] base record of each warp group, [Vf_pad] records per vertex
    std::vector<uint8_t> einc;                // the records, warp-interleaved
    int einc_bytes = 0, n_einc = 0;           // record size; live (edge, free endpoint) incidences
};

// Free vertex p walks its live incident edges in edge-index order (the reference's
// accumulation order, _kernels.pyx:102-139).  Its correction from edge (a, b) is
//   -(w_p scale) (x_p - x_q),  scale = m ks (dist - rest) / (dist (w_a + w_b) + (1 - m)),
// bitwise the reference's (-w_a scale) dx for p = a and (w_b scale) dx for p = b, since
// x_b - x_a = -(x_a - x_b) exactly and the squares / weight sum are symmetric.
// fp32 byte-offset programs whose rest lengths take few distinct fp32 values (a structured
// slab has 2) use 4-byte records: {neighbour offset (16) | 8 x pair index (16)} with a small table
// of (rest length, coefficient) pairs -- coefficient = -k_s w_p / (w_p + w_q), i.e. -k_s / 2,
// or -k_s for a pinned neighbour (uniform free mass) -- half the L1 footprint of the edge
// stream and one shared load for both operands.  Pair 0 is the null record {0, 0} (a gap of
// the conflict-free rounds): its term is exactly zero.
// static_cnt gains one per live incidence (and per null record that reads its own position).
GatherProgram build_gather(const GatherSpec &gs, std::vector<int32_t> &static_cnt) {
    const ts_scene_desc &d = *gs.d;
    const int E = d.n_edge;
    const double *w = d.inverse_mass;
    const std::vector<char> &edge_live = *gs.edge_live;
    const std::vector<int> &o2s = *gs.o2s, &s2o = *gs.s2o;
    const PinCopies &pc = *gs.pc;
    const int Vf = gs.Vf, Vf_pad = gs.Vf_pad, G = gs.G, Vstore = gs.Vstore, R = gs.R;
    const bool boff = gs.boff, compact = gs.compact, packed = gs.packed;
    const auto &own_free = gs.own_free;
    const auto &is_free = gs.is_free;
    GatherProgram out;
    std::vector<float> rl_tab;
    std::vector<int> rl_idx(E, -1);
    if (boff && 12 * Vstore <= 65535) {
        std::vector<float> vals;
        for (int e = 0; e < E; ++e) if (edge_live[e]) vals.push_back((float)d.rest_length[e]);
        std::sort(vals.begin(), vals.end());
        vals.erase(std::unique(vals.begin(), vals.end()), vals.end());
        if ((int)vals.size() <= 256) {
            rl_tab = vals;
            for (int e = 0; e < E; ++e)
                if (edge_live[e])
                    rl_idx[e] = (int)(std::lower_bound(vals.begin(), vals.end(), (float)d.rest_length[e]) - vals.begin());
        }
    }
    out.einc_bytes = !rl_tab.empty() ? 4 : ((R == 4 && compact) ? 8 : 16);
    const int einc_bytes = out.einc_bytes;
    std::vector<float> &pair_tab = out.pair_tab;     // RLTAB section of 4-byte programs: {rl, coef} pairs
    auto pair_index = [&](int e, bool pinned_nbr) {   // 1 + 2 * rest-length index + pinned
        return 1 + 2 * rl_idx[e] + (pinned_nbr ? 1 : 0);
    };
    if (einc_bytes == 4) {
        pair_tab.assign(2 * (1 + 2 * rl_tab.size()), 0.0f);
        const float ks_f = (float)d.k_s;
        for (size_t i = 0; i < rl_tab.size(); ++i)
            for (int pin = 0; pin < 2; ++pin) {
                const int k = 1 + 2 * (int)i + pin;
                pair_tab[2 * k] = rl_tab[i];
                pair_tab[2 * k + 1] = -(pin ? ks_f : 0.5f * ks_f);
            }
    }
    out.eregion.assign(G, 0);
    out.evalence.assign(Vf_pad, 0);
    std::vector<int32_t> &eregion = out.eregion, &evalence = out.evalence;
    std::vector<uint8_t> &einc = out.einc;
    int &n_einc = out.n_einc;
    {
        std::vector<std::vector<int>> lists(Vf_pad);
        for (int e = 0; e < E; ++e) {
            if (!edge_live[e]) continue;
            const int a = d.edges[2 * e], b = d.edges[2 * e + 1];
            if (own_free(a)) lists[o2s[a]].push_back(e);
            if (own_free(b)) lists[o2s[b]].push_back(e);
        }
        // fp32: the order of a vertex's edges is free (fp64 keeps edge-index order, the reference's
        // summation order).  In round k the 32 lanes of a warp read their k-th neighbours: permute
        // each lane's list so the neighbours of one round sit in distinct banks as far as possible
        // (deterministic local search, sum over rounds of the largest bank multiplicity)
        // a pinned neighbour may be read from any of its copies (PinCopies): a second move kind
        std::vector<std::vector<int>> ecopy(Vf_pad);
        for (int p = 0; p < Vf_pad; ++p) ecopy[p].assign(lists[p].size(), 0);
        auto other = [&](int p, int e) {
            const int a = d.edges[2 * e], b = d.edges[2 * e + 1];
            return o2s[a == s2o[p] ? b : a];
        };
        auto nbr_pos = [&](int p, int k) { return pc.pos(other(p, lists[p][k]), ecopy[p][k]); };
        if (packed && einc_bytes == 4) colour_gather_rounds(lists, ecopy, G, Vf, pc, other);
        else if (R == 4 && gs.schedule) order_gather_rounds(lists, ecopy, G, pc, other, nbr_pos);
        int base = 0;
        for (int g = 0; g < G; ++g) {
            int kmax = 0;
            for (int p = 32 * g; p < 32 * g + 32; ++p) kmax = std::max(kmax, (int)lists[p].size());
            eregion[g] = base;
            base += 32 * kmax;
        }
        einc.assign(((size_t)base + 64) * einc_bytes, 0);   // + two padding rows: unclamped prefetches
        // null records read a pinned position on a bank their round leaves free (no conflict; a
        // pinned neighbour is never within 1e-12 of a free vertex, so the null is not degenerate),
        // or -- when no such position exists -- their own position (dx = 0: degenerate, counted in
        // static_cnt so the applied count is unchanged)
        std::vector<int> pin_at_bank(32, -1);
        for (int q = Vf_pad; q < Vstore; ++q)
            if (s2o[q] >= 0 && !is_free(s2o[q]) && pin_at_bank[q % 32] < 0) pin_at_bank[q % 32] = q;
        std::vector<int> null_pos((size_t)G * 64, -2);   // per (warp, round): chosen position (-1: own)
        auto null_for = [&](int g, int k) {
            int &np = null_pos[(size_t)g * 64 + std::min(k, 63)];
            if (np != -2 && k < 64) return np;
            std::vector<char> used(32, 0);
            for (int q = 32 * g; q < std::min(Vf, 32 * g + 32); ++q)
                if (k < (int)lists[q].size() && lists[q][k] >= 0) used[nbr_pos(q, k) % 32] = 1;
            int pos = -1;
            for (int b = 0; b < 32 && pos < 0; ++b) if (!used[b] && pin_at_bank[b] >= 0) pos = pin_at_bank[b];
            if (k < 64) np = pos;
            return pos;
        };
        for (int p = 0; p < Vf; ++p) {
            const int self = s2o[p];
            evalence[p] = (int)lists[p].size();
            for (int k = 0; k < evalence[p]; ++k) {
                const int e = lists[p][k];
                if (e < 0) {   // null record (4-byte programs): pair 0, a zero term
                    uint8_t *rec = einc.data() + (size_t)(eregion[p / 32] + 32 * k + p % 32) * einc_bytes;
                    const int np = null_for(p / 32, k);
                    const uint32_t word = (uint32_t)(12 * (np >= 0 ? np : p)) & 0xffffu;
                    if (np < 0) static_cnt[p] += 1;   // own position: counted degenerate every substep
                    std::memcpy(rec, &word, 4);
                    continue;
                }
                ++n_einc;
                static_cnt[p] += 1;
                const int a = d.edges[2 * e], b = d.edges[2 * e + 1];
                const int q = a == self ? b : a;
                const int qpos = nbr_pos(p, k);
                // bit 31: the neighbour is pinned (w = 0); with uniform free mass that fixes the
                // weight ratio (compact fp32 records), and halo neighbours of a cluster part are free
                const int32_t nbr = (boff ? 12 * qpos : qpos) | (is_free(q) ? 0 : (int32_t)0x80000000u);
                uint8_t *rec = einc.data() + (size_t)(eregion[p / 32] + 32 * k + p % 32) * einc_bytes;
                const double rl = d.rest_length[e];
                if (einc_bytes == 4) {
                    // upper half: the pair's byte offset in the table (8 B per pair): one shift to decode
                    const uint32_t word = (uint32_t)(nbr & 0xffff) | ((uint32_t)(8 * pair_index(e, !is_free(q))) << 16);
                    std::memcpy(rec, &word, 4);
                    continue;
                }
                std::memcpy(rec, &nbr, 4);
                if (einc_bytes == 8) {
                    const float f = (float)rl;
                    std::memcpy(rec + 4, &f, 4);
                } else if (R == 8) {
                    std::memcpy(rec + 8, &rl, 8);
                } else {
                    const float coef = (float)(d.k_s * w[self] / (w[self] + w[q]));
                    const float f = (float)rl;
                    std::memcpy(rec + 4, &coef, 4);
                    std::memcpy(rec + 8, &f, 4);
                }
            }
        }
    }
    return out;
}

// ---------------------------------------------------------------------------
// compile_program: one CTA's program for a scene (or one part of a cluster program), in stages.
// Each stage reads the members the earlier ones set; every stage that can reject the input
// returns a status (err holds the message).
// ---------------------------------------------------------------------------
class ProgramCompiler {
public:
    ProgramCompiler(const ts_scene_desc &d_, const ts_layout_opts &o_, const PartSpec *part_, std::string &err_)
        : d(d_), o(o_), part(part_), err(err_) {}

    int run(std::vector<uint8_t> &blob, ts_layout_info &info) {
        int st;
        if ((st = validate()) != TS_OK) return st;
        live_constraints();
        local_set();
        if ((st = storage_order()) != TS_OK) return st;
        collect_items();
        if ((st = chunking()) != TS_OK) return st;
        schedule();
        if ((st = assign_slots()) != TS_OK) return st;
        emit_tables();
        compact_streams();
        if (eg) {   // owner-gathered edges (build_gather)
            GatherSpec gs{&d, &edge_live, &o2s, &s2o, &pc, [this](int v) { return own_free(v); },
                          [this](int v) { return is_free(v); }, Vf, Vf_pad, G, Vstore, R,
                          boff, compact, packed, o.schedule_banks >= 0};
            gp = build_gather(gs, static_cnt);
        }
        cluster_tables();
        wsplit = warp_split(chunk_rec, gp.evalence, eg, B, VPT, Vf);
        assemble(blob, info);
        return TS_OK;
    }

private:
    const ts_scene_desc &d;
    const ts_layout_opts &o;
    const PartSpec *part;
    std::string &err;

    int fail(int status, const char *msg) { err = msg; return status; }

    // ---- inputs -------------------------------------------------------------
    int V = 0, E = 0, T = 0, F = 0, A = 0, prec = 0, R = 4;
    const double *w = nullptr;
    bool eg = false;
    bool is_free(int v) const { return w[v] > 0.0; }
    // cluster part: this CTA of the env's cluster owns (updates, writes back) part->own vertices
    // and reads a halo of other parts' vertices, refreshed over DSMEM every substep
    bool own(int v) const { return !part || part->own[v] != 0; }
    bool own_free(int v) const { return is_free(v) && own(v); }

    int validate() {
        V = d.n_vert; E = d.n_edge; T = d.n_tet; F = d.n_face; A = d.n_att;
        prec = o.precision;
        if (prec != TS_F32 && prec != TS_F64) return fail(TS_ERR_INVALID, "precision must be TS_F32 or TS_F64");
        R = prec == TS_F64 ? 8 : 4;
        if (V < 0 || E < 0 || T < 0 || F < 0 || A < 0) return fail(TS_ERR_INVALID, "negative counts");
        if (V > 0 && (!d.positions_rest || !d.inverse_mass)) return fail(TS_ERR_INVALID, "missing vertex arrays");
        auto bad_vid = [&](int v) { return v < 0 || v >= V; };
        for (int i = 0; i < 2 * E; ++i) if (bad_vid(d.edges[i])) return fail(TS_ERR_INVALID, "edge vertex index out of range");
        for (int i = 0; i < 4 * T; ++i) if (bad_vid(d.tets[i])) return fail(TS_ERR_INVALID, "tet vertex index out of range");
        for (int i = 0; i < 3 * F; ++i) if (bad_vid(d.faces[i])) return fail(TS_ERR_INVALID, "face vertex index out of range");
        for (int i = 0; i < A; ++i) {
            if (bad_vid(d.att_vertex[i])) return fail(TS_ERR_INVALID, "attachment vertex out of range");
            if (d.att_is_face[i])
                for (int k = 0; k < 3; ++k)
                    if (bad_vid(d.att_faces[3 * i + k])) return fail(TS_ERR_INVALID, "attachment face vertex out of range");
        }
        w = d.inverse_mass;
        // edge_gather: distance constraints are gathered by the owner thread of each free vertex
        // (no phase-1 items, no slots); only attachments and tets go through slots
        // (the default; measured on B200, 4096 envs, reach_1170, with the gather done next to the
        // phase-1 tets: fp32 0.677 vs 0.949 ms/step, fp64 3.58 vs 3.64 ms/step)
        eg = part || o.edge_gather >= 0;
        return TS_OK;
    }

    // ---- live constraints and per-vertex incidence counts ---------------
    std::vector<int> inc, inc_e;
    std::vector<char> edge_live, att_live, tet_live;
    std::vector<double> att_wv, att_wc;

    void live_constraints() {
        inc.assign(V, 0); inc_e.assign(V, 0);
        edge_live.assign(E, 0); att_live.assign(A, 0); tet_live.assign(T, 0);
        for (int e = 0; e < E; ++e) {
            int a = d.edges[2 * e], b = d.edges[2 * e + 1];
            edge_live[e] = (w[a] + w[b]) > 0.0;  // _kernels.pyx:111 skips wsum <= 0
            if (edge_live[e]) { inc[a] += is_free(a); inc[b] += is_free(b); inc_e[a] += is_free(a); inc_e[b] += is_free(b); }
        }
        att_wv.assign(A, 0.0); att_wc.assign(A, 0.0);
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
    }

    // ---- local vertex set (parts: owned + halo) ---------------------------
    std::vector<char> local;
    std::vector<int> faces_local;
    int Floc = 0;
    bool local_tet(int t) const {
        if (!tet_live[t]) return false;
        if (!part) return true;
        for (int k = 0; k < 4; ++k) if (own_free(d.tets[4 * t + k])) return true;
        return false;
    }
    bool local_edge(int e) const {
        return edge_live[e] && (!part || own_free(d.edges[2 * e]) || own_free(d.edges[2 * e + 1]));
    }
    bool local_att(int i) const {
        if (!att_live[i]) return false;
        if (!part || own_free(d.att_vertex[i])) return true;
        if (d.att_is_face[i]) for (int k = 0; k < 3; ++k) if (own_free(d.att_faces[3 * i + k])) return true;
        return false;
    }

    void local_set() {
        local.assign(V, part ? 0 : 1);
        if (part) {
            for (int v = 0; v < V; ++v) if (own(v)) local[v] = 1;
            for (int e = 0; e < E; ++e) if (local_edge(e)) local[d.edges[2 * e]] = local[d.edges[2 * e + 1]] = 1;
            for (int t = 0; t < T; ++t) if (local_tet(t)) for (int k = 0; k < 4; ++k) local[d.tets[4 * t + k]] = 1;
            for (int i = 0; i < A; ++i) if (local_att(i)) {
                local[d.att_vertex[i]] = 1;
                if (d.att_is_face[i]) for (int k = 0; k < 3; ++k) local[d.att_faces[3 * i + k]] = 1;
            }
            faces_local = part->faces;
            for (int f : faces_local) for (int k = 0; k < 3; ++k) local[d.faces[3 * f + k]] = 1;
        } else {
            faces_local.resize(F);
            std::iota(faces_local.begin(), faces_local.end(), 0);
        }
        Floc = (int)faces_local.size();
    }

    // ---- storage order -------------------------------------------------
    int Vf = 0, Vf_pad = 0, Vown = 0, Vstore = 0, B = 0, VPT = 1, G = 0;
    PinCopies pc;
    std::vector<int> s2o, o2s;
    void place_copies() {   // s2o of the pinned copies from the primaries' (final) positions
        for (int p = Vf_pad; p < Vown; ++p)
            for (int j = 1; j < pc.n; ++j) s2o[pc.pos(p, j)] = s2o[p];
    }

    int storage_order() {
        // [owned free (cost-sorted) | pad | owned pinned | pad | halo (other parts' vertices) | pad]
        std::vector<int> free_v, pinned_v, halo_v;
        for (int v = 0; v < V; ++v) {
            if (!local[v]) continue;
            if (!own(v)) halo_v.push_back(v);
            else (is_free(v) ? free_v : pinned_v).push_back(v);
        }
        // warps own vertices of similar per-substep gather cost: an owner-gathered edge costs about
        // three slot reads (it recomputes the correction), a slot one
        std::vector<int> cost(V);
        for (int v = 0; v < V; ++v) cost[v] = eg ? inc[v] + 2 * inc_e[v] : inc[v];
        std::stable_sort(free_v.begin(), free_v.end(), [&](int a, int b) { return cost[a] > cost[b]; });
        Vf = (int)free_v.size();
        Vf_pad = roundup(Vf, 32);
        Vown = Vf_pad + roundup((int)pinned_v.size(), 32);
        // pinned copies (PinCopies): fp32 single-CTA gather programs with a bank schedule (TS_PIN_COPIES
        // overrides: 1, 2, 4 or 8)
        pc.Vf_pad = Vf_pad; pc.Vown = Vown; pc.Np_pad = Vown - Vf_pad;
        // (not for distance-only programs: the edges kernel is latency-bound and their coloured rounds
        // measured 8% slower, profiles/r02m config 2)
        if (prec == TS_F32 && !part && eg && o.schedule_banks >= 0 && pc.Np_pad > 0 && T > 0) pc.n = 4;
        if (const char *env = std::getenv("TS_PIN_COPIES")) {
            const int c = std::atoi(env);
            if (c == 1 || ((c == 2 || c == 4 || c == 8) && prec == TS_F32 && !part && pc.Np_pad > 0)) pc.n = c;
        }
        Vstore = Vown + roundup((int)halo_v.size(), 32) + (pc.n - 1) * pc.Np_pad;
        if (part && part->force_Vstore) {
            if (part->force_Vstore < Vstore) return fail(TS_ERR_INVALID, "forced Vstore too small");
            Vstore = part->force_Vstore;
        }
        s2o.assign(Vstore, -1); o2s.assign(V, -1);
        for (int i = 0; i < Vf; ++i) { s2o[i] = free_v[i]; o2s[free_v[i]] = i; }
        for (size_t i = 0; i < pinned_v.size(); ++i) { s2o[Vf_pad + i] = pinned_v[i]; o2s[pinned_v[i]] = Vf_pad + (int)i; }
        for (size_t i = 0; i < halo_v.size(); ++i) { s2o[Vown + i] = halo_v[i]; o2s[halo_v[i]] = Vown + (int)i; }
        place_copies();

        // fp32: one thread per free vertex (3 CTAs/SM fit); fp64 runs 1 CTA/SM (shared memory), so it
        // takes 1.5x the threads to widen phase 1 (measured on B200: 3.81 vs 4.30 ms at 4096 envs)
        // cluster parts: 1.5x too -- one env's CTAs run a few warps each and are latency-bound
        // fp64 programs of at most 320 free positions: one thread per vertex and two CTAs per SM
        // (step2_kernel) beat 1.5x threads at one CTA per SM
        const bool wide = (R == 8 && Vf_pad > 320) || part;
        B = o.block_threads > 0 ? o.block_threads
                                : std::min(512, std::max(64, wide ? roundup(Vf_pad * 3 / 2, 32) : Vf_pad));
        if (part && part->force_B) B = part->force_B;
        if (B % 32 != 0 || B < 32 || B > 512) return fail(TS_ERR_INVALID, "block_threads must be a multiple of 32 in [32, 512]");
        VPT = std::max(1, (Vf_pad + B - 1) / B);
        if (VPT > 8) return fail(TS_ERR_UNSUPPORTED, "mesh too large for one CTA per environment (more than 8 vertices per thread)");
        G = Vf_pad / 32;
        return TS_OK;
    }

    // ---- items per kind (constraint index order) -----------------------
    std::vector<Item> kinds[3];

    void collect_items() {
        auto P = [&](int v) { return o2s[v]; };
        for (int e = 0; e < E; ++e) if (local_edge(e)) {
            Item it{}; it.kind = TS_CHUNK_EDGE; it.index = e; it.nroles = 2;
            it.vid[0] = d.edges[2 * e]; it.vid[1] = d.edges[2 * e + 1];
            it.pos[0] = P(it.vid[0]); it.pos[1] = P(it.vid[1]);
            kinds[0].push_back(it);
        }
        for (int i = 0; i < A; ++i) if (local_att(i)) {
            Item it{}; it.kind = TS_CHUNK_ATT; it.index = i;
            it.vid[0] = d.att_vertex[i];
            it.pos[0] = P(it.vid[0]);
            if (d.att_is_face[i]) {
                it.nroles = 4;
                for (int k = 0; k < 3; ++k) { it.vid[1 + k] = d.att_faces[3 * i + k]; it.pos[1 + k] = P(it.vid[1 + k]); }
            } else it.nroles = 1;
            kinds[1].push_back(it);
        }
        for (int t = 0; t < T; ++t) if (local_tet(t)) {
            Item it{}; it.kind = TS_CHUNK_TET; it.index = t; it.nroles = 4;
            for (int k = 0; k < 4; ++k) { it.vid[k] = d.tets[4 * t + k]; it.pos[k] = P(it.vid[k]); }
            kinds[2].push_back(it);
        }
    }

    // ---- chunking by slot budget ---------------------------------------
    struct ChunkBuild { std::vector<Item> items; std::vector<int> val; std::vector<int> kmax; int padded; };
    std::vector<ChunkBuild> chunks;
    int budget = 0, n_chunks = 0, grasp_chunk = 0;

    int chunking() {
        // The reference's per-vertex accumulation order is the constraint sequence
        // [live edges..., grasp, live attachments..., live tets...].  Chunks are
        // contiguous ranges of that sequence (kinds may mix); the grasp is spliced
        // into the chunk where the edges end, after each vertex's edge slots.
        std::vector<Item> seq;
        for (int k = eg ? 1 : 0; k < 3; ++k) seq.insert(seq.end(), kinds[k].begin(), kinds[k].end());
        // slot budget per chunk: explicit, or what the CTA's shared memory leaves next to the positions
        budget = o.max_chunk_slots > 0 ? o.max_chunk_slots : (1 << 30);
        if (o.max_chunk_slots <= 0) {
            const int fixed = ts_smem_layout_bytes(Vstore, 0, Vf_pad, Floc, R, eg ? 1 : 0);
            const int avail = (TS_SMEM_LIMIT - fixed) / (3 * R) - 32;    // minus a margin of 32 slots
            if (avail < 7 * Floc || avail < 64)
                return fail(TS_ERR_UNSUPPORTED, "mesh too large for one CTA per environment (shared memory); use a cluster program");
            budget = avail;
        }
        size_t i = 0;
        while (i < seq.size()) {
            ChunkBuild c;
            c.val.assign(Vf_pad, 0); c.kmax.assign(G, 0); c.padded = 0;
            while (i < seq.size()) {
                const Item &it = seq[i];
                // default layout: a new chunk at every kind change (measured fastest on B200 for
                // reach_1170: 2 chunks at 3 CTAs/SM beat 1 mixed chunk at 2 CTAs/SM)
                if (!eg && o.max_chunk_slots == 0 && !c.items.empty() && c.items.back().kind != it.kind) break;
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
        n_chunks = (int)chunks.size();
        // grasp chunk: the chunk holding the first non-edge item (n_chunks if there is none)
        grasp_chunk = n_chunks;
        if (eg) grasp_chunk = 0;   // after the owner's edges, before any slot (gsplit = 0)
        else {
            const size_t n_edges = kinds[0].size();
            if (n_edges < seq.size()) {
                size_t pos = 0;
                for (int c = 0; c < n_chunks; ++c) {
                    if (n_edges < pos + chunks[c].items.size()) { grasp_chunk = c; break; }
                    pos += chunks[c].items.size();
                }
            }
        }
        return TS_OK;
    }

    // ---- phase-1 schedule (per chunk, per kind) ----------------------------
    bool packed = false;
    int bank_mod = 32, total_conf = 0;
    std::vector<TsChunk> chunk_rec;
    std::vector<Item> all_items[3];

    void schedule() {
        const bool sched = o.schedule_banks >= 0;
        const char *pack_env = std::getenv("TS_PACK_TETS");   // development switch: 0 = round-1 schedule
        packed = pc.n > 1 && sched && o.schedule_banks != 2 && (!pack_env || std::atoi(pack_env) != 0);
        bank_mod = (R == 8) ? 16 : 32;
        chunk_rec.assign(n_chunks, TsChunk{});
        for (int c = 0; c < n_chunks; ++c) {
            ChunkBuild &cb = chunks[c];
            TsChunk &r = chunk_rec[c];
            std::memset(&r, 0, sizeof(r));
            int begin[3], count[3];
            for (int k = 0; k < 3; ++k) {
                const int kind = k == 0 ? TS_CHUNK_EDGE : (k == 1 ? TS_CHUNK_ATT : TS_CHUNK_TET);
                std::vector<Item> part_items;
                for (const Item &it : cb.items) if (it.kind == kind) { part_items.push_back(it); part_items.back().chunk = c; }
                int conf = 0;
                // tets may get idle lanes (TS_TET_HOLES per 32-item batch) where no conflict-free
                // item is left; every tet still runs exactly once (off by default: slower on B200)
                // (packed programs re-batch their tets from scratch below: no greedy schedule for them)
                std::vector<Item> s = schedule_items(part_items, bank_mod, 32,
                                                     sched && kind != TS_CHUNK_ATT && !(packed && kind == TS_CHUNK_TET),
                                                     &conf, (kind == TS_CHUNK_TET && o.schedule_banks >= 0) ? g_tet_holes : 0);
                begin[k] = (int)all_items[k].size();
                count[k] = (int)s.size();
                all_items[k].insert(all_items[k].end(), s.begin(), s.end());
            }
            r.edge_begin = begin[0]; r.edge_count = count[0];
            r.att_begin = begin[1]; r.att_count = count[1];
            r.tet_begin = begin[2]; r.tet_count = count[2];
            r.region_off = c * G;
            r.val_off = c * Vf_pad;
        }
        if (packed) pack();
        // joint refinement: item order, vertex lanes inside each warp, role order (see bank_refine)
        if (sched && o.schedule_banks != 2 && !packed) refine();
        // final positions of every role (pinned corners: the copy they read)
        for (int k = 0; k < 3; ++k)
            for (Item &it : all_items[k])
                for (int r = 0; r < it.nroles; ++r) it.pos[r] = pc.pos(o2s[it.vid[r]], it.copy[r]);
        total_conf = 0;
        for (int c = 0; c < n_chunks; ++c) {
            TsChunk &r = chunk_rec[c];
            r.conflicts = batch_conflicts(all_items[0], r.edge_begin, r.edge_count, bank_mod) +
                          batch_conflicts(all_items[2], r.tet_begin, r.tet_count, bank_mod);
            total_conf += r.conflicts;
        }
    }

    // fp32 gather programs with pinned copies: lanes balanced for the owner edge gather, then tets
    // packed into conflict-free batches (balance_lanes, pack_tet_batches)
    void pack() {
        std::vector<std::vector<int>> nbrs(V);
        std::vector<int> tetval(V, 0);
        for (int e = 0; e < E; ++e) {
            if (!local_edge(e)) continue;
            const int a = d.edges[2 * e], b = d.edges[2 * e + 1];
            if (own_free(a)) nbrs[a].push_back(b);
            if (own_free(b)) nbrs[b].push_back(a);
        }
        for (const Item &it : kinds[2]) for (int r = 0; r < 4; ++r) if (is_free(it.vid[r])) tetval[it.vid[r]]++;
        int nb_tot = 0;
        for (int c = 0; c < n_chunks; ++c) nb_tot = std::max(nb_tot, (chunk_rec[c].tet_count + 31) / 32);
        balance_lanes(nbrs, tetval, o2s, s2o, Vf, 4 * nb_tot - 8);
        place_copies();
        std::vector<Item> tets_out;
        int resid = 0;
        for (int c = 0; c < n_chunks; ++c) {
            std::vector<Item> part_items;
            for (int i = 0; i < chunk_rec[c].tet_count; ++i) {
                const Item &it = all_items[2][chunk_rec[c].tet_begin + i];
                if (it.index >= 0) {
                    part_items.push_back(it);
                    part_items.back().sign = 1;
                    for (int r = 0; r < 4; ++r) part_items.back().copy[r] = 0;
                }
            }
            std::sort(part_items.begin(), part_items.end(), [](const Item &x, const Item &y) { return x.index < y.index; });
            for (Item &it : part_items) for (int r = 0; r < 4; ++r) it.vid[r] = d.tets[4 * it.index + r];   // reference corner order
            resid += pack_tet_batches(part_items, o2s, s2o, pc, Vstore);
            chunk_rec[c].tet_begin = (int)tets_out.size();
            chunk_rec[c].tet_count = (int)part_items.size();
            tets_out.insert(tets_out.end(), part_items.begin(), part_items.end());
        }
        all_items[2].swap(tets_out);
        if (std::getenv("TS_DEBUG_REFINE")) std::fprintf(stderr, "pack_tet_batches: residual %d\n", resid);
    }

    // the round-1 schedule: simulated-annealing refinement of item order, lanes and roles, then edges
    // by bipartite edge colouring
    void refine() {
        std::vector<ListRef> lists;
        for (int c = 0; c < n_chunks; ++c) {
            if (chunk_rec[c].edge_count) lists.push_back({&all_items[0], chunk_rec[c].edge_begin, chunk_rec[c].edge_count});
            if (chunk_rec[c].tet_count) lists.push_back({&all_items[2], chunk_rec[c].tet_begin, chunk_rec[c].tet_count});
        }
        bank_refine(lists, o2s, s2o, Vf, Vf_pad, Vown, bank_mod, /*permute_tets=*/R == 4, o.refine_iters, pc);
        place_copies();
        // edges: exact conflict-free batches by bipartite edge colouring (with the final positions)
        std::vector<Item> edges_out;
        for (int c = 0; c < n_chunks; ++c) {
            std::vector<Item> part_items(all_items[0].begin() + chunk_rec[c].edge_begin,
                                         all_items[0].begin() + chunk_rec[c].edge_begin + chunk_rec[c].edge_count);
            for (Item &it : part_items) for (int r = 0; r < it.nroles; ++r) it.pos[r] = o2s[it.vid[r]];
            std::vector<Item> colored = part_items;
            if (edge_coloring_schedule(colored, o2s, s2o, Vf_pad, bank_mod)) {
                for (Item &it : colored) for (int r = 0; r < it.nroles; ++r) it.pos[r] = o2s[it.vid[r]];
                if (batch_conflicts(colored, 0, (int)colored.size(), bank_mod) <
                    batch_conflicts(part_items, 0, (int)part_items.size(), bank_mod))
                    part_items.swap(colored);
            }
            chunk_rec[c].edge_begin = (int)edges_out.size();
            chunk_rec[c].edge_count = (int)part_items.size();
            edges_out.insert(edges_out.end(), part_items.begin(), part_items.end());
        }
        all_items[0].swap(edges_out);
    }

    // ---- slot assignment (reference per-vertex order, final positions) --------
    std::vector<int32_t> region, valence, static_cnt, gsplit;
    int slot_cap = 0, n_slots_total = 0;

    int assign_slots() {
        // Slots are numbered per vertex in the constraint sequence order (edges,
        // attachments, tets, each by index) whatever the phase-1 schedule is.
        region.assign((size_t)n_chunks * G, 0); valence.assign((size_t)n_chunks * Vf_pad, 0);
        static_cnt.assign(Vf_pad, 0); gsplit.assign(Vf_pad, 0);
        slot_cap = 0; n_slots_total = 0;
        for (int c = 0; c < n_chunks; ++c) {
            TsChunk &rec = chunk_rec[c];
            // items of this chunk in sequence order
            std::vector<Item *> seqc;
            for (int k = 0; k < 3; ++k) {
                const int b0 = k == 0 ? rec.edge_begin : (k == 1 ? rec.att_begin : rec.tet_begin);
                const int n0 = k == 0 ? rec.edge_count : (k == 1 ? rec.att_count : rec.tet_count);
                std::vector<Item *> part_items;
                for (int i = 0; i < n0; ++i) part_items.push_back(&all_items[k][b0 + i]);
                std::sort(part_items.begin(), part_items.end(), [](const Item *x, const Item *y) { return x->index < y->index; });
                seqc.insert(seqc.end(), part_items.begin(), part_items.end());
            }
            std::vector<int> kmax(G, 0), val(Vf_pad, 0);
            for (Item *it : seqc)
                for (int r = 0; r < it->nroles; ++r)
                    if (it->pos[r] < Vf_pad) { const int p = it->pos[r]; kmax[p / 32] = std::max(kmax[p / 32], ++val[p]); }
            int base = 0;
            for (int g = 0; g < G; ++g) { region[(size_t)c * G + g] = base; base += 32 * kmax[g]; }
            rec.slot_count = base;
            // pinned endpoints get no slot (-1: the kernel predicates that store off; every store then
            // has exactly one writer, so the step is clean under compute-sanitizer racecheck)
            slot_cap = std::max(slot_cap, base);
            std::vector<int> k_next(Vf_pad, 0);
            for (Item *it : seqc) {
                for (int r = 0; r < it->nroles; ++r) {
                    const int p = it->pos[r];
                    if (p >= Vf_pad) { it->slot[r] = -1; continue; }
                    it->slot[r] = region[(size_t)c * G + p / 32] + 32 * k_next[p] + (p % 32);
                    k_next[p]++;
                    if (c == grasp_chunk && it->kind == TS_CHUNK_EDGE) gsplit[p] = k_next[p];
                }
            }
            for (int p = 0; p < Vf_pad; ++p) {
                valence[(size_t)c * Vf_pad + p] = k_next[p];
                static_cnt[p] += k_next[p];
                n_slots_total += k_next[p];
            }
        }
        // contact records reuse the slot buffer: 3F records x 7 reals <= 3 arrays x S reals
        slot_cap = std::max(slot_cap, 7 * Floc);
        slot_cap = roundup(std::max(slot_cap, 32), 32);
        if (part && part->force_slot_cap) {
            if (part->force_slot_cap < slot_cap) return fail(TS_ERR_INVALID, "forced slot capacity too small");
            slot_cap = part->force_slot_cap;
        }
        return TS_OK;
    }

    // ---- emit: the full (uncompressed) tables ----------------------------------
    int nE = 0, nA = 0, nT = 0;
    std::vector<int32_t> edge_idx, tet_idx, tet_slot, att_idx, att_slot;
    std::vector<double> edge_par, tet_rv, att_par, att_anc, wst, rest;
    std::vector<int32_t> faces_s, faces_o, face_gid;

    void emit_tables() {
        nE = (int)all_items[0].size(); nA = (int)all_items[1].size(); nT = (int)all_items[2].size();
        edge_idx.assign(4 * (size_t)nE, 0); tet_idx.assign(4 * (size_t)nT, 0); tet_slot.assign(4 * (size_t)nT, 0);
        att_idx.assign(4 * (size_t)nA, 0); att_slot.assign(4 * (size_t)nA, 0);
        edge_par.assign(4 * (size_t)nE, 0.0); tet_rv.assign(nT, 0.0);
        att_par.assign(4 * (size_t)nA, 0.0); att_anc.assign(4 * (size_t)nA, 0.0);
        for (int i = 0; i < nE; ++i) {
            const Item &it = all_items[0][i];
            const int a = it.vid[0], b = it.vid[1];   // roles may be swapped by the bank refinement
            edge_idx[4 * i + 0] = it.pos[0]; edge_idx[4 * i + 1] = it.pos[1];
            edge_idx[4 * i + 2] = it.slot[0]; edge_idx[4 * i + 3] = it.slot[1];
            if (it.index < 0) {   // padding lane of a colour class: pinned endpoints, no slot
                edge_par[4 * i + 0] = 0.0; edge_par[4 * i + 1] = 0.0; edge_par[4 * i + 2] = 0.0;
                edge_par[4 * i + 3] = 1.0;
                continue;
            }
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
            if (it.index < 0) {   // idle lane of a batch: slot -1 (compact: 0xffff) tells the kernel to skip it
                for (int k = 0; k < 4; ++k) { tet_idx[4 * i + k] = 0; tet_slot[4 * i + k] = -1; }
                tet_rv[i] = 0.0;
                continue;
            }
            for (int k = 0; k < 4; ++k) { tet_idx[4 * i + k] = it.pos[k]; tet_slot[4 * i + k] = it.slot[k]; }
            // fp32 build works with unscaled cross products G = 6 grad: it needs 6 V0
            tet_rv[i] = R == 8 ? d.rest_volume[it.index] : it.sign * 6.0 * d.rest_volume[it.index];
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
        wst.assign(Vstore, 0.0);
        for (int p = 0; p < Vstore; ++p) if (s2o[p] >= 0) wst[p] = w[s2o[p]];
        faces_s.assign(3 * (size_t)Floc, 0); faces_o.assign(3 * (size_t)Floc, 0); face_gid.assign(Floc, 0);
        for (int i = 0; i < Floc; ++i) {
            const int f = faces_local[i];
            face_gid[i] = f;
            for (int k = 0; k < 3; ++k) { faces_o[3 * i + k] = d.faces[3 * f + k]; faces_s[3 * i + k] = o2s[d.faces[3 * f + k]]; }
        }
        rest.assign(3 * (size_t)V, 0.0);
        for (int i = 0; i < 3 * V; ++i) rest[i] = d.positions_rest[i];
    }

    // ---- compact 16-bit item streams ---------------------------------------
    double w_free = 0.0;
    bool compact = false, boff = false, narrow = false;
    std::vector<float> rv_tab;
    std::vector<uint32_t> edge_c, tet_c;

    void compact_streams() {
        // Every mesh built by load_scene has one inverse mass for all free vertices
        // (mesh.py:217: uniform mass), so an edge needs only its rest length: the
        // per-endpoint weights follow from which endpoints are pinned.
        bool uniform = true;
        w_free = 0.0;
        for (int v = 0; v < V; ++v)
            if (is_free(v)) {
                if (w_free == 0.0) w_free = w[v];
                else if (w[v] != w_free) uniform = false;
            }
        compact = o.compact >= 0 && uniform && Vstore <= 65535 && slot_cap <= 65535;
        // fp32 gather programs: the compact tet stream and the edge records carry BYTE offsets
        // (12 x position / slot index) so the kernel addresses shared memory without multiplies;
        // the streams are padded by one CTA's worth of zero items so prefetches need no clamp
        boff = compact && eg && R == 4 && 12 * Vstore <= 65535 && 12 * slot_cap <= 65535;
        const int scale_b = boff ? 12 : 1;
        // narrow layout (program.h): legal when nothing reads neighbour positions in phase 2 (the
        // distance-only program gathers edges there) and no cluster peer reads the ping-pong copy.
        // Narrow programs put the positions first, so byte-offset streams address positions and
        // slots from ONE base (slot offsets carry + 12 Vstore) -- which must fit the 16-bit fields
        {
            int maxval = 0;
            for (int v : valence) maxval = std::max(maxval, v);
            const char *nv = std::getenv("TS_NARROW");
            // (distance-only gather programs stay wide: a narrow one needs a second barrier between the
            // gather and the in-place apply, measured slower even at 4 CTAs / SM, profiles/r02j)
            narrow = !part && (n_chunks >= 1 || !eg) && maxval <= 255 && !(nv && nv[0] == '0') &&
                     (!boff || 12 * (Vstore + slot_cap) < 65535);
        }
        const int slot_b0 = (narrow && boff) ? 12 * Vstore : 0;
        // rest volumes as a dictionary index in the spare top bits of the four 16-bit position
        // offsets (2 bits each; needs 12 Vstore < 16384) when few distinct 6 V0 values exist
        std::vector<int> rv_idx(nT, 0);
        if (boff && 12 * Vstore < 16384) {
            std::vector<float> vals;
            for (int i = 0; i < nT; ++i) if (all_items[2][i].index >= 0) vals.push_back((float)tet_rv[i]);
            std::sort(vals.begin(), vals.end());
            vals.erase(std::unique(vals.begin(), vals.end()), vals.end());
            if (!vals.empty() && (int)vals.size() <= 256) {
                rv_tab = vals;
                for (int i = 0; i < nT; ++i)
                    if (all_items[2][i].index >= 0)
                        rv_idx[i] = (int)(std::lower_bound(vals.begin(), vals.end(), (float)tet_rv[i]) - vals.begin());
            }
        }
        edge_c.assign(compact ? 4 * (size_t)nE : 0, 0);
        tet_c.assign(compact ? 4 * ((size_t)nT + B) : 0, 0);
        if (!compact) return;
        auto pk = [](int lo, int hi) { return (uint32_t)(lo & 0xffff) | ((uint32_t)(hi & 0xffff) << 16); };
        for (int i = 0; i < nE; ++i) {
            edge_c[4 * i + 0] = pk(edge_idx[4 * i + 0], edge_idx[4 * i + 1]);
            edge_c[4 * i + 1] = pk(edge_idx[4 * i + 2], edge_idx[4 * i + 3]);
            const double rl = edge_par[4 * i + 0];
            if (R == 8) { std::memcpy(&edge_c[4 * i + 2], &rl, 8); }
            else { const float f = (float)rl; std::memcpy(&edge_c[4 * i + 2], &f, 4); edge_c[4 * i + 3] = 0; }
        }
        for (int i = 0; i < nT; ++i) {
            // an idle lane (dummy item) reads the corner "Vf_pad" -- never a free vertex, so even if it
            // is executed it touches no degenerate counter; its slot fields are all absent
            const Item &ti = all_items[2][i];
            const bool idle = ti.index < 0 && boff;
            auto po = [&](int k) { return idle ? scale_b * (ti.idle_pos ? ti.pos[k] : Vf_pad) : scale_b * tet_idx[4 * i + k]; };
            tet_c[4 * i + 0] = pk(po(0), po(1));
            tet_c[4 * i + 1] = pk(po(2), po(3));
            if (!rv_tab.empty()) {   // index bits 2k, 2k+1 in bits 14-15 of 16-bit field k
                const uint32_t r = (uint32_t)rv_idx[i];
                tet_c[4 * i + 0] |= ((r & 3u) << 14) | (((r >> 2) & 3u) << 30);
                tet_c[4 * i + 1] |= (((r >> 4) & 3u) << 14) | (((r >> 6) & 3u) << 30);
            }
            // slot fields: byte offsets (boff) or indices; 0xffff = no slot (pinned corner; all four:
            // an idle lane of the bank schedule) -- never a multiple of 12 nor a valid index
            auto so = [&](int s) { return s < 0 ? 0xffff : slot_b0 + scale_b * s; };
            tet_c[4 * i + 2] = pk(so(tet_slot[4 * i + 0]), so(tet_slot[4 * i + 1]));
            tet_c[4 * i + 3] = pk(so(tet_slot[4 * i + 2]), so(tet_slot[4 * i + 3]));
        }
    }

    // ---- owner-gathered edges, cluster tables, warp split ------------------------
    GatherProgram gp;
    std::vector<int32_t> send_off, send, face_own, wsplit;

    // cluster part: halo sends and face-vertex owners
    void cluster_tables() {
        if (!(part && part->halo_of)) return;
        send_off.assign(Vf_pad + 1, 0);
        for (int p = 0; p < Vf_pad; ++p) {
            if (p < Vf)
                for (const auto &rp : (*part->halo_of)[s2o[p]]) send.push_back((rp.first << 20) | rp.second);
            send_off[p + 1] = (int32_t)send.size();
        }
        face_own.assign(3 * (size_t)Floc, -1);
        for (int i = 0; i < 3 * Floc; ++i) {
            const int v = faces_o[i];
            if (is_free(v)) face_own[i] = ((*part->owner_rank)[v] << 20) | (*part->owner_pos)[v];
        }
    }

    // ---- the blob: header + 256-byte aligned sections ------------------------------
    void assemble(std::vector<uint8_t> &blob, ts_layout_info &info) {
        const std::vector<float> &pair_tab = gp.pair_tab;
        int64_t sz[TS_SEC_COUNT];
        sz[TS_SEC_CHUNK] = (int64_t)n_chunks * sizeof(TsChunk);
        sz[TS_SEC_EDGE_IDX] = 16LL * nE;
        sz[TS_SEC_EDGE_PAR] = 4LL * R * nE;
        sz[TS_SEC_TET_IDX] = 16LL * nT;
        sz[TS_SEC_TET_SLOT] = 16LL * nT;
        sz[TS_SEC_TET_RV] = (int64_t)R * (nT + B);   // padded like the compact stream
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
        sz[TS_SEC_FACES] = 12LL * Floc;
        sz[TS_SEC_FACES_ORIG] = 12LL * Floc;
        sz[TS_SEC_REST] = 3LL * R * V;
        sz[TS_SEC_GSPLIT] = 4LL * Vf_pad;
        sz[TS_SEC_EDGE_C] = 4LL * edge_c.size();
        sz[TS_SEC_TET_C] = 4LL * tet_c.size();
        sz[TS_SEC_EINC] = (int64_t)gp.einc.size();
        sz[TS_SEC_EREGION] = 4LL * gp.eregion.size();
        sz[TS_SEC_EVAL] = 4LL * gp.evalence.size();
        sz[TS_SEC_FACE_GID] = 4LL * face_gid.size();
        sz[TS_SEC_SEND_OFF] = 4LL * send_off.size();
        sz[TS_SEC_SEND] = 4LL * send.size();
        sz[TS_SEC_FACE_OWN] = 4LL * face_own.size();
        sz[TS_SEC_WSPLIT] = 4LL * wsplit.size();
        sz[TS_SEC_RLTAB] = 4LL * pair_tab.size();
        sz[TS_SEC_RVTAB] = 4LL * rv_tab.size();
        TsProgHeader hdr{};
        hdr.compact = compact ? 1 : 0;
        hdr.w_free = w_free;
        hdr.magic = TS_PROG_MAGIC; hdr.version = TS_PROG_VERSION; hdr.real_bytes = R; hdr.n_sections = TS_SEC_COUNT;
        hdr.V = V; hdr.Vf = Vf; hdr.Vf_pad = Vf_pad; hdr.Vstore = Vstore;
        hdr.F = Floc; hdr.B = B; hdr.VPT = VPT; hdr.G = G;
        hdr.Vown = Vown; hdr.cluster_k = part ? part->K : 1; hdr.cluster_rank = part ? part->rank : 0;
        hdr.boff = boff ? 1 : 0;
        hdr.rvdict = rv_tab.empty() ? 0 : 1;
        hdr.n_rltab = (int)pair_tab.size() / 2; hdr.n_rvtab = (int)rv_tab.size();
        hdr.n_chunks = n_chunks; hdr.grasp_chunk = grasp_chunk; hdr.slot_capacity = slot_cap; hdr.n_att = nA;
        hdr.n_edge_items = nE; hdr.n_tet_items = nT; hdr.n_att_items = nA; hdr.bank_conflicts = total_conf;
        hdr.n_slots_total = n_slots_total;
        hdr.edge_gather = eg ? 1 : 0; hdr.einc_bytes = gp.einc_bytes;
        hdr.narrow = narrow ? 1 : 0;
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
        put(blob, hdr.off[TS_SEC_EINC], gp.einc);
        put(blob, hdr.off[TS_SEC_EREGION], gp.eregion);
        put(blob, hdr.off[TS_SEC_EVAL], gp.evalence);
        put(blob, hdr.off[TS_SEC_FACE_GID], face_gid);
        put(blob, hdr.off[TS_SEC_SEND_OFF], send_off);
        put(blob, hdr.off[TS_SEC_SEND], send);
        put(blob, hdr.off[TS_SEC_FACE_OWN], face_own);
        put(blob, hdr.off[TS_SEC_WSPLIT], wsplit);
        put(blob, hdr.off[TS_SEC_RLTAB], pair_tab);
        put(blob, hdr.off[TS_SEC_RVTAB], rv_tab);
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
        info.edge_gather = eg ? 1 : 0; info.n_edge_incidences = gp.n_einc;
        info.slot_budget = budget; info.cluster_size = part ? part->K : 1;
    }
};

}  // namespace

int compile_program(const ts_scene_desc &d, const ts_layout_opts &o, std::vector<uint8_t> &blob,
                    ts_layout_info &info, std::string &err, const PartSpec *part) {
    if (part && (int)part->own.size() != d.n_vert) { err = "part ownership mask size"; return TS_ERR_INVALID; }
    g_search_effort = part ? 0.1 : 1.0;
    g_tet_holes = 0;   // measured: 2-8 idle lanes per batch cut conflicts but cost more issue (slower)
    if (const char *env = std::getenv("TS_TET_HOLES")) g_tet_holes = std::atoi(env);
    ProgramCompiler pc(d, o, part, err);
    return pc.run(blob, info);
}


// ---------------------------------------------------------------------------
// cluster programs (large meshes): K parts, one per CTA of an env's cluster
// ---------------------------------------------------------------------------
namespace {

// recursive coordinate bisection of the free vertices (balanced counts, compact parts)
void rcb(const double *X, std::vector<int> &idx, int lo, int hi, int part0, int nparts, std::vector<int> &part_of) {
    if (nparts <= 1 || hi - lo <= 1) {
        for (int i = lo; i < hi; ++i) part_of[idx[i]] = part0;
        return;
    }
    double mn[3] = {1e300, 1e300, 1e300}, mx[3] = {-1e300, -1e300, -1e300};
    for (int i = lo; i < hi; ++i)
        for (int c = 0; c < 3; ++c) { mn[c] = std::min(mn[c], X[3 * idx[i] + c]); mx[c] = std::max(mx[c], X[3 * idx[i] + c]); }
    int axis = 0;
    for (int c = 1; c < 3; ++c) if (mx[c] - mn[c] > mx[axis] - mn[axis]) axis = c;
    std::stable_sort(idx.begin() + lo, idx.begin() + hi, [&](int a, int b) {
        const double xa = X[3 * a + axis], xb = X[3 * b + axis];
        return xa < xb || (xa == xb && a < b);
    });
    const int left = nparts / 2;
    const int mid = lo + (int)((int64_t)(hi - lo) * left / nparts);
    rcb(X, idx, lo, mid, part0, left, part_of);
    rcb(X, idx, mid, hi, part0 + left, nparts - left, part_of);
}

const int32_t *prog_section(const std::vector<uint8_t> &blob, int sec) {
    const TsProgHeader *H = reinterpret_cast<const TsProgHeader *>(blob.data());
    return reinterpret_cast<const int32_t *>(blob.data() + H->off[sec]);
}

}  // namespace

int compile_cluster(const ts_scene_desc &d, const ts_layout_opts &o_in, int K, std::vector<uint8_t> &blob,
                    ts_layout_info &info, std::string &err) {
    const int V = d.n_vert, E = d.n_edge, F = d.n_face;
    if (V <= 0) { err = "cluster programs need vertices"; return TS_ERR_INVALID; }
    for (int i = 0; i < 2 * E; ++i) if (d.edges[i] < 0 || d.edges[i] >= V) { err = "edge vertex index out of range"; return TS_ERR_INVALID; }
    for (int i = 0; i < 3 * F; ++i) if (d.faces[i] < 0 || d.faces[i] >= V) { err = "face vertex index out of range"; return TS_ERR_INVALID; }
    const int R = o_in.precision == TS_F64 ? 8 : 4;
    std::vector<int> tries;
    if (K == 0) tries = {2, 4, 8, 16};
    else tries = {K};
    std::string last_err = "no cluster size fits";
    for (int k : tries) {
        if (k < 2 || k > TS_MAX_CLUSTER) { err = "cluster size must be in [2, 16]"; return TS_ERR_INVALID; }
        // ---- partition: free vertices by RCB, pinned ones follow a free neighbour -------
        const double *w = d.inverse_mass;
        std::vector<int> part_of(V, 0), freev;
        for (int v = 0; v < V; ++v) if (w[v] > 0.0) freev.push_back(v);
        rcb(d.positions_rest, freev, 0, (int)freev.size(), 0, k, part_of);
        std::vector<char> placed(V, 0);
        for (int v : freev) placed[v] = 1;
        for (int e = 0; e < E; ++e) {   // first edge (by index) to a free vertex decides a pinned vertex
            const int a = d.edges[2 * e], b = d.edges[2 * e + 1];
            if (!placed[a] && placed[b] && w[b] > 0.0) { part_of[a] = part_of[b]; placed[a] = 2; }
            if (!placed[b] && placed[a] && w[a] > 0.0) { part_of[b] = part_of[a]; placed[b] = 2; }
        }
        std::vector<PartSpec> ps(k);
        for (int r = 0; r < k; ++r) {
            ps[r].rank = r; ps[r].K = k;
            ps[r].own.assign(V, 0);
        }
        for (int v = 0; v < V; ++v) ps[part_of[v]].own[v] = 1;
        for (int f = 0; f < F; ++f) {   // a face goes to the owner of its first free vertex
            int r = part_of[d.faces[3 * f]];
            for (int j = 0; j < 3; ++j) if (w[d.faces[3 * f + j]] > 0.0) { r = part_of[d.faces[3 * f + j]]; break; }
            ps[r].faces.push_back(f);
        }
        // ---- pass 1: natural sizes, storage orders ------------------------------------
        // (again with a common slot budget if the parts' largest sizes together overflow)
        ts_layout_opts o = o_in;
        std::vector<std::vector<uint8_t>> blobs(k);
        std::vector<ts_layout_info> infos(k);
        bool ok = true;
        int maxB = 0, maxVs = 0, maxSl = 0;
        for (int attempt = 0; attempt < 2; ++attempt) {
            ok = true;
            for (int r = 0; r < k && ok; ++r) {
                std::string e2;
                if (compile_program(d, o, blobs[r], infos[r], e2, &ps[r]) != TS_OK) { ok = false; last_err = e2; }
            }
            if (!ok) break;
            maxB = maxVs = maxSl = 0;
            int maxVfp = 0, maxF = 0;
            for (int r = 0; r < k; ++r) {
                const TsProgHeader *H = reinterpret_cast<const TsProgHeader *>(blobs[r].data());
                maxB = std::max(maxB, infos[r].block_threads);
                maxVs = std::max(maxVs, infos[r].n_store);
                maxSl = std::max(maxSl, infos[r].slot_capacity);
                maxVfp = std::max(maxVfp, H->Vf_pad);
                maxF = std::max(maxF, H->F);
            }
            if (ts_smem_layout_bytes(maxVs, maxSl, maxVfp, maxF, R, 1) <= TS_SMEM_LIMIT) break;
            ok = false;
            last_err = "cluster part exceeds shared memory";
            const int fixed = ts_smem_layout_bytes(maxVs, 0, maxVfp, maxF, R, 1);
            const int common = (TS_SMEM_LIMIT - fixed) / (3 * R) - 32 - 32 * 64;   // margin: region padding
            if (common < 7 * maxF || common < 256) break;
            o.max_chunk_slots = common;
        }
        if (!ok) continue;
        std::vector<std::vector<int>> o2s(k);
        std::vector<int> owner_rank(V, -1), owner_pos(V, -1);
        std::vector<std::vector<std::pair<int, int>>> halo_of(V);
        for (int r = 0; r < k; ++r) {
            const int32_t *q = prog_section(blobs[r], TS_SEC_O2S);
            o2s[r].assign(q, q + V);
            for (int v = 0; v < V; ++v) {
                if (o2s[r][v] < 0) continue;
                if (ps[r].own[v]) { owner_rank[v] = r; owner_pos[v] = o2s[r][v]; }
                else halo_of[v].push_back({r, o2s[r][v]});
            }
        }
        // ---- pass 2: common layout sizes + halo sends / face owners ---------------------
        for (int r = 0; r < k && ok; ++r) {
            ps[r].force_B = maxB; ps[r].force_Vstore = maxVs; ps[r].force_slot_cap = maxSl;
            ps[r].halo_of = &halo_of; ps[r].owner_rank = &owner_rank; ps[r].owner_pos = &owner_pos;
            ts_layout_opts o2 = o;
            o2.max_chunk_slots = infos[r].slot_budget;   // the same chunking as pass 1
            std::string e2;
            if (compile_program(d, o2, blobs[r], infos[r], e2, &ps[r]) != TS_OK) { ok = false; last_err = e2; break; }
            const int32_t *q = prog_section(blobs[r], TS_SEC_O2S);
            if (!std::equal(q, q + V, o2s[r].begin())) { err = "cluster part storage order changed between passes"; return TS_ERR_INVALID; }
        }
        if (!ok) continue;
        // ---- assemble ---------------------------------------------------------------------
        TsClusterHeader ch{};
        ch.magic = TS_CLUSTER_MAGIC; ch.K = k; ch.n_vert = V; ch.n_face = F;
        int64_t off = ((int64_t)sizeof(TsClusterHeader) + 255) / 256 * 256;
        for (int r = 0; r < k; ++r) {
            ch.part_off[r] = off; ch.part_bytes[r] = (int64_t)blobs[r].size();
            off += ((int64_t)blobs[r].size() + 255) / 256 * 256;
        }
        ch.total_bytes = off;
        blob.assign((size_t)off, 0);
        std::memcpy(blob.data(), &ch, sizeof(ch));
        for (int r = 0; r < k; ++r) std::memcpy(blob.data() + ch.part_off[r], blobs[r].data(), blobs[r].size());
        info = infos[0];
        int nfree = 0, nslots = 0, ninc = 0;
        for (int r = 0; r < k; ++r) { nfree += infos[r].n_free; nslots += infos[r].n_slots_total; ninc += infos[r].n_edge_incidences; }
        info.n_free = nfree; info.n_slots_total = nslots; info.n_edge_incidences = ninc;
        info.cluster_size = k; info.program_bytes = off;
        return TS_OK;
    }
    err = last_err;
    return TS_ERR_UNSUPPORTED;
}

}  // namespace ts
