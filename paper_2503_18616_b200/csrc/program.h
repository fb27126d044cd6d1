// program.h -- compiled scene program shared by the host compiler and the
// sm_100a kernels.  One flat blob: a header with byte offsets of typed
// sections.  Uploaded once per handle; every CTA (one environment each)
// reads the same blob through L1/L2.
//
// Vertex "storage positions": free vertices (w > 0) first, sorted by
// incidence count (descending) so each warp owns vertices of similar
// valence; then pinned vertices.  The owner thread of free position p is
// p % B (B = CTA size, a multiple of 32), so its lane is p % 32.  Shared
// memory arrays indexed by p therefore place p in bank p % 32.
//
// Constraint "slots": every (constraint, free endpoint) incidence owns one
// slot in the chunk's slot buffer.  The slots of free position p in chunk c
// are region(c, p/32) + k*32 + p%32 for k = 0..valence(c,p)-1, in the
// reference's per-vertex accumulation order (constraint index, then role),
// so the owner's sequential sum reproduces _kernels.pyx's accumulation
// order exactly (edges -> grasp -> attachments -> tets, each by index).
#pragma once
#include <stdint.h>

#define TS_PROG_MAGIC 0x54534231  // "TSB1"
#define TS_PROG_VERSION 4

enum TsChunkKind { TS_CHUNK_EDGE = 0, TS_CHUNK_ATT = 1, TS_CHUNK_TET = 2 };

enum TsSection {
    TS_SEC_CHUNK = 0,     // TsChunk[n_chunks]
    TS_SEC_EDGE_IDX,      // int4 {pa, pb, sa, sb}   storage pos, slot (-1: pinned endpoint)
    TS_SEC_EDGE_PAR,      // Real4 {rest_len, wa, wb, wsum}
    TS_SEC_TET_IDX,       // int4 {pa, pb, pc, pd}
    TS_SEC_TET_SLOT,      // int4 {sa, sb, sc, sd}
    TS_SEC_TET_RV,        // Real rest volume
    TS_SEC_ATT_IDX,       // int4 {vtx, f0, f1, f2}
    TS_SEC_ATT_SLOT,      // int4 slots of vtx, f0, f1, f2
    TS_SEC_ATT_PAR,       // Real4 {rest, k, wv, wc}
    TS_SEC_ATT_ANCHOR,    // Real4 {ax, ay, az, is_face}
    TS_SEC_REGION,        // int32 [n_chunks][G] base slot of group g's region
    TS_SEC_VALENCE,       // int32 [n_chunks][Vf_pad]
    TS_SEC_STATIC_CNT,    // int32 [Vf_pad] total incidences over all chunks
    TS_SEC_S2O,           // int32 [Vstore] storage pos -> original vertex (-1 padding)
    TS_SEC_O2S,           // int32 [V] original vertex -> storage pos
    TS_SEC_W,             // Real [Vstore] inverse mass (0 for padding)
    TS_SEC_FACES,         // int32 [F][3] surface faces in storage positions
    TS_SEC_FACES_ORIG,    // int32 [F][3] surface faces, original ids (plugin outputs)
    TS_SEC_REST,          // Real [V][3] rest positions, original order (reset)
    TS_SEC_GSPLIT,        // int32 [Vf_pad] slots of p in the grasp chunk that precede the grasp
    // compact 16-bit item streams (uniform free-vertex mass, < 65536 positions / slots):
    // the whole phase-1 stream of reach_1170 fits in L1 and is shared by every CTA on an SM
    TS_SEC_EDGE_C,        // uint4 {pa | pb << 16, sa | sb << 16, rest (fp32 bits | fp64 lo), fp64 hi}
    TS_SEC_TET_C,         // uint4 {pa | pb << 16, pc | pd << 16, sa | sb << 16, sc | sd << 16}
    // owner-gathered distance constraints (edge_gather programs): every free vertex walks its own
    // incident edges in edge-index order and recomputes each correction from the position
    // snapshot, so edges need neither phase-1 items nor slots nor a barrier of their own
    TS_SEC_EINC,          // records, warp-interleaved like slots: incidence k of lane l at
                          //   eregion[g] + 32k + l.  einc_bytes = 8: {nbr pos, fp32 rest}
                          //   (uniform-mass fp32); 16: {nbr pos, fp32 coef | 0, fp64/fp32 rest}
    TS_SEC_EREGION,       // int32 [G] base record of group g
    TS_SEC_EVAL,          // int32 [Vf_pad] live incident edges of p
    TS_SEC_FACE_GID,      // int32 [F] global surface-face index of local face i (contact order key)
    // cluster parts only (one CTA of an env's thread-block cluster):
    TS_SEC_SEND_OFF,      // int32 [Vf_pad + 1] CSR offsets of the halo sends of owned free vertex p
    TS_SEC_SEND,          // int32 [n] (dest rank << 20) | dest storage position
    TS_SEC_FACE_OWN,      // int32 [F][3] (owner rank << 20) | owner position of a free face vertex, -1 pinned
    // phase-1 work split: int32 [n_chunks][B/32 + 1] first tet item of each warp (relative to the
    // chunk).  Contiguous ranges of 32-item batches, sized so that a warp's owner edge gather
    // (done in phase 1 of chunk 0, it needs only the position snapshot) plus its tet items is
    // about the same for every warp
    TS_SEC_WSPLIT,
    TS_SEC_RLTAB,         // float [] distinct rest lengths (4-byte edge records index it)
    TS_SEC_RVTAB,         // float [] distinct 6 V0 values (rvdict programs: index in the tet stream)
    TS_SEC_COUNT
};

// A chunk is a contiguous range of the reference's constraint sequence
// [edges..., attachments..., tets...]; it may hold items of all three kinds.
struct TsChunk {
    int32_t edge_begin, edge_count, att_begin, att_count;
    int32_t tet_begin, tet_count, slot_count, region_off;
    int32_t val_off, conflicts, pad0, pad1;
};

#define TS_SMEM_HEAD 1792       // [scalars + capsules: 1280 | rest-length table | 6V0 table]
#define TS_TAB_OFF 1280         // the two dictionary tables of fast programs, TS_TAB_CAP floats each
#define TS_TAB_CAP 64       // scalar block + capsule parameters, at the start of shared memory

// Shared memory one CTA needs for a program (the kernel's carve, step_kernel.cuh): positions
// (x2 when ping-ponged), slot buffer / contact records, degenerate counters, contact bitmap,
// scalar block.
// narrow programs (single CTA, >= 1 chunk, every chunk valence <= 255): phase 2 writes positions in
// place (nothing reads a neighbour's position after the phase-1 barrier) and the degenerate-constraint
// counters are bytes -- 6 KB less per CTA for reach_1170.  Layout order: narrow [head | positions |
// slots | counters | bitmap] (one base for both, byte-offset slot fields carry + 12 Vstore); wide
// [head | slots | positions | ping-pong | counters | bitmap] (slots at a constant offset in every
// CTA of a cluster)
inline int ts_smem_layout_bytes(int Vstore, int slot_cap, int Vf_pad, int F, int real_bytes, int ping_pong,
                                int narrow = 0) {
    size_t b = 0;
    b += (size_t)3 * Vstore * real_bytes * (ping_pong && !narrow ? 2 : 1);
    b += (size_t)3 * slot_cap * real_bytes;
    b += (size_t)(narrow ? 1 : 4) * Vf_pad;
    b += (size_t)4 * ((3 * F + 31) / 32);
    b = (b + 15) / 16 * 16;
    b += TS_SMEM_HEAD;
    return (int)b;
}
#define TS_SMEM_LIMIT 232448   // B200 opt-in shared memory per CTA (227 KiB)

// A cluster program: K part programs, one per CTA rank of an environment's cluster.
#define TS_CLUSTER_MAGIC 0x54534331  // "TSC1"
#define TS_MAX_CLUSTER 16
struct TsClusterHeader {
    int32_t magic, K, n_vert, n_face;
    int64_t part_off[TS_MAX_CLUSTER], part_bytes[TS_MAX_CLUSTER];
    int64_t total_bytes;
};

struct TsProgHeader {
    int32_t magic, version, real_bytes, n_sections;
    int32_t V, Vf, Vf_pad, Vstore;
    int32_t F, B, VPT, G;
    int32_t n_chunks, grasp_chunk, slot_capacity, n_att;
    int32_t n_edge_items, n_tet_items, n_att_items, bank_conflicts;
    int32_t n_slots_total, compact, edge_gather, einc_bytes;
    int32_t Vown, cluster_k, cluster_rank, boff;   // Vown: end of the owned (written-back) positions;
                                                   // boff: fp32 compact streams hold byte offsets
    int32_t rvdict, narrow;                        // rvdict: tet rest volumes dictionary-coded;
                                                   // narrow: one position buffer, 8-bit degenerate counters
    int32_t n_rltab, n_rvtab;                      // dictionary sizes (RLTAB / RVTAB entries)
    double w_free;   // the common inverse mass of free vertices (compact programs)
    int64_t off[TS_SEC_COUNT];
    int64_t total_bytes;
};
