// step_common.h -- host/device parameter blocks for the fused env-step kernel.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "program.h"

// What one launch does (bit flags).
enum TsModeBits {
    TS_M_CMD_ACTIONS = 1 << 0,   // EnvBatch.step: targets = drag + clip(a)*scale, angle = held
    TS_M_CMD_TARGETS = 1 << 1,   // Simulation.step(targets, angles)
    TS_M_CMD_OVERRIDE = 1 << 2,  // pose supplied externally (validation)
    TS_M_GRASP = 1 << 3,         // ToolBatch.update_grasps
    TS_M_SUBSTEPS = 1 << 4,      // run_substeps
    TS_M_CONTACTS = 1 << 5,      // detect + resolve contacts
    TS_M_ENV = 1 << 6,           // reward / done / auto-reset / obs
    TS_M_DETECT_ONLY = 1 << 7,   // plugin detect_contacts: write rows, no resolve
    TS_M_EXT_GRASP = 1 << 8,     // plugin run_substeps: grasp vertex + drag from arrays
    TS_M_CHECK_ACTIONS = 1 << 9  // abort (no state change) if *bad_flag != 0
};

// Scene constants (fp64 as in the reference; the kernel casts to Real where
// the solver runs in Real).
struct TsParams {
    double h, damp, g[3], ks, kv, k_contact;
    int32_t substeps, contact_iters;
    double rcm[3], shaft_r, clamp_r, clamp_len, grasp_r2;
    double start_axis[3], start_jaw[3], start_reach, start_clamp;
    double held_angle, held_cos, held_sin;
    double target[3], action_scale, success_thr;
    double w_l, w_d, w_s, reward_scale;
    double lo[3], hi[3];
    int64_t max_steps;
    double start_distance, target_obs[3];
    int64_t n_face;           // surface faces of the whole mesh (detect_contacts row capacity 3F)
    int32_t ablate, pad_a;    // development only (TS_ABLATE env var): skip phases to time them
    // fp32 copies of the solver constants (read straight from the constant bank by the fp32 build)
    float h_f, inv_h_f, damp_f, g_f[3], ks_f, hks_f, kv_f, pad_f;
};

inline void ts_finish_params(TsParams &S) {
    S.h_f = (float)S.h; S.inv_h_f = (float)(1.0 / S.h); S.damp_f = (float)S.damp;
    for (int c = 0; c < 3; ++c) S.g_f[c] = (float)S.g[c];
    S.ks_f = (float)S.ks; S.hks_f = (float)(0.5 * S.ks); S.kv_f = (float)S.kv; S.pad_f = 0.0f;
}

// Decoded device program (pointers into the uploaded blob).
struct TsDevProg {
    int32_t V, Vf, Vf_pad, Vstore, F, B, VPT, G;
    int32_t n_chunks, grasp_chunk, slot_cap, cbits_words;
    const TsChunk *chunks;
    const int4 *edge_idx;
    const void *edge_par;
    const int4 *tet_idx;
    const int4 *tet_slot;
    const void *tet_rv;
    const int4 *att_idx;
    const int4 *att_slot;
    const void *att_par;
    const void *att_anchor;
    const int32_t *region;
    const int32_t *valence;
    const int32_t *static_cnt;
    const int32_t *s2o;
    const int32_t *o2s;
    const void *w;
    const int32_t *faces;
    const int32_t *faces_orig;
    const void *rest;
    const int32_t *gsplit;
    int32_t compact;          // 1: use the 16-bit streams below
    double w_free;            // common inverse mass of free vertices (compact programs)
    const uint4 *edge_c;
    const uint4 *tet_c;
    int32_t narrow;           // single position buffer + byte degenerate counters (program.h)
    int32_t fast;             // the reach-scene shape: fast_step_kernel (step_kernel.cuh)
    int32_t edges_ok;         // the shared window matches TS_SMEM_WINDOW: edges_step_kernel allowed
    int32_t real_bytes;       // 4 (fp32 state) or 8 (fp64)
    const void *pf_base;      // the handle's whole device program (all parts): cmd_kernel prefetches
    int64_t pf_bytes;         //   it into L2 so the step kernel's first program reads do not go to HBM
    int32_t edge_gather;      // 1: owner-gathered edges (records below), positions double-buffered
    int32_t einc_bytes;       // 8 or 16
    const void *einc;
    const int32_t *eregion;
    const int32_t *evalence;
    const int32_t *face_gid;  // [F] global face index (contact emission key)
    // cluster parts (cluster_k > 1): one CTA of an env's thread-block cluster
    int32_t Vown;             // end of the owned (written-back) storage positions
    int32_t boff;             // fp32 compact streams carry byte offsets (12 x index), padded
    const int32_t *wsplit;    // [n_chunks][B/32 + 1] first tet item of each warp in a chunk
    int32_t rvdict;           // tet 6 V0 as a dictionary index in the stream's spare bits
    const float *rltab;       // distinct rest lengths (4-byte edge records)
    const float *rvtab;       // distinct 6 V0 values (rvdict)
    int32_t n_rltab, n_rvtab; // their sizes (fast programs keep both in shared memory: TS_TAB_OFF)
    int32_t cluster_k, cluster_rank;
    const int32_t *send_off;  // [Vf_pad + 1]
    const int32_t *send;      // (rank << 20) | storage position of a halo copy
    const int32_t *face_own;  // [F][3] (rank << 20) | position of a free face vertex's owner, -1 pinned
};

// Tool pose of one env (ToolBatch row, tool.py:263-302), fp64.
struct TsPose { double ax[3], jw[3], reach, clamp; };

// Per-env command block: written by the per-env command kernel (tool command,
// grasp release, capsule rows, the step's reward distance), read by the step
// kernel (which adds the grasp search result, divergence and contact count)
// and finished by the per-env epilogue kernel (reward / done / reset / obs).
// The two scalar stages run one THREAD per env instead of one thread of a
// 320-thread CTA while the rest of the CTA waits at a barrier.
struct TsCmd {
    double caps[3][7];        // capsule rows (tool.py:347-370)
    double drag[3];           // drag point after the command
    TsPose pose;              // tool pose after the command
    double dist;              // env mode: |drag - target|, env.py:103-108
    int32_t gv;               // grasp vertex (original id, -1 none) -- final after the step kernel
    int32_t need_search;      // clamp engaged and nothing held: nearest-vertex search
    int32_t clipped, rejected;
    int32_t pre_done;         // env mode: success || steps + 1 >= max (done unless diverged)
    int32_t any_bad;          // step kernel: non-finite position after the step
    int32_t n_contacts;       // step kernel: contacts resolved
    int32_t pad;
};

// Per-launch pointers (device).
struct TsLaunch {
    int32_t mode;
    int64_t n_env;
    // state
    void *x, *v;
    double *axis, *jaw, *reach, *clamp;
    int64_t *grasp_vertex;
    uint8_t *grasped;
    int64_t *steps;
    double *l_prev, *ep_return;
    // inputs
    const void *actions; int32_t actions_f32;
    const double *targets, *angles;
    const double *ovr_axis, *ovr_jaw, *ovr_reach, *ovr_clamp;
    const uint8_t *ovr_clipped;
    const int64_t *ext_gv;        // plugin run_substeps
    const double *ext_drag;
    const double *ext_caps;       // plugin detect: (N,3,7)
    const int32_t *bad_flag;
    // outputs
    void *obs, *final_obs; int32_t obs_f64;
    double *reward, *distance, *ret_out;
    uint8_t *terminated, *truncated, *success, *diverged, *clipped, *rejected, *done_mask;
    int32_t *contacts;
    int64_t *len_out;
    // plugin detect outputs (capacity 3F rows per env)
    int32_t *det_count, *det_face, *det_cap;
    double *det_depth, *det_dir, *det_bary;
    TsCmd *cmd;                   // (n_env,) per-env command blocks (handle-owned scratch)
};

// Shared-memory layout sizes (bytes) for one CTA.
inline int ts_smem_bytes(const TsDevProg &P, int real_bytes) {
    return ts_smem_layout_bytes(P.Vstore, P.slot_cap, P.Vf_pad, P.F, real_bytes, P.edge_gather, P.narrow);
}

// command kernel -> fused step kernel -> epilogue kernel, stream ordered
// step-kernel launch bounds (overridable with -D for experiments: build.py TS_NVCC_FLAGS)
#ifndef TS_STEP_MAXT
#define TS_STEP_MAXT 512
#endif
#ifndef TS_STEP_MINB
#define TS_STEP_MINB 2
#endif
#ifndef TS_EDGES_MAXT
#define TS_EDGES_MAXT 512
#endif
#ifndef TS_EDGES_MINB
#define TS_EDGES_MINB 2
#endif
// fp32 shape-specialised kernels (step_kernel.cuh): the reach-scene shape, and distance-only programs
// .shared address of the first byte of dynamic shared memory in a non-cluster launch on sm_100
// (the fast kernel's constant addressing, step_kernel.cuh lds3c); probed by the library at handle
// creation (ts_smem_window), which keeps the fast kernel off if the device reports another value
#define TS_SMEM_WINDOW 0x400u
uint32_t ts_smem_window(int device);

inline bool ts_use_fast_kernel(const TsDevProg &P, int ablate) {
    return P.fast && P.B <= TS_STEP_MAXT && !(ablate & 256);
}
inline bool ts_use_edges_kernel(const TsDevProg &P) {   // P.edges_ok: the shared window probe matched
    return P.n_chunks == 0 && P.VPT == 1 && P.B <= TS_EDGES_MAXT && P.edges_ok && P.einc_bytes == 4 &&
           2 * P.n_rltab <= TS_TAB_CAP;
}
template <typename Real>
cudaError_t ts_launch_step(const TsDevProg &P, const TsParams &S, const TsLaunch &L, int grid,
                           int smem, cudaStream_t stream, bool pdl = false);
// large meshes: `n_clusters` clusters of K CTAs (part programs `parts`, device array)
template <typename Real>
cudaError_t ts_launch_cluster_step(const TsDevProg *parts, int VPT, int K, int B, const TsParams &S,
                                   const TsLaunch &L, int n_clusters, int smem, cudaStream_t stream);
cudaError_t ts_launch_cmd(const TsDevProg &P, const TsParams &S, const TsLaunch &L, cudaStream_t stream,
                          bool pdl = false);
// pdl: programmatic dependent launch -- the kernel may start while the previous kernel of the
// stream (this library's own command / step kernel) runs, and waits (griddepcontrol.wait) before it
// reads that kernel's results
cudaError_t ts_launch_epilogue(const TsDevProg &P, const TsParams &S, const TsLaunch &L, cudaStream_t stream,
                               bool pdl = false);
template <typename Real>
cudaError_t ts_launch_reset(const TsDevProg &P, const TsParams &S, const TsLaunch &L,
                            const uint8_t *mask, int observe_only, cudaStream_t stream);
cudaError_t ts_launch_check_actions(const void *actions, int actions_f32, int64_t n,
                                    int32_t *flag, cudaStream_t stream);
cudaError_t ts_launch_uniform_dev(double *out, int64_t n, int64_t first, uint64_t seed, uint64_t *counter,
                                  cudaStream_t stream);
cudaError_t ts_launch_uniform(double *out, int64_t n, int64_t first, uint64_t seed, uint64_t counter,
                              cudaStream_t stream);
