// capi.cu -- C-ABI of the B200 env step (include/tissuesim_b200.h).
#include <atomic>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/tissuesim_b200.h"
#include "compiler.h"
#include "step_common.h"

namespace {
thread_local std::string g_err;
std::atomic<int64_t> g_launches{0};

int fail(int code, const std::string &msg) {
    g_err = msg;
    return code;
}
int cuda_fail(cudaError_t e, const char *what) {
    g_err = std::string(what) + ": " + cudaGetErrorString(e);
    return TS_ERR_CUDA;
}
}  // namespace

struct ts_handle {
    int device = 0;
    int precision = TS_F32;
    std::vector<uint8_t> host_blob;
    void *dev_blob = nullptr;
    TsDevProg prog{};
    TsParams params{};
    ts_layout_info info{};
    int smem = 0;
    int max_grid = 0;   // 0 = one CTA per environment
    TsCmd *cmd = nullptr;   // per-env command blocks (grown on demand)
    int64_t cmd_cap = 0;
    std::vector<cudaEvent_t> tev;   // step-kernel timing events (pairs), see ts_kernel_timing
    int64_t tev_used = 0;
    int cluster_k = 1;                  // > 1: thread-block cluster program (large meshes)
    std::vector<TsDevProg> parts;       // decoded part programs (host copies)
    TsDevProg *dev_parts = nullptr;     // the same, on the device (cluster kernel argument)
    int64_t n_vert = 0;                 // scene vertex count (typed-entry shape checks)
};

static const char *ts_kernel_name_for(const TsDevProg &P, int real_bytes, int cluster_k, int ablate) {
    static const char *names[] = {
        "tsk::fast_step_kernel<float>", "tsk::edges_step_kernel<float>",
        "tsk::step_kernel<float, 1>", "tsk::step_kernel<float, 2>", "tsk::step_kernel<float, 4>",
        "tsk::step_kernel<float, 8>", "tsk::step_kernel<double, 1>", "tsk::step_kernel<double, 2>",
        "tsk::step_kernel<double, 4>", "tsk::step_kernel<double, 8>",
        "tsk::cluster_step_kernel<float, 1>", "tsk::cluster_step_kernel<float, 2>",
        "tsk::cluster_step_kernel<float, 4>", "tsk::cluster_step_kernel<double, 1>",
        "tsk::cluster_step_kernel<double, 2>", "tsk::cluster_step_kernel<double, 4>"};
    const int d = real_bytes == 8;
    if (cluster_k > 1) return names[10 + 3 * d + (P.VPT <= 1 ? 0 : P.VPT <= 2 ? 1 : 2)];
    if (d && P.VPT == 1 && P.B <= 320 && !(ablate & 2048)) return "tsk::step2_kernel<double>";
    if (!d && ts_use_fast_kernel(P, ablate)) return names[0];
    if (!d && ts_use_edges_kernel(P)) return names[1];
    const int v = P.VPT <= 1 ? 0 : P.VPT == 2 ? 1 : P.VPT <= 4 ? 2 : 3;   // VPT 3 runs the 4 kernel
    return names[2 + 4 * d + v];
}

extern "C" {

const char *ts_last_error(void) { return g_err.c_str(); }
int32_t ts_abi_version(void) { return TS_ABI_VERSION; }
int64_t ts_launch_count(void) { return g_launches.load(); }

static ts_layout_opts default_opts() {
    ts_layout_opts o;
    std::memset(&o, 0, sizeof(o));
    return o;
}

// One CTA per env when the mesh fits (or cluster_size == 1), else a K-CTA cluster program.
static int compile_any(const ts_scene_desc &d, const ts_layout_opts &o, std::vector<uint8_t> &blob,
                       ts_layout_info &inf, std::string &err) {
    if (o.cluster_size >= 2) return ts::compile_cluster(d, o, o.cluster_size, blob, inf, err);
    int rc = ts::compile_program(d, o, blob, inf, err);
    if (rc == TS_ERR_UNSUPPORTED && o.cluster_size == 0) {
        std::string e2;
        rc = ts::compile_cluster(d, o, 0, blob, inf, e2);
        if (rc != TS_OK) err += "; " + e2;
    }
    return rc;
}

int32_t ts_compile_program(const ts_scene_desc *desc, const ts_layout_opts *opts, void *buf, int64_t *bytes,
                           ts_layout_info *info) {
    if (!desc || !bytes) return fail(TS_ERR_INVALID, "null argument");
    ts_layout_opts o = opts ? *opts : default_opts();
    std::vector<uint8_t> blob;
    ts_layout_info inf;
    std::string err;
    int rc = compile_any(*desc, o, blob, inf, err);
    if (rc != TS_OK) return fail(rc, err);
    if (info) *info = inf;
    if (buf) {
        if (*bytes < (int64_t)blob.size()) {
            *bytes = (int64_t)blob.size();   // report the size needed
            return fail(TS_ERR_INVALID, "buffer too small");
        }
        std::memcpy(buf, blob.data(), blob.size());
    }
    *bytes = (int64_t)blob.size();
    return TS_OK;
}

static void decode_part(const uint8_t *host, const uint8_t *b, TsDevProg &P) {
    const TsProgHeader *H = reinterpret_cast<const TsProgHeader *>(host);
    P.V = H->V; P.Vf = H->Vf; P.Vf_pad = H->Vf_pad; P.Vstore = H->Vstore;
    P.F = H->F; P.B = H->B; P.VPT = H->VPT; P.G = H->G;
    P.n_chunks = H->n_chunks; P.grasp_chunk = H->grasp_chunk; P.slot_cap = H->slot_capacity;
    P.cbits_words = (3 * H->F + 31) / 32;
    P.chunks = reinterpret_cast<const TsChunk *>(b + H->off[TS_SEC_CHUNK]);
    P.edge_idx = reinterpret_cast<const int4 *>(b + H->off[TS_SEC_EDGE_IDX]);
    P.edge_par = b + H->off[TS_SEC_EDGE_PAR];
    P.tet_idx = reinterpret_cast<const int4 *>(b + H->off[TS_SEC_TET_IDX]);
    P.tet_slot = reinterpret_cast<const int4 *>(b + H->off[TS_SEC_TET_SLOT]);
    P.tet_rv = b + H->off[TS_SEC_TET_RV];
    P.att_idx = reinterpret_cast<const int4 *>(b + H->off[TS_SEC_ATT_IDX]);
    P.att_slot = reinterpret_cast<const int4 *>(b + H->off[TS_SEC_ATT_SLOT]);
    P.att_par = b + H->off[TS_SEC_ATT_PAR];
    P.att_anchor = b + H->off[TS_SEC_ATT_ANCHOR];
    P.region = reinterpret_cast<const int32_t *>(b + H->off[TS_SEC_REGION]);
    P.valence = reinterpret_cast<const int32_t *>(b + H->off[TS_SEC_VALENCE]);
    P.static_cnt = reinterpret_cast<const int32_t *>(b + H->off[TS_SEC_STATIC_CNT]);
    P.s2o = reinterpret_cast<const int32_t *>(b + H->off[TS_SEC_S2O]);
    P.o2s = reinterpret_cast<const int32_t *>(b + H->off[TS_SEC_O2S]);
    P.w = b + H->off[TS_SEC_W];
    P.faces = reinterpret_cast<const int32_t *>(b + H->off[TS_SEC_FACES]);
    P.faces_orig = reinterpret_cast<const int32_t *>(b + H->off[TS_SEC_FACES_ORIG]);
    P.rest = b + H->off[TS_SEC_REST];
    P.gsplit = reinterpret_cast<const int32_t *>(b + H->off[TS_SEC_GSPLIT]);
    P.compact = H->compact;
    P.w_free = H->w_free;
    P.edge_c = reinterpret_cast<const uint4 *>(b + H->off[TS_SEC_EDGE_C]);
    P.tet_c = reinterpret_cast<const uint4 *>(b + H->off[TS_SEC_TET_C]);
    P.edge_gather = H->edge_gather;
    P.narrow = H->narrow;
    P.fast = H->real_bytes == 4 && H->VPT == 1 && H->n_chunks == 1 && H->grasp_chunk == 0 && H->edge_gather &&
             H->einc_bytes == 4 && H->boff && H->rvdict && H->narrow && H->n_att_items == 0 &&
             H->n_edge_items == 0 && H->cluster_k == 1 && H->compact && 2 * H->n_rltab <= TS_TAB_CAP &&
             H->n_rvtab <= TS_TAB_CAP;
    P.einc_bytes = H->einc_bytes;
    P.einc = b + H->off[TS_SEC_EINC];
    P.eregion = reinterpret_cast<const int32_t *>(b + H->off[TS_SEC_EREGION]);
    P.evalence = reinterpret_cast<const int32_t *>(b + H->off[TS_SEC_EVAL]);
    P.face_gid = reinterpret_cast<const int32_t *>(b + H->off[TS_SEC_FACE_GID]);
    P.Vown = H->Vown; P.cluster_k = H->cluster_k; P.cluster_rank = H->cluster_rank; P.boff = H->boff;
    P.real_bytes = H->real_bytes;
    P.send_off = reinterpret_cast<const int32_t *>(b + H->off[TS_SEC_SEND_OFF]);
    P.send = reinterpret_cast<const int32_t *>(b + H->off[TS_SEC_SEND]);
    P.face_own = reinterpret_cast<const int32_t *>(b + H->off[TS_SEC_FACE_OWN]);
    P.wsplit = reinterpret_cast<const int32_t *>(b + H->off[TS_SEC_WSPLIT]);
    P.rvdict = H->rvdict;
    P.rltab = reinterpret_cast<const float *>(b + H->off[TS_SEC_RLTAB]);
    P.rvtab = reinterpret_cast<const float *>(b + H->off[TS_SEC_RVTAB]);
    P.n_rltab = H->n_rltab; P.n_rvtab = H->n_rvtab;
}

static void fill_params(const ts_scene_desc &d, TsParams &S) {
    S.h = d.dt / d.substeps;   // SolverParams.h, solver.py:92-94
    // damping factor, _kernels.pyx:592
    if (d.damping == 0.0) S.damp = 1.0;
    else { double v = 1.0 - d.damping * S.h; S.damp = (v > 0.0) ? v : 0.0; }
    for (int c = 0; c < 3; ++c) S.g[c] = d.gravity[c];
    S.ks = d.k_s; S.kv = d.k_v; S.k_contact = d.k_contact;
    S.substeps = d.substeps; S.contact_iters = d.contact_iterations;
    for (int c = 0; c < 3; ++c) {
        S.rcm[c] = d.rcm[c]; S.start_axis[c] = d.start_axis[c]; S.start_jaw[c] = d.start_jaw[c];
        S.target[c] = d.target[c]; S.lo[c] = d.workspace_low[c]; S.hi[c] = d.workspace_high[c];
        S.target_obs[c] = d.target_obs[c];
    }
    S.shaft_r = d.shaft_radius; S.clamp_r = d.clamp_radius; S.clamp_len = d.clamp_length;
    S.grasp_r2 = d.grasp_radius2;
    S.start_reach = d.start_reach; S.start_clamp = d.start_clamp;
    S.held_angle = d.held_clamp_angle; S.held_cos = d.held_cos; S.held_sin = d.held_sin;
    S.action_scale = d.action_scale; S.success_thr = d.success_threshold;
    S.w_l = d.w_distance; S.w_d = d.w_delta; S.w_s = d.w_success; S.reward_scale = d.reward_scale;
    S.max_steps = d.max_episode_steps; S.start_distance = d.start_distance;
    S.n_face = d.n_face;
    // development ablation switch (results are wrong when set): 1 tets, 2 slot sums, 4 edge
    // gather, 8 contacts, 16 grasp search, 64 the whole substep loop, 128 slot sums capped at 12
    S.ablate = 0;
    if (const char *env = std::getenv("TS_ABLATE")) S.ablate = std::atoi(env);
    ts_finish_params(S);
}

static int32_t create_handle(const ts_scene_desc *desc, const ts_layout_opts &o, int32_t device, ts_handle *h,
                             ts_handle **out);

int32_t ts_create(const ts_scene_desc *desc, const ts_layout_opts *opts, int32_t device, ts_handle **out) {
    if (!desc || !out) return fail(TS_ERR_INVALID, "null argument");
    if (desc->substeps < 1) return fail(TS_ERR_INVALID, "substeps must be >= 1");
    if (desc->dt <= 0.0) return fail(TS_ERR_INVALID, "dt must be positive");
    ts_layout_opts o = opts ? *opts : default_opts();
    ts_handle *h = new ts_handle();
    h->device = device;
    h->precision = o.precision;
    std::string err;
    int rc = compile_any(*desc, o, h->host_blob, h->info, err);
    if (rc != TS_OK) { delete h; return fail(rc, err); }
    return create_handle(desc, o, device, h, out);
}

int32_t ts_create_from_program(const ts_scene_desc *desc, const void *program, int64_t bytes,
                               const ts_layout_info *info, int32_t device, ts_handle **out) {
    if (!desc || !program || !info || !out) return fail(TS_ERR_INVALID, "null argument");
    if (desc->substeps < 1) return fail(TS_ERR_INVALID, "substeps must be >= 1");
    if (desc->dt <= 0.0) return fail(TS_ERR_INVALID, "dt must be positive");
    if (bytes < (int64_t)sizeof(TsProgHeader)) return fail(TS_ERR_INVALID, "program too small");
    const int32_t magic = *reinterpret_cast<const int32_t *>(program);
    if (magic == TS_PROG_MAGIC) {
        const TsProgHeader *H = reinterpret_cast<const TsProgHeader *>(program);
        if (H->version != TS_PROG_VERSION || H->total_bytes != bytes || H->V != desc->n_vert)
            return fail(TS_ERR_INVALID, "program does not match this library / scene");
    } else if (magic == TS_CLUSTER_MAGIC) {
        const TsClusterHeader *C = reinterpret_cast<const TsClusterHeader *>(program);
        if (C->total_bytes != bytes || C->n_vert != desc->n_vert)
            return fail(TS_ERR_INVALID, "program does not match this scene");
    } else {
        return fail(TS_ERR_INVALID, "not a compiled scene program");
    }
    ts_layout_opts o = default_opts();
    o.precision = info->precision;
    ts_handle *h = new ts_handle();
    h->device = device;
    h->precision = info->precision;
    h->info = *info;
    h->host_blob.assign(reinterpret_cast<const uint8_t *>(program), reinterpret_cast<const uint8_t *>(program) + bytes);
    return create_handle(desc, o, device, h, out);
}

static int32_t create_handle(const ts_scene_desc *desc, const ts_layout_opts &o, int32_t device, ts_handle *h,
                             ts_handle **out) {
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) { delete h; return cuda_fail(e, "cudaSetDevice"); }
    e = cudaMalloc(&h->dev_blob, h->host_blob.size());
    if (e != cudaSuccess) { delete h; return cuda_fail(e, "cudaMalloc(program)"); }
    e = cudaMemcpy(h->dev_blob, h->host_blob.data(), h->host_blob.size(), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) { cudaFree(h->dev_blob); delete h; return cuda_fail(e, "cudaMemcpy(program)"); }
    const uint8_t *hb = h->host_blob.data();
    const uint8_t *db = reinterpret_cast<const uint8_t *>(h->dev_blob);
    const int R = o.precision == TS_F64 ? 8 : 4;
    if (reinterpret_cast<const TsClusterHeader *>(hb)->magic == TS_CLUSTER_MAGIC) {
        const TsClusterHeader *CH = reinterpret_cast<const TsClusterHeader *>(hb);
        h->cluster_k = CH->K;
        h->parts.resize(CH->K);
        for (int r = 0; r < CH->K; ++r) decode_part(hb + CH->part_off[r], db + CH->part_off[r], h->parts[r]);
        h->prog = h->parts[0];
        h->smem = 0;
        for (int r = 0; r < CH->K; ++r) h->smem = std::max(h->smem, ts_smem_bytes(h->parts[r], R));
        e = cudaMalloc(&h->dev_parts, sizeof(TsDevProg) * CH->K);
        if (e == cudaSuccess)
            e = cudaMemcpy(h->dev_parts, h->parts.data(), sizeof(TsDevProg) * CH->K, cudaMemcpyHostToDevice);
        if (e != cudaSuccess) { cudaFree(h->dev_blob); delete h; return cuda_fail(e, "cluster programs"); }
    } else {
        decode_part(hb, db, h->prog);
        h->smem = ts_smem_bytes(h->prog, R);
        const bool window_ok = ts_smem_window(device) == TS_SMEM_WINDOW;   // else the generic kernel
        if (!window_ok) h->prog.fast = 0;
        h->prog.edges_ok = window_ok ? 1 : 0;
    }
    // L2 prefetch of the program by the command kernel: small programs only -- a multi-MB cluster
    // program's bulk prefetches keep the command kernel alive longer than they save (52,359-tet
    // slab, one env: 155.6 -> 187 us/step with it)
    const int64_t pf = (int64_t)h->host_blob.size() / 16 * 16;
    h->prog.pf_base = pf <= (512 << 10) ? h->dev_blob : nullptr;
    h->prog.pf_bytes = pf <= (512 << 10) ? pf : 0;
    fill_params(*desc, h->params);
    h->n_vert = desc->n_vert;
    int max_smem = 0;
    cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    if (h->smem > max_smem) {
        char buf[256];
        std::snprintf(buf, sizeof(buf), "layout needs %d B of shared memory per CTA, device allows %d; "
                      "lower max_chunk_slots", h->smem, max_smem);
        cudaFree(h->dev_blob); delete h;
        return fail(TS_ERR_UNSUPPORTED, buf);
    }
    h->info.smem_bytes = h->smem;
    *out = h;
    return TS_OK;
}

int32_t ts_destroy(ts_handle *h) {
    if (!h) return TS_OK;
    if (h->dev_blob) cudaFree(h->dev_blob);
    if (h->cmd) cudaFree(h->cmd);
    if (h->dev_parts) cudaFree(h->dev_parts);
    for (cudaEvent_t ev : h->tev) cudaEventDestroy(ev);
    delete h;
    return TS_OK;
}

int32_t ts_query(const ts_handle *h, ts_layout_info *info) {
    if (!h || !info) return fail(TS_ERR_INVALID, "null argument");
    *info = h->info;
    return TS_OK;
}

static void fill_state(TsLaunch &L, const ts_env_state *st) {
    L.x = st->x; L.v = st->v;
    L.axis = st->tool_axis; L.jaw = st->tool_jaw; L.reach = st->tool_reach; L.clamp = st->tool_clamp;
    L.grasp_vertex = st->grasp_vertex; L.grasped = st->grasped;
    L.steps = st->steps; L.l_prev = st->l_prev; L.ep_return = st->ep_return;
}

// One step = command kernel (one thread per env) -> fused step kernel (one CTA per env)
// -> epilogue kernel (one thread per env), stream ordered.
static int launch(ts_handle *h, const TsLaunch &L_in, cudaStream_t s) {
    if (L_in.n_env <= 0) return TS_OK;
    if (L_in.n_env > h->cmd_cap) {
        // grown outside the steady state (the first step at a batch size); not graph-capturable
        TsCmd *nb = nullptr;
        cudaError_t e = cudaMalloc(&nb, (size_t)L_in.n_env * sizeof(TsCmd));
        if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(command blocks)");
        if (h->cmd) { cudaStreamSynchronize(s); cudaFree(h->cmd); }
        h->cmd = nb; h->cmd_cap = L_in.n_env;
    }
    TsLaunch L = L_in;
    L.cmd = h->cmd;
    int grid = (int)std::min<int64_t>(L.n_env, h->max_grid > 0 ? h->max_grid : (int64_t)1 << 30);
    const bool timed = 2 * h->tev_used + 1 < (int64_t)h->tev.size();
    cudaError_t e = ts_launch_cmd(h->prog, h->params, L, s, !(h->params.ablate & 1024));
    if (e != cudaSuccess) return cuda_fail(e, "command kernel launch");
    // programmatic dependent launch of step and epilogue (each overlaps its predecessor's tail);
    // off while the step kernel is being timed, so its events bracket exactly its own execution
    const bool pdl = !timed && !(h->params.ablate & 1024);
    if (timed) cudaEventRecord(h->tev[2 * h->tev_used], s);
    if (h->cluster_k > 1)
        e = h->precision == TS_F64
                ? ts_launch_cluster_step<double>(h->dev_parts, h->prog.VPT, h->cluster_k, h->prog.B, h->params, L,
                                                 grid, h->smem, s)
                : ts_launch_cluster_step<float>(h->dev_parts, h->prog.VPT, h->cluster_k, h->prog.B, h->params, L,
                                                grid, h->smem, s);
    else
        e = h->precision == TS_F64 ? ts_launch_step<double>(h->prog, h->params, L, grid, h->smem, s, pdl)
                                   : ts_launch_step<float>(h->prog, h->params, L, grid, h->smem, s, pdl);
    if (e != cudaSuccess) return cuda_fail(e, "step kernel launch");
    if (timed) cudaEventRecord(h->tev[2 * h->tev_used++ + 1], s);
    e = ts_launch_epilogue(h->prog, h->params, L, s, pdl);
    if (e != cudaSuccess) return cuda_fail(e, "epilogue kernel launch");
    g_launches.fetch_add(3);
    return TS_OK;
}

int32_t ts_env_step(ts_handle *h, const ts_env_state *st, int64_t num_envs, const void *actions,
                    int32_t actions_f32, const ts_step_out *out, const ts_tool_override *ovr,
                    int32_t *bad_action_flag, void *stream) {
    if (!h || !st || !out) return fail(TS_ERR_INVALID, "null argument");
    if (!actions && !ovr) return fail(TS_ERR_INVALID, "actions required");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    TsLaunch L;
    std::memset(&L, 0, sizeof(L));
    fill_state(L, st);
    L.n_env = num_envs;
    L.mode = TS_M_GRASP | TS_M_SUBSTEPS | TS_M_CONTACTS | TS_M_ENV;
    if (ovr) {
        L.mode |= TS_M_CMD_OVERRIDE;
        L.ovr_axis = ovr->axis; L.ovr_jaw = ovr->jaw; L.ovr_reach = ovr->reach; L.ovr_clamp = ovr->clamp;
        L.ovr_clipped = ovr->clipped;
    } else {
        L.mode |= TS_M_CMD_ACTIONS;
        L.actions = actions; L.actions_f32 = actions_f32;
    }
    if (bad_action_flag) {
        if (!actions) return fail(TS_ERR_INVALID, "action check needs actions");
        cudaError_t e = ts_launch_check_actions(actions, actions_f32, num_envs, bad_action_flag, s);
        if (e != cudaSuccess) return cuda_fail(e, "action check launch");
        g_launches.fetch_add(1);
        L.mode |= TS_M_CHECK_ACTIONS;
        L.bad_flag = bad_action_flag;
    }
    L.obs = out->obs; L.final_obs = out->final_obs; L.obs_f64 = out->obs_f64;
    L.reward = out->reward; L.distance = out->distance; L.ret_out = out->episode_return;
    L.terminated = out->terminated; L.truncated = out->truncated; L.success = out->success;
    L.diverged = out->diverged; L.clipped = out->clipped; L.done_mask = out->done_mask;
    L.contacts = out->contacts; L.len_out = out->episode_length;
    return launch(h, L, s);
}

int32_t ts_env_reset(ts_handle *h, const ts_env_state *st, int64_t num_envs, const uint8_t *mask, void *obs,
                     int32_t obs_f64, void *stream) {
    if (!h || !st) return fail(TS_ERR_INVALID, "null argument");
    TsLaunch L;
    std::memset(&L, 0, sizeof(L));
    fill_state(L, st);
    L.n_env = num_envs;
    L.obs = obs; L.obs_f64 = obs_f64;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (num_envs <= 0) return TS_OK;
    cudaError_t e = h->precision == TS_F64 ? ts_launch_reset<double>(h->prog, h->params, L, mask, 0, s)
                                           : ts_launch_reset<float>(h->prog, h->params, L, mask, 0, s);
    if (e != cudaSuccess) return cuda_fail(e, "reset kernel launch");
    g_launches.fetch_add(1);
    return TS_OK;
}

int32_t ts_env_observe(ts_handle *h, const ts_env_state *st, int64_t num_envs, void *obs, int32_t obs_f64,
                       void *stream) {
    if (!h || !st || !obs) return fail(TS_ERR_INVALID, "null argument");
    TsLaunch L;
    std::memset(&L, 0, sizeof(L));
    fill_state(L, st);
    L.n_env = num_envs;
    L.obs = obs; L.obs_f64 = obs_f64;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (num_envs <= 0) return TS_OK;
    cudaError_t e = h->precision == TS_F64 ? ts_launch_reset<double>(h->prog, h->params, L, nullptr, 1, s)
                                           : ts_launch_reset<float>(h->prog, h->params, L, nullptr, 1, s);
    if (e != cudaSuccess) return cuda_fail(e, "observe kernel launch");
    g_launches.fetch_add(1);
    return TS_OK;
}

int32_t ts_sim_step(ts_handle *h, const ts_env_state *st, int64_t num_envs, const double *targets,
                    const double *angles, const ts_tool_override *ovr, uint8_t *clipped, uint8_t *rejected,
                    uint8_t *diverged, int32_t *contacts, void *stream) {
    if (!h || !st) return fail(TS_ERR_INVALID, "null argument");
    TsLaunch L;
    std::memset(&L, 0, sizeof(L));
    fill_state(L, st);
    L.n_env = num_envs;
    L.mode = TS_M_GRASP | TS_M_SUBSTEPS | TS_M_CONTACTS;
    if (ovr) {
        L.mode |= TS_M_CMD_OVERRIDE;
        L.ovr_axis = ovr->axis; L.ovr_jaw = ovr->jaw; L.ovr_reach = ovr->reach; L.ovr_clamp = ovr->clamp;
        L.ovr_clipped = ovr->clipped;
    } else if (targets) {
        L.mode |= TS_M_CMD_TARGETS;
        L.targets = targets; L.angles = angles;
    }
    L.clipped = clipped; L.rejected = rejected; L.diverged = diverged; L.contacts = contacts;
    return launch(h, L, reinterpret_cast<cudaStream_t>(stream));
}

int32_t ts_run_substeps(ts_handle *h, void *x, void *v, int64_t num_envs, const int64_t *grasp_vertex,
                        const double *drag_points, const double *gravity, double hstep, int32_t substeps,
                        double damping, void *stream) {
    if (!h || !x || !v || !grasp_vertex || !drag_points || !gravity) return fail(TS_ERR_INVALID, "null argument");
    if (substeps < 0) return fail(TS_ERR_INVALID, "substeps must be >= 0");
    TsLaunch L;
    std::memset(&L, 0, sizeof(L));
    L.x = x; L.v = v; L.n_env = num_envs;
    L.mode = TS_M_SUBSTEPS | TS_M_EXT_GRASP;
    L.ext_gv = grasp_vertex; L.ext_drag = drag_points;
    // per-call solver parameters, as the plugin protocol passes them (_kernels.pyx:583, 592)
    const TsParams saved = h->params;
    TsParams &S = h->params;
    S.h = hstep; S.substeps = substeps;
    for (int c = 0; c < 3; ++c) S.g[c] = gravity[c];
    if (damping == 0.0) S.damp = 1.0;
    else { double dv = 1.0 - damping * hstep; S.damp = (dv > 0.0) ? dv : 0.0; }
    ts_finish_params(S);
    int rc = substeps > 0 ? launch(h, L, reinterpret_cast<cudaStream_t>(stream)) : TS_OK;
    h->params = saved;
    return rc;
}

int32_t ts_detect_contacts(ts_handle *h, const void *x, int64_t num_envs, const double *caps, int32_t *count,
                           int32_t *face, int32_t *cap, double *depth, double *dir, double *bary, void *stream) {
    if (!h || !x || !caps || !count || !face || !cap || !depth || !dir || !bary)
        return fail(TS_ERR_INVALID, "null argument");
    TsLaunch L;
    std::memset(&L, 0, sizeof(L));
    L.x = const_cast<void *>(x); L.v = const_cast<void *>(x); L.n_env = num_envs;
    L.mode = TS_M_DETECT_ONLY;
    L.ext_caps = caps;
    L.det_count = count; L.det_face = face; L.det_cap = cap; L.det_depth = depth; L.det_dir = dir; L.det_bary = bary;
    return launch(h, L, reinterpret_cast<cudaStream_t>(stream));
}

int32_t ts_uniform_actions(double *actions, int64_t num_envs, int64_t first_env, uint64_t seed, uint64_t counter,
                           void *stream) {
    if (!actions) return fail(TS_ERR_INVALID, "null argument");
    if (num_envs <= 0) return TS_OK;
    cudaError_t e = ts_launch_uniform(actions, 3 * num_envs, 3 * first_env, seed, counter,
                                      reinterpret_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "uniform kernel launch");
    g_launches.fetch_add(1);
    return TS_OK;
}

int32_t ts_kernel_timing(ts_handle *h, int32_t enable, int32_t max_launches) {
    if (!h) return fail(TS_ERR_INVALID, "null argument");
    for (cudaEvent_t ev : h->tev) cudaEventDestroy(ev);
    h->tev.clear();
    h->tev_used = 0;
    if (!enable) return TS_OK;
    if (max_launches < 1) return fail(TS_ERR_INVALID, "max_launches must be >= 1");
    h->tev.resize(2 * (size_t)max_launches);
    for (auto &ev : h->tev) {
        cudaError_t e = cudaEventCreate(&ev);
        if (e != cudaSuccess) return cuda_fail(e, "cudaEventCreate");
    }
    return TS_OK;
}

const char *ts_step_kernel_name(ts_handle *h) {
    if (!h) { fail(TS_ERR_INVALID, "null handle"); return ""; }
    return ts_kernel_name_for(h->prog, h->precision == TS_F64 ? 8 : 4, h->cluster_k, h->params.ablate);
}

int32_t ts_kernel_time(ts_handle *h, double *total_ms, int64_t *launches) {
    if (!h || !total_ms || !launches) return fail(TS_ERR_INVALID, "null argument");
    double tot = 0.0;
    for (int64_t i = 0; i < h->tev_used; ++i) {
        cudaError_t e = cudaEventSynchronize(h->tev[2 * i + 1]);
        if (e != cudaSuccess) return cuda_fail(e, "cudaEventSynchronize");
        float ms = 0.0f;
        e = cudaEventElapsedTime(&ms, h->tev[2 * i], h->tev[2 * i + 1]);
        if (e != cudaSuccess) return cuda_fail(e, "cudaEventElapsedTime");
        tot += ms;
    }
    *total_ms = tot;
    *launches = h->tev_used;
    h->tev_used = 0;
    return TS_OK;
}

int32_t ts_uniform_actions_dev(double *actions, int64_t num_envs, int64_t first_env, uint64_t seed,
                               uint64_t *counter, void *stream) {
    if (!actions || !counter) return fail(TS_ERR_INVALID, "null argument");
    if (num_envs <= 0) return TS_OK;
    cudaError_t e = ts_launch_uniform_dev(actions, 3 * num_envs, 3 * first_env, seed, counter,
                                          reinterpret_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "uniform kernel launch");
    g_launches.fetch_add(3 * num_envs <= 65536 ? 1 : 2);
    return TS_OK;
}

int32_t ts_graph_launch_sync(void *graph_exec, void *stream) {
    if (!graph_exec) return fail(TS_ERR_INVALID, "null graph");
    const cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    cudaError_t e = cudaGraphLaunch(reinterpret_cast<cudaGraphExec_t>(graph_exec), s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(e, "graph launch");
    return TS_OK;
}

int32_t ts_graph_launch(void *graph_exec, void *stream) {
    if (!graph_exec) return fail(TS_ERR_INVALID, "null graph");
    const cudaError_t e = cudaGraphLaunch(reinterpret_cast<cudaGraphExec_t>(graph_exec),
                                          reinterpret_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "graph launch");
    return TS_OK;
}

int32_t ts_stream_sync(void *stream) {
    const cudaError_t e = cudaStreamSynchronize(reinterpret_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "stream synchronize");
    return TS_OK;
}

int32_t ts_set_max_grid(ts_handle *h, int32_t max_grid) {
    if (!h) return fail(TS_ERR_INVALID, "null argument");
    h->max_grid = max_grid;
    return TS_OK;
}

}  // extern "C"

// ---- typed (DLPack) entries ----------------------------------------------------------------
namespace {
enum Kind { K_REAL, K_F64, K_F32_OR_F64, K_I64, K_I32, K_U8 };

// Checks one DLTensor against (kind, shape) and returns its data address in *out.  Shape entries
// of -1 are free.  NULL tensors are accepted only when `optional`.
// host_ok: pinned host memory (kDLCUDAHost) is accepted too -- the kernels read / write it in place
// through the unified address space (zero-copy actions and step outputs)
int check_dl(const ts_handle *h, const DLTensor *t, const char *name, Kind kind, int ndim, const int64_t *shape,
             bool optional, void **out, int *is_f64 = nullptr, bool host_ok = false) {
    *out = nullptr;
    if (!t) {
        if (optional) return TS_OK;
        return fail(TS_ERR_INVALID, std::string(name) + ": tensor required");
    }
    char buf[320];
    // pinned host memory: kDLCUDAHost, or kDLCPU whose address the CUDA runtime knows as page-locked
    // (torch exports pinned tensors as kDLCPU); the kernels then use its device alias
    void *host_alias = nullptr;
    if (host_ok && (t->device.device_type == kDLCUDAHost || t->device.device_type == kDLCPU) && t->data) {
        cudaPointerAttributes attr;
        if (cudaPointerGetAttributes(&attr, t->data) == cudaSuccess && attr.type == cudaMemoryTypeHost &&
            attr.devicePointer)
            host_alias = attr.devicePointer;
        else
            cudaGetLastError();   // clear the lookup error of a pageable pointer
    }
    const bool pinned_host = host_alias != nullptr;
    if (t->device.device_type != kDLCUDA && t->device.device_type != kDLCUDAManaged && !pinned_host) {
        std::snprintf(buf, sizeof(buf), "%s: expected a CUDA tensor%s, got DLPack device type %d", name,
                      host_ok ? " or pinned host memory" : "", (int)t->device.device_type);
        return fail(TS_ERR_INVALID, buf);
    }
    if (!pinned_host && t->device.device_id != h->device) {
        std::snprintf(buf, sizeof(buf), "%s: tensor is on cuda:%d, the handle on cuda:%d", name,
                      (int)t->device.device_id, h->device);
        return fail(TS_ERR_INVALID, buf);
    }
    const DLDataType d = t->dtype;
    bool ok = d.lanes == 1;
    bool f64 = false;
    switch (kind) {
        case K_REAL: f64 = h->precision == TS_F64; ok = ok && d.code == kDLFloat && d.bits == (f64 ? 64 : 32); break;
        case K_F64: f64 = true; ok = ok && d.code == kDLFloat && d.bits == 64; break;
        case K_F32_OR_F64: f64 = d.bits == 64; ok = ok && d.code == kDLFloat && (d.bits == 32 || d.bits == 64); break;
        case K_I64: ok = ok && d.code == kDLInt && d.bits == 64; break;
        case K_I32: ok = ok && d.code == kDLInt && d.bits == 32; break;
        case K_U8: ok = ok && (d.code == kDLUInt || d.code == kDLBool) && d.bits == 8; break;
    }
    if (!ok) {
        static const char *want[] = {"", "float64", "float32 or float64", "int64", "int32", "uint8 or bool"};
        std::snprintf(buf, sizeof(buf), "%s: dtype (code %d, %d bits, %d lanes) is not %s", name, (int)d.code,
                      (int)d.bits, (int)d.lanes,
                      kind == K_REAL ? (h->precision == TS_F64 ? "float64 (fp64 handle)" : "float32 (fp32 handle)")
                                     : want[kind]);
        return fail(TS_ERR_INVALID, buf);
    }
    if (is_f64) *is_f64 = f64;
    bool shape_ok = t->ndim == ndim && (ndim == 0 || t->shape);
    for (int i = 0; shape_ok && i < ndim; ++i) shape_ok = shape[i] < 0 || t->shape[i] == shape[i];
    if (!shape_ok) {
        std::string got = "(";
        for (int i = 0; i < t->ndim && t->shape; ++i) got += std::to_string(t->shape[i]) + (i + 1 < t->ndim ? "," : "");
        std::string exp = "(";
        for (int i = 0; i < ndim; ++i) exp += (shape[i] < 0 ? std::string("*") : std::to_string(shape[i])) + (i + 1 < ndim ? "," : "");
        return fail(TS_ERR_INVALID, std::string(name) + ": shape " + got + ") where " + exp + ") is required");
    }
    if (t->strides) {   // compact row-major (dimensions of extent 1 may carry any stride)
        int64_t expect = 1;
        for (int i = ndim - 1; i >= 0; --i) {
            if (t->shape[i] != 1 && t->strides[i] != expect)
                return fail(TS_ERR_INVALID, std::string(name) + ": tensor is not contiguous (row-major)");
            expect *= t->shape[i];
        }
    }
    if (!t->data) {
        int64_t numel = 1;
        for (int i = 0; i < ndim; ++i) numel *= t->shape[i];
        if (numel) return fail(TS_ERR_INVALID, std::string(name) + ": null data");
    }
    void *base = pinned_host ? host_alias : t->data;
    *out = base ? reinterpret_cast<char *>(base) + t->byte_offset : nullptr;
    return TS_OK;
}

#define TS_CHECK(expr) do { int rc_ = (expr); if (rc_ != TS_OK) return rc_; } while (0)

int env_state_dl(const ts_handle *h, const ts_env_tensors *st, ts_env_state &o, int64_t &n) {
    if (!st || !st->x) return fail(TS_ERR_INVALID, "state: x required");
    if (st->x->ndim != 3 || !st->x->shape) return fail(TS_ERR_INVALID, "x: shape (N,V,3) required");
    n = st->x->shape[0];
    const int64_t V = h->n_vert;
    const int64_t nv3[3] = {n, V, 3}, n3[2] = {n, 3}, n1[1] = {n}, nv[2] = {n, V};
    void *p;
    TS_CHECK(check_dl(h, st->x, "x", K_REAL, 3, nv3, false, &o.x));
    TS_CHECK(check_dl(h, st->v, "v", K_REAL, 3, nv3, false, &o.v));
    TS_CHECK(check_dl(h, st->tool_axis, "tool_axis", K_F64, 2, n3, false, &p)); o.tool_axis = (double *)p;
    TS_CHECK(check_dl(h, st->tool_jaw, "tool_jaw", K_F64, 2, n3, false, &p)); o.tool_jaw = (double *)p;
    TS_CHECK(check_dl(h, st->tool_reach, "tool_reach", K_F64, 1, n1, false, &p)); o.tool_reach = (double *)p;
    TS_CHECK(check_dl(h, st->tool_clamp, "tool_clamp", K_F64, 1, n1, false, &p)); o.tool_clamp = (double *)p;
    TS_CHECK(check_dl(h, st->grasp_vertex, "grasp_vertex", K_I64, 1, n1, false, &p)); o.grasp_vertex = (int64_t *)p;
    TS_CHECK(check_dl(h, st->grasped, "grasped", K_U8, 2, nv, false, &p)); o.grasped = (uint8_t *)p;
    TS_CHECK(check_dl(h, st->steps, "steps", K_I64, 1, n1, false, &p)); o.steps = (int64_t *)p;
    TS_CHECK(check_dl(h, st->l_prev, "l_prev", K_F64, 1, n1, false, &p)); o.l_prev = (double *)p;
    TS_CHECK(check_dl(h, st->ep_return, "ep_return", K_F64, 1, n1, false, &p)); o.ep_return = (double *)p;
    return TS_OK;
}

int override_dl(const ts_handle *h, const ts_tool_override_tensors *t, int64_t n, ts_tool_override &o) {
    const int64_t n3[2] = {n, 3}, n1[1] = {n};
    void *p;
    TS_CHECK(check_dl(h, t->axis, "override axis", K_F64, 2, n3, false, &p)); o.axis = (const double *)p;
    TS_CHECK(check_dl(h, t->jaw, "override jaw", K_F64, 2, n3, false, &p)); o.jaw = (const double *)p;
    TS_CHECK(check_dl(h, t->reach, "override reach", K_F64, 1, n1, false, &p)); o.reach = (const double *)p;
    TS_CHECK(check_dl(h, t->clamp, "override clamp", K_F64, 1, n1, false, &p)); o.clamp = (const double *)p;
    TS_CHECK(check_dl(h, t->clipped, "override clipped", K_U8, 1, n1, true, &p)); o.clipped = (const uint8_t *)p;
    return TS_OK;
}
}  // namespace

extern "C" {

int32_t ts_env_step_dl(ts_handle *h, const ts_env_tensors *st, const DLTensor *actions,
                       const ts_step_out_tensors *out, const ts_tool_override_tensors *ovr,
                       const DLTensor *bad_action_flag, void *stream) {
    if (!h || !st || !out) return fail(TS_ERR_INVALID, "null argument");
    ts_env_state s;
    int64_t n;
    TS_CHECK(env_state_dl(h, st, s, n));
    const int64_t n3[2] = {n, 3}, n1[1] = {n}, n6[2] = {n, 6}, one[1] = {1};
    void *a = nullptr, *p;
    int a64 = 1;
    TS_CHECK(check_dl(h, actions, "actions", K_F32_OR_F64, 2, n3, ovr != nullptr, &a, &a64, true));
    ts_tool_override o{};
    if (ovr) TS_CHECK(override_dl(h, ovr, n, o));
    ts_step_out so{};
    int obs64 = 1, fin64 = -1;
    TS_CHECK(check_dl(h, out->obs, "obs", K_F32_OR_F64, 2, n6, true, &so.obs, &obs64, true));
    TS_CHECK(check_dl(h, out->final_obs, "final_obs", K_F32_OR_F64, 2, n6, true, &so.final_obs, &fin64, true));
    if (out->obs && out->final_obs && obs64 != fin64)
        return fail(TS_ERR_INVALID, "final_obs: dtype must equal obs's");
    so.obs_f64 = out->obs ? obs64 : (out->final_obs ? fin64 : 1);
    TS_CHECK(check_dl(h, out->reward, "reward", K_F64, 1, n1, true, &p, nullptr, true)); so.reward = (double *)p;
    TS_CHECK(check_dl(h, out->distance, "distance", K_F64, 1, n1, true, &p, nullptr, true)); so.distance = (double *)p;
    TS_CHECK(check_dl(h, out->episode_return, "episode_return", K_F64, 1, n1, true, &p, nullptr, true)); so.episode_return = (double *)p;
    TS_CHECK(check_dl(h, out->episode_length, "episode_length", K_I64, 1, n1, true, &p, nullptr, true)); so.episode_length = (int64_t *)p;
    TS_CHECK(check_dl(h, out->contacts, "contacts", K_I32, 1, n1, true, &p, nullptr, true)); so.contacts = (int32_t *)p;
    TS_CHECK(check_dl(h, out->terminated, "terminated", K_U8, 1, n1, true, &p, nullptr, true)); so.terminated = (uint8_t *)p;
    TS_CHECK(check_dl(h, out->truncated, "truncated", K_U8, 1, n1, true, &p, nullptr, true)); so.truncated = (uint8_t *)p;
    TS_CHECK(check_dl(h, out->success, "success", K_U8, 1, n1, true, &p, nullptr, true)); so.success = (uint8_t *)p;
    TS_CHECK(check_dl(h, out->diverged, "diverged", K_U8, 1, n1, true, &p, nullptr, true)); so.diverged = (uint8_t *)p;
    TS_CHECK(check_dl(h, out->clipped, "clipped", K_U8, 1, n1, true, &p, nullptr, true)); so.clipped = (uint8_t *)p;
    TS_CHECK(check_dl(h, out->done_mask, "done_mask", K_U8, 1, n1, true, &p, nullptr, true)); so.done_mask = (uint8_t *)p;
    void *flag = nullptr;
    TS_CHECK(check_dl(h, bad_action_flag, "bad_action_flag", K_I32, 1, one, true, &flag));
    return ts_env_step(h, &s, n, a, a ? !a64 : 0, &so, ovr ? &o : nullptr, (int32_t *)flag, stream);
}

int32_t ts_env_reset_dl(ts_handle *h, const ts_env_tensors *st, const DLTensor *mask, const DLTensor *obs,
                        void *stream) {
    if (!h || !st) return fail(TS_ERR_INVALID, "null argument");
    ts_env_state s;
    int64_t n;
    TS_CHECK(env_state_dl(h, st, s, n));
    const int64_t n1[1] = {n}, n6[2] = {n, 6};
    void *m, *o;
    int o64 = 1;
    TS_CHECK(check_dl(h, mask, "mask", K_U8, 1, n1, true, &m));
    TS_CHECK(check_dl(h, obs, "obs", K_F32_OR_F64, 2, n6, true, &o, &o64));
    return ts_env_reset(h, &s, n, (const uint8_t *)m, o, o64, stream);
}

int32_t ts_env_observe_dl(ts_handle *h, const ts_env_tensors *st, const DLTensor *obs, void *stream) {
    if (!h || !st) return fail(TS_ERR_INVALID, "null argument");
    ts_env_state s;
    int64_t n;
    TS_CHECK(env_state_dl(h, st, s, n));
    const int64_t n6[2] = {n, 6};
    void *o;
    int o64 = 1;
    TS_CHECK(check_dl(h, obs, "obs", K_F32_OR_F64, 2, n6, false, &o, &o64));
    return ts_env_observe(h, &s, n, o, o64, stream);
}

int32_t ts_sim_step_dl(ts_handle *h, const ts_env_tensors *st, const DLTensor *targets, const DLTensor *angles,
                       const ts_tool_override_tensors *ovr, const DLTensor *clipped, const DLTensor *rejected,
                       const DLTensor *diverged, const DLTensor *contacts, void *stream) {
    if (!h || !st) return fail(TS_ERR_INVALID, "null argument");
    ts_env_state s;
    int64_t n;
    TS_CHECK(env_state_dl(h, st, s, n));
    const int64_t n3[2] = {n, 3}, n1[1] = {n};
    void *t, *a, *c, *r, *d, *k;
    TS_CHECK(check_dl(h, targets, "targets", K_F64, 2, n3, true, &t));
    TS_CHECK(check_dl(h, angles, "angles", K_F64, 1, n1, true, &a));
    ts_tool_override o{};
    if (ovr) TS_CHECK(override_dl(h, ovr, n, o));
    TS_CHECK(check_dl(h, clipped, "clipped", K_U8, 1, n1, true, &c));
    TS_CHECK(check_dl(h, rejected, "rejected", K_U8, 1, n1, true, &r));
    TS_CHECK(check_dl(h, diverged, "diverged", K_U8, 1, n1, true, &d));
    TS_CHECK(check_dl(h, contacts, "contacts", K_I32, 1, n1, true, &k));
    return ts_sim_step(h, &s, n, (const double *)t, (const double *)a, ovr ? &o : nullptr, (uint8_t *)c,
                       (uint8_t *)r, (uint8_t *)d, (int32_t *)k, stream);
}

int32_t ts_run_substeps_dl(ts_handle *h, const DLTensor *x, const DLTensor *v, const DLTensor *grasp_vertex,
                           const DLTensor *drag_points, const double *gravity, double hstep, int32_t substeps,
                           double damping, void *stream) {
    if (!h || !x) return fail(TS_ERR_INVALID, "null argument");
    if (x->ndim != 3 || !x->shape) return fail(TS_ERR_INVALID, "x: shape (N,V,3) required");
    const int64_t n = x->shape[0];
    const int64_t nv3[3] = {n, h->n_vert, 3}, n3[2] = {n, 3}, n1[1] = {n};
    void *px, *pv, *pg, *pd;
    TS_CHECK(check_dl(h, x, "x", K_REAL, 3, nv3, false, &px));
    TS_CHECK(check_dl(h, v, "v", K_REAL, 3, nv3, false, &pv));
    TS_CHECK(check_dl(h, grasp_vertex, "grasp_vertex", K_I64, 1, n1, false, &pg));
    TS_CHECK(check_dl(h, drag_points, "drag_points", K_F64, 2, n3, false, &pd));
    if (n == 0) return TS_OK;
    return ts_run_substeps(h, px, pv, n, (const int64_t *)pg, (const double *)pd, gravity, hstep, substeps,
                           damping, stream);
}

int32_t ts_detect_contacts_dl(ts_handle *h, const DLTensor *x, const DLTensor *caps, const DLTensor *count,
                              const DLTensor *face, const DLTensor *cap, const DLTensor *depth, const DLTensor *dir,
                              const DLTensor *bary, void *stream) {
    if (!h || !x) return fail(TS_ERR_INVALID, "null argument");
    if (x->ndim != 3 || !x->shape) return fail(TS_ERR_INVALID, "x: shape (N,V,3) required");
    const int64_t n = x->shape[0], F3 = 3 * (int64_t)h->params.n_face;
    const int64_t nv3[3] = {n, h->n_vert, 3}, c37[3] = {n, 3, 7}, n1[1] = {n}, nf[2] = {n, F3}, nf3[3] = {n, F3, 3};
    void *px, *pc, *pn, *pf, *pk, *pd, *pr, *pb;
    TS_CHECK(check_dl(h, x, "x", K_REAL, 3, nv3, false, &px));
    TS_CHECK(check_dl(h, caps, "caps", K_F64, 3, c37, false, &pc));
    TS_CHECK(check_dl(h, count, "count", K_I32, 1, n1, false, &pn));
    TS_CHECK(check_dl(h, face, "face", K_I32, 2, nf, false, &pf));
    TS_CHECK(check_dl(h, cap, "cap", K_I32, 2, nf, false, &pk));
    TS_CHECK(check_dl(h, depth, "depth", K_F64, 2, nf, false, &pd));
    TS_CHECK(check_dl(h, dir, "dir", K_F64, 3, nf3, false, &pr));
    TS_CHECK(check_dl(h, bary, "bary", K_F64, 3, nf3, false, &pb));
    if (n == 0) return TS_OK;
    return ts_detect_contacts(h, px, n, (const double *)pc, (int32_t *)pn, (int32_t *)pf, (int32_t *)pk,
                              (double *)pd, (double *)pr, (double *)pb, stream);
}

}  // extern "C"

// ---------------------------------------------------------------------------
// small helper kernels
// ---------------------------------------------------------------------------
__global__ void check_actions_kernel(const void *actions, int f32, int64_t n, int32_t *flag) {
    __shared__ int any;
    if (threadIdx.x == 0) any = 0;
    __syncthreads();
    int bad = 0;
    for (int64_t i = threadIdx.x; i < 3 * n; i += blockDim.x) {
        const double a = f32 ? (double)reinterpret_cast<const float *>(actions)[i]
                             : reinterpret_cast<const double *>(actions)[i];
        bad |= !isfinite(a);
    }
    if (bad) atomicOr(&any, 1);
    __syncthreads();
    if (threadIdx.x == 0) *flag = any;
}

cudaError_t ts_launch_check_actions(const void *actions, int actions_f32, int64_t n, int32_t *flag,
                                    cudaStream_t stream) {
    check_actions_kernel<<<1, 1024, 0, stream>>>(actions, actions_f32, n, flag);
    return cudaGetLastError();
}

__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// element i of the whole (multi-GPU) batch depends only on (seed, counter, global index)
__global__ void uniform_kernel(double *out, int64_t n, int64_t first, uint64_t seed, uint64_t counter,
                               uint64_t *dev_counter) {
    if (dev_counter) counter = *dev_counter;   // graph replays: the counter lives on the device
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t r = splitmix64(seed ^ splitmix64(counter * 0x100000001B3ull + (uint64_t)(i + first)));
        out[i] = 2.0 * ((double)(r >> 11) * (1.0 / 9007199254740992.0)) - 1.0;
    }
}

cudaError_t ts_launch_uniform(double *out, int64_t n, int64_t first, uint64_t seed, uint64_t counter,
                              cudaStream_t stream) {
    int grid = (int)((n + 255) / 256);
    if (grid > 4096) grid = 4096;
    uniform_kernel<<<grid, 256, 0, stream>>>(out, n, first, seed, counter, nullptr);
    return cudaGetLastError();
}

__global__ void counter_kernel(uint64_t *c) { *c += 1; }

// small draws: one block reads the device counter, draws, and bumps it itself (one launch)
__global__ void __launch_bounds__(1024) uniform_bump_kernel(double *out, int64_t n, int64_t first, uint64_t seed,
                                                            uint64_t *dev_counter) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");   // the command kernel may start its prologue
    const uint64_t counter = *dev_counter;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const uint64_t r = splitmix64(seed ^ splitmix64(counter * 0x100000001B3ull + (uint64_t)(i + first)));
        out[i] = 2.0 * ((double)(r >> 11) * (1.0 / 9007199254740992.0)) - 1.0;
    }
    __syncthreads();   // every thread has read the counter
    if (threadIdx.x == 0) *dev_counter = counter + 1;
}

cudaError_t ts_launch_uniform_dev(double *out, int64_t n, int64_t first, uint64_t seed, uint64_t *counter,
                                  cudaStream_t stream) {
    if (n <= 65536) {   // <= 21845 envs: one block (a few microseconds), one launch
        uniform_bump_kernel<<<1, 1024, 0, stream>>>(out, n, first, seed, counter);
        return cudaGetLastError();
    }
    int grid = (int)((n + 255) / 256);
    if (grid > 4096) grid = 4096;
    uniform_kernel<<<grid, 256, 0, stream>>>(out, n, first, seed, 0, counter);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    counter_kernel<<<1, 1, 0, stream>>>(counter);   // stream order: after every read of *counter
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// shared-memory bandwidth probe: the measured denominator of the roofline
// (the env step is bound by on-chip shared memory, not HBM).  Every warp
// streams conflict-free 128-bit loads over a 64 KiB buffer; bytes counted =
// 16 B x 32 lanes per LDS.128 wavefront group.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) smem_probe_kernel(int iters, float *sink) {
    extern __shared__ float4 sbuf[];
    const int n4 = 4096;   // 64 KiB
    for (int i = threadIdx.x; i < n4; i += blockDim.x) sbuf[i] = make_float4(i, i + 1, i + 2, i + 3);
    __syncthreads();
    float4 acc = make_float4(0, 0, 0, 0);
    int idx = threadIdx.x;
#pragma unroll 1
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const float4 q = sbuf[(idx + k * 512) & (n4 - 1)];
            acc.x += q.x; acc.y += q.y; acc.z += q.z; acc.w += q.w;
        }
        idx = (idx + 32) & (n4 - 1);
    }
    if (acc.x + acc.y + acc.z + acc.w == 1.2345f) sink[threadIdx.x] = acc.x;
}

// The .shared address of the first dynamic shared-memory byte of a non-cluster launch (once per
// device): the fast step kernel's constant shared addresses assume TS_SMEM_WINDOW.
static __global__ void smem_window_kernel(uint32_t *out) {
    extern __shared__ __align__(16) unsigned char raw[];
    if (threadIdx.x == 0) *out = (uint32_t)__cvta_generic_to_shared(raw);
}

uint32_t ts_smem_window(int device) {
    static uint32_t cached[64];
    static bool have[64];
    if (device < 0 || device >= 64) return 0;
    if (have[device]) return cached[device];
    uint32_t *d = nullptr, v = 0;
    if (cudaMalloc(&d, sizeof(uint32_t)) == cudaSuccess) {
        smem_window_kernel<<<1, 32, 1024>>>(d);
        if (cudaMemcpy(&v, d, sizeof(uint32_t), cudaMemcpyDeviceToHost) != cudaSuccess) v = 0;
        cudaFree(d);
    }
    cached[device] = v;
    have[device] = true;
    return v;
}

extern "C" int32_t ts_smem_probe(int32_t device, int32_t iters, double *gbs_out) {
    if (!gbs_out) return fail(TS_ERR_INVALID, "null argument");
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    float *sink = nullptr;
    e = cudaMalloc(&sink, 1024 * sizeof(float));
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc");
    const int smem = 4096 * 16;
    cudaFuncSetAttribute(smem_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int grid = sms * 2, block = 1024;
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    smem_probe_kernel<<<grid, block, smem>>>(iters / 10 + 1, sink);   // warm-up
    cudaEventRecord(a);
    smem_probe_kernel<<<grid, block, smem>>>(iters, sink);
    cudaEventRecord(b);
    e = cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a); cudaEventDestroy(b);
    cudaFree(sink);
    if (e != cudaSuccess) return cuda_fail(e, "smem probe");
    g_launches.fetch_add(2);
    const double bytes = (double)grid * block * (double)iters * 8.0 * 16.0;
    *gbs_out = bytes / (ms * 1e-3) / 1e9;
    return TS_OK;
}
