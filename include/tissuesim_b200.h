/*
 * tissuesim_b200.h -- C-ABI of the B200 (sm_100a) tissue-reach environment step.
 *
 * Plain C: plain pointers and sizes, no torch or CUDA types in signatures
 * (streams are passed as void* = cudaStream_t).  Ownership: every array
 * passed in is BORROWED for the duration of the call (device arrays until
 * the launched work completes on `stream`); the library never frees caller
 * memory.  A handle owns only the compiled scene program on the device.
 * Threading: one caller per handle (the reference's env is "externally
 * single-caller"); all work is stream-ordered and graph-capturable.
 * Errors: every entry returns TS_OK (0) or a negative status; the message is
 * in ts_last_error() (thread-local).  Divergence is NOT an error in env mode
 * (flag + auto-reset, env.py:164-174).
 *
 * Which reference interface each entry replaces (paths relative to
 * /root/reference/pkg/src/tissuesim/):
 *   ts_create / ts_destroy   Simulation.__init__ state packing      solver.py:255-306
 *                            + backends.get_backend                 backends/__init__.py:37-49
 *   ts_env_step              EnvBatch.step                           env.py:144-197
 *                            (-> Simulation.step solver.py:322-366 ->
 *                                ToolBatch.apply_commands tool.py:307-345,
 *                                ToolBatch.update_grasps tool.py:372-389,
 *                                backend.run_substeps _kernels.pyx:577,
 *                                backend.detect_contacts _kernels.pyx:797,
 *                                collision.resolve_contact_arrays collision.py:55)
 *   ts_env_reset             EnvBatch.reset / Simulation.reset_instances
 *                                                                     env.py:123-142, solver.py:314-320
 *   ts_sim_step              Simulation.step (targets/angles or none) solver.py:322-366
 *   ts_run_substeps          backend.run_substeps (plugin protocol)   _kernels.pyx:577-674
 *   ts_detect_contacts       backend.detect_contacts (plugin protocol) _kernels.pyx:797-947
 */
#ifndef TISSUESIM_B200_H
#define TISSUESIM_B200_H

#include <stdint.h>

/* DLPack (https://github.com/dmlc/dlpack, ABI v1): the typed tensor descriptor of the *_dl
 * entries.  The subset below is layout-identical to dlpack.h; include dlpack.h first to use it. */
#ifndef DLPACK_MAJOR_VERSION
#ifdef __cplusplus
extern "C" {
#endif
typedef enum { kDLCPU = 1, kDLCUDA = 2, kDLCUDAHost = 3, kDLCUDAManaged = 13 } DLDeviceType;
typedef enum { kDLInt = 0, kDLUInt = 1, kDLFloat = 2, kDLBool = 6 } DLDataTypeCode;
typedef struct { DLDeviceType device_type; int32_t device_id; } DLDevice;
typedef struct { uint8_t code; uint8_t bits; uint16_t lanes; } DLDataType;
typedef struct {
    void *data;
    DLDevice device;
    int32_t ndim;
    DLDataType dtype;
    int64_t *shape;
    int64_t *strides;        /* in elements; NULL = compact row-major */
    uint64_t byte_offset;
} DLTensor;
typedef struct DLManagedTensor {
    DLTensor dl_tensor;
    void *manager_ctx;
    void (*deleter)(struct DLManagedTensor *self);
} DLManagedTensor;
#ifdef __cplusplus
}
#endif
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define TS_ABI_VERSION 3

enum ts_status {
    TS_OK = 0,
    TS_ERR_INVALID = -1,     /* bad argument / scene (maps to ValidationError) */
    TS_ERR_CUDA = -2,        /* CUDA runtime failure */
    TS_ERR_NOMEM = -3,
    TS_ERR_UNSUPPORTED = -4  /* layout does not fit the device (e.g. shared memory) */
};

enum ts_precision { TS_F32 = 0, TS_F64 = 1 };

/* Scene description: everything Simulation/EnvBatch derive from a scene
 * (mesh.py:508-524 + solver.py:264-301 + env.py:40-58).  All host pointers,
 * float64 / int32, vertex indices in the scene's original numbering. */
typedef struct ts_scene_desc {
    int32_t n_vert, n_edge, n_tet, n_face, n_att;
    const double *positions_rest;  /* (V,3) */
    const double *inverse_mass;    /* (V,)  0 for pinned */
    const int32_t *edges;          /* (E,2) */
    const double *rest_length;     /* (E,)  */
    const int32_t *tets;           /* (T,4) */
    const double *rest_volume;     /* (T,)  */
    const int32_t *faces;          /* (F,3) surface faces, outward winding */
    const int32_t *att_vertex;     /* (A,)  */
    const int32_t *att_faces;      /* (A,3) face vertex ids (ignored for anchors) */
    const uint8_t *att_is_face;    /* (A,)  */
    const double *att_anchor;      /* (A,3) */
    const double *att_rest;        /* (A,)  */
    const double *att_k;           /* (A,)  */
    /* solver (SceneConfig, mesh.py:66-71) */
    double dt; int32_t substeps; double gravity[3]; double k_s, k_v, damping;
    double k_contact; int32_t contact_iterations;           /* solver.py:258 defaults 1.0, 8 */
    /* tool (mesh.py:74-80); start pose precomputed by the host exactly as
     * ToolModel.from_config (tool.py:161-173) */
    double rcm[3]; double shaft_radius, clamp_radius, clamp_length, grasp_radius2;
    double start_axis[3], start_jaw[3], start_reach, start_clamp;
    double held_clamp_angle, held_cos, held_sin;   /* cos/sin(radians(held)) from the host */
    /* task (mesh.py:83-92, env.py:24-58) */
    double target[3], action_scale, success_threshold;
    double w_distance, w_delta, w_success, reward_scale;
    double workspace_low[3], workspace_high[3];
    int64_t max_episode_steps;
    double start_distance;          /* |drag(start) - target|, env.py:103-108 */
    double target_obs[3];           /* normalized target, env.py:99-101 */
} ts_scene_desc;

/* Layout options for the scene compiler (0 = automatic). */
typedef struct ts_layout_opts {
    int32_t precision;          /* ts_precision */
    int32_t block_threads;      /* CTA size; default 32*ceil(free_verts/32) */
    int32_t max_chunk_slots;    /* slot budget per constraint chunk (0 = auto) */
    int32_t schedule_banks;     /* 1 = bank-conflict-aware item schedule (default), -1 = off */
    int32_t smem_budget;        /* bytes of shared memory per CTA to aim for (0 = auto) */
    int32_t compact;            /* 16-bit item streams when possible (default), -1 = off */
    int32_t edge_gather;        /* distance constraints gathered by the owner of each free vertex
                                   (default, 0/1), -1 = constraint-parallel phase 1 + slots */
    int32_t cluster_size;       /* CTAs per environment: 0 = auto (one CTA when the mesh fits, else the
                                   smallest thread-block cluster that holds it), 1 = one CTA, 2..16 */
    int32_t refine_iters;       /* bank-schedule search iterations: 0 = thorough default (3000 per item,
                                   at most 4 M; seconds), -1 = quick (150 per item), > 0 = explicit */
} ts_layout_opts;

typedef struct ts_layout_info {
    int32_t precision, block_threads, vertices_per_thread, n_chunks;
    int32_t n_free, n_store, slot_capacity, smem_bytes;
    int32_t n_edge_items, n_tet_items, n_att_items, n_slots_total;
    int32_t bank_conflicts_p1;  /* residual phase-1 conflicts of the schedule (extra wavefronts / substep) */
    int32_t compact;            /* 1 when the program uses the 16-bit item streams */
    int32_t edge_gather;        /* 1 when distance constraints are owner-gathered */
    int32_t n_edge_incidences;  /* (edge, free endpoint) records of the owner gather */
    int32_t slot_budget;        /* slot budget per chunk the compiler used */
    int32_t cluster_size;       /* CTAs per environment (1, or the thread-block cluster size) */
    int64_t program_bytes;
} ts_layout_info;

/* Per-env state: caller-owned DEVICE arrays, C-contiguous.
 * Real = float (TS_F32) or double (TS_F64). */
typedef struct ts_env_state {
    void *x;                 /* (N,V,3) Real  positions   (Simulation.x) */
    void *v;                 /* (N,V,3) Real  velocities  (Simulation.v) */
    double *tool_axis;       /* (N,3)  ToolBatch.axis */
    double *tool_jaw;        /* (N,3)  ToolBatch.jaw_dir */
    double *tool_reach;      /* (N,)   ToolBatch.reach */
    double *tool_clamp;      /* (N,)   ToolBatch.clamp_angle (degrees) */
    int64_t *grasp_vertex;   /* (N,)   -1 = none */
    uint8_t *grasped;        /* (N,V)  per-vertex grasp flag */
    int64_t *steps;          /* (N,)   EnvBatch._steps */
    double *l_prev;          /* (N,)   EnvBatch._l_prev */
    double *ep_return;       /* (N,)   EnvBatch._return */
} ts_env_state;

/* Outputs of one env step (DEVICE arrays; any may be NULL to skip). */
typedef struct ts_step_out {
    void *obs;               /* (N,6) float32 or float64 (obs_f64) */
    double *reward;          /* (N,) */
    uint8_t *terminated;     /* (N,) */
    uint8_t *truncated;      /* (N,) */
    double *distance;        /* (N,) info["distance"] */
    uint8_t *success;        /* (N,) */
    uint8_t *diverged;       /* (N,) */
    uint8_t *clipped;        /* (N,) */
    int32_t *contacts;       /* (N,) contacts resolved this step */
    double *episode_return;  /* (N,) before auto-reset */
    int64_t *episode_length; /* (N,) before auto-reset */
    uint8_t *done_mask;      /* (N,) */
    void *final_obs;         /* (N,6) same dtype as obs; zero rows when not done */
    int32_t obs_f64;
} ts_step_out;

/* Optional externally supplied tool poses (validation: inject the oracle's
 * post-command poses so transcendental-function ulps do not enter). */
typedef struct ts_tool_override {
    const double *axis, *jaw, *reach, *clamp;  /* (N,3),(N,3),(N,),(N,) post-command */
    const uint8_t *clipped;                    /* (N,) */
} ts_tool_override;

typedef struct ts_handle ts_handle;

const char *ts_last_error(void);
int32_t ts_abi_version(void);

int32_t ts_create(const ts_scene_desc *desc, const ts_layout_opts *opts, int32_t device,
                  ts_handle **out);
/* ts_create from a program ts_compile_program made earlier (same library build, same scene):
 * skips the compile (the bank-schedule search takes seconds).  `info` is what the compile
 * reported.  Replaces the same reference step as ts_create. */
int32_t ts_create_from_program(const ts_scene_desc *desc, const void *program, int64_t bytes,
                               const ts_layout_info *info, int32_t device, ts_handle **out);
int32_t ts_destroy(ts_handle *h);
int32_t ts_query(const ts_handle *h, ts_layout_info *info);

/* Host-side copy of the compiled scene program (for inspection/tests; no GPU needed).
 * Call with buf=NULL to get the size. */
int32_t ts_compile_program(const ts_scene_desc *desc, const ts_layout_opts *opts,
                           void *buf, int64_t *bytes, ts_layout_info *info);

/* EnvBatch.step on device.  actions: (N,3) device float64 (actions_f32=0) or
 * float32.  If `bad_action_flag` is non-NULL the step first checks every
 * action for finiteness; if any is non-finite NO state is modified and
 * *bad_action_flag (device int32) is set to 1 (deferred ValidationError). */
int32_t ts_env_step(ts_handle *h, const ts_env_state *st, int64_t num_envs,
                    const void *actions, int32_t actions_f32,
                    const ts_step_out *out, const ts_tool_override *ovr,
                    int32_t *bad_action_flag, void *stream);

/* EnvBatch.reset for rows with mask[i] != 0 (mask NULL = all rows).
 * obs (optional, (N,6)) receives observations of ALL rows (caller slices). */
int32_t ts_env_reset(ts_handle *h, const ts_env_state *st, int64_t num_envs,
                     const uint8_t *mask, void *obs, int32_t obs_f64, void *stream);

/* Observations (N,6) of all rows from the current tool state (EnvBatch._observe_rows). */
int32_t ts_env_observe(ts_handle *h, const ts_env_state *st, int64_t num_envs, void *obs,
                       int32_t obs_f64, void *stream);

/* Cap the grid (0 = one CTA per environment); CTAs then loop over environments. */
int32_t ts_set_max_grid(ts_handle *h, int32_t max_grid);

/* Simulation.step: targets (N,3) float64 device or NULL (no command), angles
 * (N,) or NULL (keep).  Outputs optional: clipped, rejected, diverged (u8),
 * contacts (i32), all (N,). */
int32_t ts_sim_step(ts_handle *h, const ts_env_state *st, int64_t num_envs,
                    const double *targets, const double *angles,
                    const ts_tool_override *ovr,
                    uint8_t *clipped, uint8_t *rejected, uint8_t *diverged, int32_t *contacts,
                    void *stream);

/* Plugin protocol run_substeps: x, v (N,V,3) Real, grasp_vertex (N,) int64,
 * drag_points (N,3) float64 -- DEVICE arrays; topology, k_s, k_v come from the
 * handle (create a handle for the arrays you want to run); gravity (host,
 * 3 doubles), step h, substeps and damping are per call as in the reference
 * (_kernels.pyx:577-592).  In place on x, v. */
int32_t ts_run_substeps(ts_handle *h, void *x, void *v, int64_t num_envs,
                        const int64_t *grasp_vertex, const double *drag_points,
                        const double *gravity, double hstep, int32_t substeps, double damping,
                        void *stream);

/* Plugin protocol detect_contacts for N position sets against N×3 capsule
 * rows (N,3,7) float64.  Outputs (DEVICE): count (N,) int32 and, per env,
 * rows in emission order (capsule-major, face-minor) into arrays with
 * capacity 3F per env: face (N,3F) i32, cap (N,3F) i32, depth (N,3F) f64,
 * dir (N,3F,3) f64, bary (N,3F,3) f64. */
int32_t ts_detect_contacts(ts_handle *h, const void *x, int64_t num_envs, const double *caps,
                           int32_t *count, int32_t *face, int32_t *cap, double *depth,
                           double *dir, double *bary, void *stream);

/* ---- Typed (DLPack) entries: the product boundary ------------------------------------------
 * The same calls as above with every array passed as a DLTensor (what torch.utils.dlpack /
 * __dlpack__ hand over, zero-copy).  Each tensor is checked before anything is launched:
 * device (kDLCUDA / kDLCUDAManaged on the handle's device), dtype (code, bits, lanes = 1),
 * ndim, shape (N from x's leading dimension, V from the scene) and compact row-major strides;
 * byte_offset is honoured.  Any mismatch returns TS_ERR_INVALID naming the tensor, the way the
 * reference's typed memoryviews reject a wrong buffer at entry (_kernels.pyx:577-585).
 * Dtypes: x, v Real = float32 (TS_F32 handle) / float64 (TS_F64); tool_* float64;
 * grasp_vertex, steps int64; grasped uint8 or bool; l_prev, ep_return float64.
 * ts_env_step_dl also takes its actions and step outputs in pinned host memory (kDLCUDAHost, or
 * kDLCPU at a page-locked address, as torch exports torch.empty(..., pin_memory=True)): the
 * command kernel reads the actions and the epilogue writes the outputs in place over the bus
 * (zero-copy; EnvBatch.step_numpy does this).  Pageable host memory is rejected. */
typedef struct ts_env_tensors {
    const DLTensor *x, *v;                                   /* (N,V,3) Real */
    const DLTensor *tool_axis, *tool_jaw;                    /* (N,3) f64 */
    const DLTensor *tool_reach, *tool_clamp;                 /* (N,) f64 */
    const DLTensor *grasp_vertex;                            /* (N,) i64 */
    const DLTensor *grasped;                                 /* (N,V) u8/bool */
    const DLTensor *steps;                                   /* (N,) i64 */
    const DLTensor *l_prev, *ep_return;                      /* (N,) f64 */
} ts_env_tensors;

/* Outputs (any may be NULL): obs / final_obs (N,6) float32 or float64 (both the same dtype),
 * reward / distance / episode_return (N,) f64, flags (N,) bool/u8, contacts (N,) i32,
 * episode_length (N,) i64. */
typedef struct ts_step_out_tensors {
    const DLTensor *obs, *reward, *terminated, *truncated, *distance, *success, *diverged, *clipped;
    const DLTensor *contacts, *episode_return, *episode_length, *done_mask, *final_obs;
} ts_step_out_tensors;

/* Tool-pose injection, typed: axis, jaw (N,3) f64; reach, clamp (N,) f64; clipped (N,) u8/bool
 * or NULL. */
typedef struct ts_tool_override_tensors {
    const DLTensor *axis, *jaw, *reach, *clamp, *clipped;
} ts_tool_override_tensors;

/* EnvBatch.step (env.py:144-197): actions (N,3) float32/float64 on the device (or NULL with an
 * override); bad_action_flag (1,) int32 or NULL, as ts_env_step. */
int32_t ts_env_step_dl(ts_handle *h, const ts_env_tensors *st, const DLTensor *actions,
                       const ts_step_out_tensors *out, const ts_tool_override_tensors *ovr,
                       const DLTensor *bad_action_flag, void *stream);

/* EnvBatch.reset (env.py:123-142): mask (N,) u8/bool or NULL (all rows); obs (N,6) f32/f64 or
 * NULL. */
int32_t ts_env_reset_dl(ts_handle *h, const ts_env_tensors *st, const DLTensor *mask,
                        const DLTensor *obs, void *stream);

/* EnvBatch._observe_rows (env.py:99-115): obs (N,6) f32/f64 of all rows. */
int32_t ts_env_observe_dl(ts_handle *h, const ts_env_tensors *st, const DLTensor *obs, void *stream);

/* Simulation.step (solver.py:322-366): targets (N,3) f64 or NULL, angles (N,) f64 or NULL;
 * outputs clipped / rejected / diverged (N,) bool/u8, contacts (N,) i32, each optional. */
int32_t ts_sim_step_dl(ts_handle *h, const ts_env_tensors *st, const DLTensor *targets,
                       const DLTensor *angles, const ts_tool_override_tensors *ovr,
                       const DLTensor *clipped, const DLTensor *rejected, const DLTensor *diverged,
                       const DLTensor *contacts, void *stream);

/* backend.run_substeps (_kernels.pyx:577-592): x, v (N,V,3) Real, grasp_vertex (N,) i64,
 * drag_points (N,3) f64; gravity host (3) doubles. */
int32_t ts_run_substeps_dl(ts_handle *h, const DLTensor *x, const DLTensor *v,
                           const DLTensor *grasp_vertex, const DLTensor *drag_points,
                           const double *gravity, double hstep, int32_t substeps, double damping,
                           void *stream);

/* backend.detect_contacts (_kernels.pyx:797-947): x (N,V,3) Real, caps (N,3,7) f64; count (N,)
 * i32, face / cap (N,3F) i32, depth (N,3F) f64, dir / bary (N,3F,3) f64. */
int32_t ts_detect_contacts_dl(ts_handle *h, const DLTensor *x, const DLTensor *caps,
                              const DLTensor *count, const DLTensor *face, const DLTensor *cap,
                              const DLTensor *depth, const DLTensor *dir, const DLTensor *bary,
                              void *stream);

/* Uniform(-1,1) actions (N,3) float64 on device from a counter-based hash of
 * (seed, counter, global env index first_env + i): a multi-GPU shard draws
 * exactly the actions the single-GPU run draws for the same global envs. */
int32_t ts_uniform_actions(double *actions, int64_t num_envs, int64_t first_env, uint64_t seed,
                           uint64_t counter, void *stream);

/* The same draw with the counter in DEVICE memory (uint64), incremented by the call in stream
 * order: a captured CUDA graph replays a fresh action batch every time. */
int32_t ts_uniform_actions_dev(double *actions, int64_t num_envs, int64_t first_env, uint64_t seed,
                               uint64_t *counter, void *stream);

/* Measured shared-memory bandwidth of the device (GB/s, whole GPU): the
 * roofline denominator for the on-chip-bound env step. */
int32_t ts_smem_probe(int32_t device, int32_t iters, double *gbs_out);

/* Kernel launches issued by this library since load (for bench accounting). */
int64_t ts_launch_count(void);

/* Device time of the fused step kernel alone (the roofline's denominator): while enabled, every
 * step-kernel launch of this handle is bracketed by CUDA events on its own stream (capacity
 * `max_launches`, further launches are not timed).  ts_kernel_time waits for the recorded
 * events, returns the summed milliseconds and the number of timed launches, and clears them.
 * enable = 0 releases the events. */
int32_t ts_kernel_timing(ts_handle *h, int32_t enable, int32_t max_launches);
int32_t ts_kernel_time(ts_handle *h, double *total_ms, int64_t *launches);

/* Name of the fused step kernel this handle launches (the layout-specialised instantiation the
 * program selects), as ncu prints it -- for profiles and the bench's roofline line. */
const char *ts_step_kernel_name(ts_handle *h);

/* Launch an instantiated CUDA graph (cudaGraphExec_t) on `stream` and wait for it: the steady
 * state of the host-buffer step (EnvBatch.step_numpy: the recorded H2D action copy, the step's
 * kernels and the D2H output copy) in one call. */
int32_t ts_graph_launch_sync(void *graph_exec, void *stream);

/* The same in two halves: launch (asynchronous) and wait for the stream -- the caller does host
 * work (the next output block's allocation) while the graph runs. */
int32_t ts_graph_launch(void *graph_exec, void *stream);
int32_t ts_stream_sync(void *stream);

#ifdef __cplusplus
}
#endif
#endif /* TISSUESIM_B200_H */
