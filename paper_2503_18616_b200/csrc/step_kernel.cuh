// step_kernel.cuh -- the fused tissue-reach environment step for sm_100a.
//
// One CTA owns one environment for the whole outer step (grid-stride over
// environments).  Positions live in shared memory (SoA, storage order), each
// free vertex's velocity lives in the registers of its owner thread, and the
// step never touches HBM between loading the state and writing it back:
//
//   tool command + capsule rows     thread 0, fp64      tool.py:307-370
//   grasp release / nearest vertex  block argmin, fp64  tool.py:372-389
//   substeps x S:                                        _kernels.pyx:260-352
//     predict                       owner threads
//     per constraint chunk:
//       phase 1  constraint-parallel: correction vectors -> slots (smem)
//       phase 2  vertex-parallel: owner sums its slots in reference order
//     apply + damping (+ next predict)   owner threads
//   contacts: face-parallel AABB + PGD witness search,   _kernels.pyx:797-947
//             then ordered sequential push-out            collision.py:55-73
//   divergence guard                                      solver.py:357-365
//   reward / done / auto-reset / obs                      env.py:144-197
//
// Real = double with -fmad=false reproduces the reference's fp64 arithmetic
// bit for bit (same expression trees, same per-vertex summation order).
// Real = float is the throughput build (same algorithm, fp32 storage).
#pragma once
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <type_traits>

#include "step_common.h"

// loop unroll factors of the fast kernel's hot loops (development overrides: -DTS_TET_UNROLL=...)
#ifndef TS_TET_UNROLL
#define TS_TET_UNROLL 2
#endif
#ifndef TS_SLOT_UNROLL
#define TS_SLOT_UNROLL 4
#endif
#ifndef TS_EDGE_UNROLL
#define TS_EDGE_UNROLL 4
#endif
constexpr int kTetUnroll = TS_TET_UNROLL, kSlotUnroll = TS_SLOT_UNROLL, kEdgeUnroll = TS_EDGE_UNROLL;

namespace tsk {

template <typename Real> struct R4;
template <> struct R4<float> { using T = float4; };
template <> struct R4<double> { using T = double4; };

__device__ __forceinline__ double cmin(double a, double b) { return (b < a) ? b : a; }   // Cython min()
__device__ __forceinline__ double cmax(double a, double b) { return (b > a) ? b : a; }   // Cython max()
__device__ __forceinline__ float cmin(float a, float b) { return (b < a) ? b : a; }
__device__ __forceinline__ float cmax(float a, float b) { return (b > a) ? b : a; }

// fp32 build: single-MUFU approximations (arguments are normal: guarded by the degeneracy tests)
__device__ __forceinline__ float rsqrt_ftz(float x) {
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float rcp_ftz(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
// contact narrow phase arithmetic: IEEE in the fp64 (bitwise) build, single-MUFU in fp32
template <typename Real> __device__ __forceinline__ Real cdiv(Real a, Real b);
template <> __device__ __forceinline__ double cdiv<double>(double a, double b) { return a / b; }
template <> __device__ __forceinline__ float cdiv<float>(float a, float b) { return a * rcp_ftz(b); }
__device__ __forceinline__ double csqrt(double x) { return sqrt(x); }
__device__ __forceinline__ float csqrt(float x) {
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
// solver constant in the build's precision (fp32 copies live in TsParams, no F2F in the loops)
template <typename Real> __device__ __forceinline__ Real prm(double d, float f);
template <> __device__ __forceinline__ double prm<double>(double d, float) { return d; }
template <> __device__ __forceinline__ float prm<float>(double, float f) { return f; }

__device__ __forceinline__ double dot3(const double *u, const double *w) {
    return u[0] * w[0] + u[1] * w[1] + u[2] * w[2];
}
__device__ __forceinline__ void cross3(const double *u, const double *w, double *o) {
    o[0] = u[1] * w[2] - u[2] * w[1];
    o[1] = u[2] * w[0] - u[0] * w[2];
    o[2] = u[0] * w[1] - u[1] * w[0];
}
__device__ __forceinline__ double norm3(const double *u) { return sqrt(dot3(u, u)); }

using Pose = TsPose;

// perpendicular_unit, tool.py:55-62
static __device__ void some_perpendicular(const double *a, double *out) {
    const bool z = fabs(a[0]) > 0.9;
    double ref[3] = {z ? 0.0 : 1.0, 0.0, z ? 1.0 : 0.0};
    const double d = dot3(a, ref);
    for (int c = 0; c < 3; ++c) out[c] = ref[c] - a[c] * d;
    const double n = norm3(out);
    for (int c = 0; c < 3; ++c) out[c] = out[c] / n;
}

// rotate_about_axis (Rodrigues), tool.py:47-52
static __device__ void rodrigues(const double *vec, const double *k, double c, double s, double *out) {
    double kx[3];
    cross3(k, vec, kx);
    const double kv = dot3(k, vec);
    for (int i = 0; i < 3; ++i) out[i] = (vec[i] * c + kx[i] * s) + k[i] * kv * (1.0 - c);
}

// ToolBatch.apply_commands for one row, tool.py:307-345
static __device__ __forceinline__ void apply_command(const TsParams &S, Pose &p, const double *tgt, double angle,
                              bool &clipped, bool &rejected) {
    double b[3];
    clipped = false;
    for (int c = 0; c < 3; ++c) {
        double t = tgt[c];
        double m = t > S.lo[c] ? t : S.lo[c];        // np.maximum (finite inputs)
        m = m < S.hi[c] ? m : S.hi[c];               // np.minimum
        b[c] = m;
        clipped |= (m != t);
    }
    double v1[3], v2[3];
    for (int c = 0; c < 3; ++c) {
        v1[c] = (S.rcm[c] + p.reach * p.ax[c]) - S.rcm[c];   // drag_points() - rcm
        v2[c] = b[c] - S.rcm[c];
    }
    const double n1 = norm3(v1), n2 = norm3(v2);
    rejected = n2 < 1e-9;
    const double n2s = rejected ? 1.0 : n2;
    double cosang = dot3(v1, v2) / (n1 * n2s);
    cosang = cosang < -1.0 ? -1.0 : (cosang > 1.0 ? 1.0 : cosang);
    double theta = acos(cosang);
    double k[3];
    cross3(v1, v2, k);
    const double kn = norm3(k);
    bool rot = (theta > 1e-9) && (kn > 0.0) && !rejected;
    if (rot) { for (int c = 0; c < 3; ++c) k[c] = k[c] / kn; }
    else { k[0] = k[1] = k[2] = 0.0; }
    if ((theta > 1e-9) && (kn == 0.0) && !rejected) {
        double u[3];
        for (int c = 0; c < 3; ++c) u[c] = v1[c] / n1;
        some_perpendicular(u, k);
        rot = true;
    }
    if (!rot) theta = 0.0;
    if (rejected) return;
    if (rot) {
        const double c = cos(theta), s = sin(theta);
        double axn[3], jwn[3];
        rodrigues(p.ax, k, c, s, axn);
        const double na = norm3(axn);
        for (int i = 0; i < 3; ++i) axn[i] = axn[i] / na;
        rodrigues(p.jw, k, c, s, jwn);
        const double d = dot3(axn, jwn);
        for (int i = 0; i < 3; ++i) jwn[i] = jwn[i] - axn[i] * d;
        const double nj = norm3(jwn);
        for (int i = 0; i < 3; ++i) { p.ax[i] = axn[i]; p.jw[i] = jwn[i] / nj; }
    }
    p.reach = p.reach + (n2 - n1);
    p.clamp = angle;
}

// ToolBatch.capsule_rows for one row, tool.py:347-370
static __device__ __forceinline__ void capsule_rows(const TsParams &S, const Pose &p, double rows[3][7]) {
    double piv[3];
    for (int c = 0; c < 3; ++c) piv[c] = S.rcm[c] + (p.reach - S.clamp_len) * p.ax[c];
    double ca, sa;
    if (p.clamp == S.held_angle) { ca = S.held_cos; sa = S.held_sin; }
    else {
        const double alpha = p.clamp * (3.141592653589793 / 180.0);  // np.radians
        ca = cos(alpha); sa = sin(alpha);
    }
    double base[3] = {S.rcm[0], S.rcm[1], S.rcm[2]};
    double dpb[3] = {piv[0] - base[0], piv[1] - base[1], piv[2] - base[2]};
    if (norm3(dpb) < 1e-9)
        for (int c = 0; c < 3; ++c) base[c] = piv[c] - 1e-6 * p.ax[c];
    for (int c = 0; c < 3; ++c) {
        const double da = ca * p.ax[c] + sa * p.jw[c];
        const double db = ca * p.ax[c] - sa * p.jw[c];
        rows[0][c] = base[c]; rows[0][3 + c] = piv[c];
        rows[1][c] = piv[c]; rows[1][3 + c] = piv[c] + S.clamp_len * da;
        rows[2][c] = piv[c]; rows[2][3 + c] = piv[c] + S.clamp_len * db;
    }
    rows[0][6] = S.shaft_r; rows[1][6] = S.clamp_r; rows[2][6] = S.clamp_r;
}

// ---------------------------------------------------------------------------
// capsule SDF (Real), _kernels.pyx:732-794
// ---------------------------------------------------------------------------
template <typename Real>
struct Cap { Real p0[3], seg[3], dd, radius, fb[3], lo[3], hi[3]; };

template <typename Real>
__device__ void make_cap(const double *row, Cap<Real> &C) {
    for (int k = 0; k < 3; ++k) { C.p0[k] = (Real)row[k]; C.seg[k] = (Real)row[3 + k] - (Real)row[k]; }
    C.radius = (Real)row[6];
    C.dd = C.seg[0] * C.seg[0] + C.seg[1] * C.seg[1] + C.seg[2] * C.seg[2];
    if (C.dd <= (Real)0) C.dd = (Real)1;
    C.fb[0] = (Real)0; C.fb[1] = C.seg[2]; C.fb[2] = -C.seg[1];
    Real fn = C.fb[0] * C.fb[0] + C.fb[1] * C.fb[1] + C.fb[2] * C.fb[2];
    if (fn < (Real)1e-20) {
        C.fb[0] = -C.seg[2]; C.fb[1] = (Real)0; C.fb[2] = C.seg[0];
        fn = C.fb[0] * C.fb[0] + C.fb[1] * C.fb[1] + C.fb[2] * C.fb[2];
    }
    fn = sqrt(fn);
    if (fn > (Real)0) { C.fb[0] /= fn; C.fb[1] /= fn; C.fb[2] /= fn; }
    for (int k = 0; k < 3; ++k) {
        C.lo[k] = cmin((Real)row[k], (Real)row[3 + k]) - C.radius;
        C.hi[k] = cmax((Real)row[k], (Real)row[3 + k]) + C.radius;
    }
}

template <typename Real>
__device__ __forceinline__ Real cap_sd(const Cap<Real> &C, const Real *q, Real *grad) {
    Real t = cdiv<Real>((q[0] - C.p0[0]) * C.seg[0] + (q[1] - C.p0[1]) * C.seg[1] + (q[2] - C.p0[2]) * C.seg[2], C.dd);
    if (t < (Real)0) t = (Real)0;
    else if (t > (Real)1) t = (Real)1;
    const Real dx = q[0] - (C.p0[0] + t * C.seg[0]);
    const Real dy = q[1] - (C.p0[1] + t * C.seg[1]);
    const Real dz = q[2] - (C.p0[2] + t * C.seg[2]);
    const Real nrm = csqrt(dx * dx + dy * dy + dz * dz);
    if (grad) {
        if (nrm > (Real)1e-12) { grad[0] = cdiv<Real>(dx, nrm); grad[1] = cdiv<Real>(dy, nrm); grad[2] = cdiv<Real>(dz, nrm); }
        else { grad[0] = C.fb[0]; grad[1] = C.fb[1]; grad[2] = C.fb[2]; }
    }
    return nrm - C.radius;
}

template <typename Real>
__device__ __forceinline__ void simplex3(Real *b) {
    Real u0 = b[0], u1 = b[1], u2 = b[2], tmp, theta;
    if (u0 < u1) { tmp = u0; u0 = u1; u1 = tmp; }
    if (u1 < u2) { tmp = u1; u1 = u2; u2 = tmp; }
    if (u0 < u1) { tmp = u0; u0 = u1; u1 = tmp; }
    if (u2 - cdiv<Real>(u0 + u1 + u2 - (Real)1, (Real)3) > (Real)0) theta = cdiv<Real>(u0 + u1 + u2 - (Real)1, (Real)3);
    else if (u1 - (u0 + u1 - (Real)1) / (Real)2 > (Real)0) theta = (u0 + u1 - (Real)1) / (Real)2;
    else theta = u0 - (Real)1;
    b[0] = cmax(b[0] - theta, (Real)0);
    b[1] = cmax(b[1] - theta, (Real)0);
    b[2] = cmax(b[2] - theta, (Real)0);
}

template <typename Real>
__device__ __forceinline__ void bary_pt(const Real *b, const Real *pa, const Real *pb, const Real *pc, Real *o) {
    o[0] = b[0] * pa[0] + b[1] * pb[0] + b[2] * pc[0];
    o[1] = b[0] * pa[1] + b[1] * pb[1] + b[2] * pc[1];
    o[2] = b[0] * pa[2] + b[1] * pb[2] + b[2] * pc[2];
}

// Narrow phase of one (face, capsule) pair that passed the AABB test.
// Returns sd; fills depth/dir/bary when sd < 0.
template <typename Real>
__device__ __forceinline__ Real witness_body(const Cap<Real> &C, const Real *pa_, const Real *pb_, const Real *pc_,
                                             int iters, Real *dir, Real *bary_out) {
    // register copies: the outputs live on the caller's stack and could alias the inputs
    const Real pa[3] = {pa_[0], pa_[1], pa_[2]}, pb[3] = {pb_[0], pb_[1], pb_[2]}, pc[3] = {pc_[0], pc_[1], pc_[2]};
    Real bary[3];
    const Real s0 = cap_sd<Real>(C, pa, nullptr);
    const Real s1 = cap_sd<Real>(C, pb, nullptr);
    const Real s2 = cap_sd<Real>(C, pc, nullptr);
    int vb = 0;
    Real best = s0;
    if (s1 < best) { vb = 1; best = s1; }
    if (s2 < best) { vb = 2; best = s2; }
    bary[0] = vb == 0 ? (Real)1 : (Real)0;
    bary[1] = vb == 1 ? (Real)1 : (Real)0;
    bary[2] = vb == 2 ? (Real)1 : (Real)0;
    Real pt[3], g[3], gb[3];
    Real step = (Real)0.5;
    for (int it = 0; it < iters; ++it) {
        bary_pt(bary, pa, pb, pc, pt);
        cap_sd<Real>(C, pt, g);
        gb[0] = g[0] * pa[0] + g[1] * pa[1] + g[2] * pa[2];
        gb[1] = g[0] * pb[0] + g[1] * pb[1] + g[2] * pb[2];
        gb[2] = g[0] * pc[0] + g[1] * pc[1] + g[2] * pc[2];
        const Real mean_g = cdiv<Real>(gb[0] + gb[1] + gb[2], (Real)3);
        gb[0] -= mean_g; gb[1] -= mean_g; gb[2] -= mean_g;
        const Real mag = cmax(cmax(fabs(gb[0]), fabs(gb[1])), fabs(gb[2]));
        bary[0] -= cdiv<Real>(step * gb[0], mag + (Real)1e-30);
        bary[1] -= cdiv<Real>(step * gb[1], mag + (Real)1e-30);
        bary[2] -= cdiv<Real>(step * gb[2], mag + (Real)1e-30);
        simplex3(bary);
        step *= (Real)0.7;
    }
    bary_pt(bary, pa, pb, pc, pt);
    Real sd = cap_sd<Real>(C, pt, g);
    if (sd > best) {
        bary[0] = vb == 0 ? (Real)1 : (Real)0;
        bary[1] = vb == 1 ? (Real)1 : (Real)0;
        bary[2] = vb == 2 ? (Real)1 : (Real)0;
        bary_pt(bary, pa, pb, pc, pt);
        sd = cap_sd<Real>(C, pt, g);
    }
    dir[0] = g[0]; dir[1] = g[1]; dir[2] = g[2];
    bary_out[0] = bary[0]; bary_out[1] = bary[1]; bary_out[2] = bary[2];
    return sd;
}
// fp32 kernels inline the narrow phase (no call frame: 0.522 -> 0.514 ms per 4096-env step); the
// fp64 kernels keep it a call (inlined they spill more: 2.966 -> 2.998 ms)
static __device__ __noinline__ double witness_f64(const Cap<double> &C, const double *pa, const double *pb, const double *pc,
                                           int iters, double *dir, double *bary) {
    return witness_body<double>(C, pa, pb, pc, iters, dir, bary);
}

template <typename Real>
__device__ __forceinline__ Real witness(const Cap<Real> &C, const Real *pa, const Real *pb, const Real *pc, int iters,
                                        Real *dir, Real *bary) {
    if constexpr (sizeof(Real) == 8) return witness_f64(C, pa, pb, pc, iters, dir, bary);
    else return witness_body<Real>(C, pa, pb, pc, iters, dir, bary);
}

template <typename Real> __device__ __forceinline__ Real fused_sq3(Real a, Real b, Real c);
// b @ b for the contact barycentrics: numpy dispatches to BLAS ddot, which
// evaluates fma(b2,b2, fma(b1,b1, b0*b0)) on the reference hosts.
template <> __device__ __forceinline__ double fused_sq3<double>(double a, double b, double c) {
    return __fma_rn(c, c, __fma_rn(b, b, a * a));
}
template <> __device__ __forceinline__ float fused_sq3<float>(float a, float b, float c) {
    return __fmaf_rn(c, c, __fmaf_rn(b, b, a * a));
}

// ---------------------------------------------------------------------------
// shared scalar block
// ---------------------------------------------------------------------------
struct Scal {
    double caps[3][7];
    double drag[3];
    double red_key[32];
    int red_idx[32];
    int gv_orig;        // grasp vertex, original id (-1 none)
    int need_search;
    int done;
    int n_contacts;
    // cluster mode: per-rank exchange slots (used in rank 0's copy) and local results
    double cl_key[TS_MAX_CLUSTER];
    int cl_idx[TS_MAX_CLUSTER];
    int cl_flag[TS_MAX_CLUSTER];
    int n_list;
    int any_bad;
};

// Component c of element i of an (n, 3) array-of-structs in shared memory.
// Word 3i + c sits in bank (3i + c) mod 32; 3 is invertible mod 32 (and mod
// 16 for 64-bit words), so lanes with distinct i mod 32 are conflict-free,
// exactly as with separate component arrays, and the three components share
// one address (immediate offsets 0/4/8) -- a third of the address arithmetic.

template <typename Real>
struct Smem {
    Real *pos;      // positions (storage order), AoS: one address per vertex, components at +0/+1/+2
    Real *alt;      // edge_gather: the other position buffer (ping-pong); == pos otherwise
    Real *slot;     // slot buffer, AoS like the positions
    __device__ __forceinline__ Real &X(int i) const { return pos[3 * i]; }
    __device__ __forceinline__ Real &Y(int i) const { return pos[3 * i + 1]; }
    __device__ __forceinline__ Real &Z(int i) const { return pos[3 * i + 2]; }
    __device__ __forceinline__ Real &SX(int i) const { return slot[3 * i]; }
    __device__ __forceinline__ Real &SY(int i) const { return slot[3 * i + 1]; }
    __device__ __forceinline__ Real &SZ(int i) const { return slot[3 * i + 2]; }
    int *deg;           // degenerate-constraint counters: int per vertex, or bytes when narrow
    int narrow;
    unsigned *cbits;
    Scal *sc;
    Cap<Real> *caps;
};

// programmatic dependent launch (sm_90+): no-ops when the kernel was launched normally
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// narrow programs' positions (and byte-offset slot fields) start at this constant address
__device__ __forceinline__ char *smem_base() {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    return reinterpret_cast<char *>(smem_raw + TS_SMEM_HEAD);
}
// fast programs' dictionary tables at a fixed shared-memory offset (no base pointer to keep live)
__device__ __forceinline__ const float *smem_tab(int byte_off) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    return reinterpret_cast<const float *>(smem_raw + byte_off);
}
// 32-bit .shared address of byte `byte_off` of the dynamic shared memory.
__device__ __forceinline__ uint32_t smem_u32(int byte_off) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    return (uint32_t)__cvta_generic_to_shared(smem_raw + byte_off);
}
// The fast kernel addresses shared memory with ld/st.shared at CONSTANT addresses: offset
// register + immediate (TS_SMEM_WINDOW + the byte offset in the dynamic block).  A generic pointer,
// or a base kept in a register, costs the CTA's shared-window computation (S2UR SR_CgaCtaId, ULEA)
// or an add in every loop iteration.  TS_SMEM_WINDOW is the .shared address of the first dynamic
// byte of a non-cluster launch; the library probes it once (ts_smem_window_probe) and selects the
// fast kernel only when it matches, and the kernel traps if launched otherwise.
#define TS_SB (TS_SMEM_WINDOW + TS_SMEM_HEAD)   // .shared address of smem_base()
__device__ __forceinline__ float lds1c(uint32_t off) {          // [off + TS_SMEM_WINDOW]
    float v;
    asm volatile("ld.shared.f32 %0, [%1+%2];" : "=f"(v) : "r"(off), "n"(TS_SMEM_WINDOW));
    return v;
}
__device__ __forceinline__ float2 lds2c(uint32_t off) {
    float2 v;
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2+%3];" : "=f"(v.x), "=f"(v.y) : "r"(off), "n"(TS_SMEM_WINDOW));
    return v;
}
// one AoS vertex / slot at byte `off` from smem_base()
__device__ __forceinline__ void lds3c(uint32_t off, float &x, float &y, float &z) {
    asm volatile("ld.shared.f32 %0, [%3+%4];\n\tld.shared.f32 %1, [%3+%5];\n\tld.shared.f32 %2, [%3+%6];"
                 : "=f"(x), "=f"(y), "=f"(z) : "r"(off), "n"(TS_SB), "n"(TS_SB + 4), "n"(TS_SB + 8));
}

__device__ __forceinline__ void deg_add(int narrow, int *deg, int i) {
    if (narrow) atomicAdd(reinterpret_cast<unsigned *>(deg) + (i >> 2), 1u << ((i & 3) * 8));
    else atomicAdd(&deg[i], 1);
}
__device__ __forceinline__ int deg_take(int narrow, int *deg, int i) {   // read and clear (phase 2)
    if (narrow) {
        unsigned char *b = reinterpret_cast<unsigned char *>(deg);
        const int d = b[i];
        if (d) b[i] = 0;
        return d;
    }
    const int d = deg[i];
    if (d) deg[i] = 0;
    return d;
}

template <typename Real>
__device__ __forceinline__ Smem<Real> carve(const TsDevProg &P, unsigned char *raw) {
    // [scalar block | capsules | slots | positions | ping-pong positions | degenerate counters |
    //  contact bitmap]: the slot buffer sits at a constant offset (no per-use address
    //  arithmetic in phase 1), and everything a cluster peer addresses over DSMEM (scalars,
    //  slots / contact records, positions, the contact key list in the counters) sits at the same
    //  offset in every CTA of the cluster (parts share Vstore and the slot capacity)
    static_assert(((sizeof(Scal) + 15) / 16) * 16 + 3 * sizeof(Cap<Real>) <= TS_TAB_OFF, "scalar block");
    Smem<Real> m;
    m.sc = reinterpret_cast<Scal *>(raw);
    m.caps = reinterpret_cast<Cap<Real> *>(raw + ((sizeof(Scal) + 15) / 16) * 16);
    Real *base = reinterpret_cast<Real *>(raw + TS_SMEM_HEAD);
    m.narrow = P.narrow;
    if (P.narrow) {   // [positions | slots | counters]
        m.pos = m.alt = base;
        m.slot = base + 3 * P.Vstore;
        m.deg = reinterpret_cast<int *>(m.slot + 3 * P.slot_cap);
    } else {          // [slots | positions | ping-pong | counters]
        const bool pp = P.edge_gather;
        m.slot = base;
        m.pos = base + 3 * P.slot_cap;
        m.alt = pp ? m.pos + 3 * P.Vstore : m.pos;
        m.deg = reinterpret_cast<int *>(m.pos + 3 * P.Vstore * (pp ? 2 : 1));
    }
    m.cbits = reinterpret_cast<unsigned *>(reinterpret_cast<unsigned char *>(m.deg) + (P.narrow ? 1 : 4) * P.Vf_pad);
    return m;
}

// ---------------------------------------------------------------------------
// phase 1: constraint-parallel correction vectors into slots
// ---------------------------------------------------------------------------
// One distance constraint: correction vectors for both endpoints into their slots.
// fp64: (wa, wb, wsum) are the reference's operands; fp32: (wa, wb) carry the
// folded coefficients ks wa / wsum, ks wb / wsum and wsum is unused.
template <typename Real>
__device__ __forceinline__ void edge_item(const Smem<Real> &m, int pa, int pb, int sa, int sb, Real rl, Real wa,
                                          Real wb, Real wsum, Real ks, int vfp) {
    const Real dx = m.X(pa) - m.X(pb);
    const Real dy = m.Y(pa) - m.Y(pb);
    const Real dz = m.Z(pa) - m.Z(pb);
    Real ca, cb;
    bool degenerate;
    if constexpr (sizeof(Real) == 8) {
        // exact build: ts_lane_edges, _kernels.pyx:121-136
        const Real dist = sqrt(dx * dx + dy * dy + dz * dz);
        const Real mm = (Real)0.5 + copysign((Real)0.5, dist - (Real)1e-12);
        const Real scale = mm * ks * (dist - rl) / (dist * wsum + ((Real)1 - mm));
        ca = -wa * scale;
        cb = wb * scale;
        degenerate = mm == (Real)0;
    } else {
        // fp32 build: c = k (1 - rest / dist)
        const float d2 = __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, dx * dx));
        degenerate = !(d2 >= 1e-24f);                    // dist < 1e-12 (coincident guard)
        const float f = degenerate ? 0.0f : __fmaf_rn(-rl, rsqrt_ftz(d2), 1.0f);
        ca = -wa * f;
        cb = wb * f;
    }
    if (sa >= 0) { m.SX(sa) = ca * dx; m.SY(sa) = ca * dy; m.SZ(sa) = ca * dz; }   // -1: pinned endpoint
    if (sb >= 0) { m.SX(sb) = cb * dx; m.SY(sb) = cb * dy; m.SZ(sb) = cb * dz; }
    if (degenerate) {
        if (pa < vfp) deg_add(m.narrow, m.deg, pa);
        if (pb < vfp) deg_add(m.narrow, m.deg, pb);
    }
}

template <typename Real>
__device__ __forceinline__ void p1_edges(const TsDevProg &P, const Smem<Real> &m, int begin, int count,
                                         Real ks) {
    const int vfp = P.Vf_pad;
    const int stride = blockDim.x;
    const int t = threadIdx.x;
    if (P.compact) {
        // 16-bit stream: {pa|pb, sa|sb, rest}; weights from the pinned flags (uniform free mass)
        const uint4 *it = P.edge_c + begin;
        const Real w = (Real)P.w_free;
        uint4 nq = make_uint4(0, 0, 0, 0);
        if (t < count) nq = __ldg(it + t);
        for (int i = t; i < count; i += stride) {
            const uint4 q = nq;
            nq = __ldg(it + min(i + stride, count - 1));   // prefetch, branch-free
            const int pa = q.x & 0xffff, pb = q.x >> 16;
            const int sa = (q.y & 0xffff) == 0xffff ? -1 : (int)(q.y & 0xffff);   // 0xffff: no slot
            const int sb = (q.y >> 16) == 0xffff ? -1 : (int)(q.y >> 16);
            Real rl, wa, wb, wsum;
            if constexpr (sizeof(Real) == 8) {
                rl = __hiloint2double((int)q.w, (int)q.z);
                wa = pa < vfp ? w : (Real)0;
                wb = pb < vfp ? w : (Real)0;
                wsum = wa + wb;
            } else {
                rl = __uint_as_float(q.z);
                const bool both = (pa < vfp) && (pb < vfp);
                wa = wb = both ? (Real)0.5 * ks : ks;       // ks w / (w + w) or ks w / w
                wsum = 0;
            }
            edge_item<Real>(m, pa, pb, sa, sb, rl, wa, wb, wsum, ks, vfp);
        }
        return;
    }
    using V4 = typename R4<Real>::T;
    const int4 *idx = P.edge_idx + begin;
    const V4 *par = reinterpret_cast<const V4 *>(P.edge_par) + begin;
    // topology of the next item is fetched one iteration ahead (hides the L2 latency)
    int4 nid = make_int4(0, 0, 0, 0);
    V4 npr{};
    if (t < count) { nid = __ldg(idx + t); npr = par[t]; }
    for (int i = t; i < count; i += stride) {
        const int4 id = nid;     // {pos a, pos b, slot a, slot b}
        const V4 pr = npr;       // fp64 {rest, wa, wb, wa + wb}; fp32 {rest, ks wa/wsum, ks wb/wsum, 0}
        {   // unconditional (clamped) prefetch: no branch in the loop body
            const int j = min(i + stride, count - 1);
            nid = __ldg(idx + j); npr = par[j];
        }
        edge_item<Real>(m, id.x, id.y, id.z, id.w, pr.x, pr.y, pr.z, pr.w, ks, vfp);
    }
}

template <typename Real>
__device__ __forceinline__ void put_slot(const Smem<Real> &m, int s, Real c, Real gx, Real gy, Real gz) {
    if (s >= 0) { m.SX(s) = c * gx; m.SY(s) = c * gy; m.SZ(s) = c * gz; }
}

template <typename Real>
__device__ __forceinline__ void store_slot(const Smem<Real> &m, int s, Real c, Real gx, Real gy, Real gz) {
    m.SX(s) = c * gx; m.SY(s) = c * gy; m.SZ(s) = c * gz;
}

template <typename Real>
__device__ __forceinline__ void tet_item(const Smem<Real> &m, int4 id, int4 sl, Real rvi, Real kv, int vfp);

// fp32 builds: sum |G|^2 of a tet's four (unscaled) gradients as three independent 4-term FMA chains
// -- a shorter dependency chain than one 12-term sum; every fp32 tet path uses this one order
__device__ __forceinline__ float tet_den(float Gax, float Gay, float Gaz, float Gbx, float Gby, float Gbz, float Gcx,
                                         float Gcy, float Gcz, float Gdx, float Gdy, float Gdz) {
    float d0 = Gax * Gax, d1 = Gbx * Gbx, d2 = Gcx * Gcx;
    d0 = __fmaf_rn(Gay, Gay, d0); d1 = __fmaf_rn(Gby, Gby, d1); d2 = __fmaf_rn(Gcy, Gcy, d2);
    d0 = __fmaf_rn(Gaz, Gaz, d0); d1 = __fmaf_rn(Gbz, Gbz, d1); d2 = __fmaf_rn(Gcz, Gcz, d2);
    d0 = __fmaf_rn(Gdx, Gdx, d0); d1 = __fmaf_rn(Gdy, Gdy, d1); d2 = __fmaf_rn(Gdz, Gdz, d2);
    return (d0 + d1) + d2;
}

// fp32 tet item on byte-offset streams (boff programs): q = {a | b << 16, c | d << 16, slot a | b << 16,
// slot c | d << 16}, all byte offsets into the position / slot buffers (no index multiplies)
__device__ __forceinline__ void tet_item_b(const char *pb, char *sb, int *deg, int narrow, uint4 q, float rvi, float kv,
                                           unsigned vfp_b, unsigned pmask) {
    // pmask = 0x3fff when the top two bits of each position field carry the 6 V0 dictionary index
    const unsigned oa = q.x & pmask, ob = (q.x >> 16) & pmask, oc = q.y & pmask, od = (q.y >> 16) & pmask;
    auto ld = [&](unsigned o) { return *reinterpret_cast<const float *>(pb + o); };
    const float ax = ld(oa), ay = ld(oa + 4), az = ld(oa + 8);
    const float bax = ld(ob) - ax, bay = ld(ob + 4) - ay, baz = ld(ob + 8) - az;
    const float cax = ld(oc) - ax, cay = ld(oc + 4) - ay, caz = ld(oc + 8) - az;
    const float dax = ld(od) - ax, day = ld(od + 4) - ay, daz = ld(od + 8) - az;
    // unscaled cross products G = 6 grad (rv holds 6 V0), as tet_item's fp32 branch
    const float Gbx = __fmaf_rn(cay, daz, -caz * day);
    const float Gby = __fmaf_rn(caz, dax, -cax * daz);
    const float Gbz = __fmaf_rn(cax, day, -cay * dax);
    const float Gcx = __fmaf_rn(day, baz, -daz * bay);
    const float Gcy = __fmaf_rn(daz, bax, -dax * baz);
    const float Gcz = __fmaf_rn(dax, bay, -day * bax);
    const float Gdx = __fmaf_rn(bay, caz, -baz * cay);
    const float Gdy = __fmaf_rn(baz, cax, -bax * caz);
    const float Gdz = __fmaf_rn(bax, cay, -bay * cax);
    const float Gax = -(Gbx + Gcx + Gdx);
    const float Gay = -(Gby + Gcy + Gdy);
    const float Gaz = -(Gbz + Gcz + Gdz);
    const float c6 = __fmaf_rn(Gdz, daz, __fmaf_rn(Gdy, day, Gdx * dax)) - rvi;
    const float den = tet_den(Gax, Gay, Gaz, Gbx, Gby, Gbz, Gcx, Gcy, Gcz, Gdx, Gdy, Gdz);
    const bool degenerate = !(den > 3.6e-17f);                  // sum|grad|^2 <= 1e-18
    const float sc = degenerate ? 0.0f : (-kv * c6) * rcp_ftz(den);
    // 0xffff: a pinned corner has no slot -- a predicated store (no branch, no shared "trash" slot,
    // so every shared word has one writer per phase)
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(sb);
    // the four corners' stores in one block, interleaved (as tet_item_fast: stays predicated)
    const unsigned sa = q.z & 0xffffu, sb_ = q.z >> 16, sc_ = q.w & 0xffffu, sd = q.w >> 16;
    asm volatile("{\n\t.reg .pred pa, pb, pc, pd;\n\t"
                 "setp.ne.u32 pa, %0, 65535;\n\tsetp.ne.u32 pb, %1, 65535;\n\t"
                 "setp.ne.u32 pc, %2, 65535;\n\tsetp.ne.u32 pd, %3, 65535;\n\t"
                 "@pa st.shared.f32 [%4], %8;\n\t@pb st.shared.f32 [%5], %11;\n\t"
                 "@pc st.shared.f32 [%6], %14;\n\t@pd st.shared.f32 [%7], %17;\n\t"
                 "@pa st.shared.f32 [%4+4], %9;\n\t@pb st.shared.f32 [%5+4], %12;\n\t"
                 "@pc st.shared.f32 [%6+4], %15;\n\t@pd st.shared.f32 [%7+4], %18;\n\t"
                 "@pa st.shared.f32 [%4+8], %10;\n\t@pb st.shared.f32 [%5+8], %13;\n\t"
                 "@pc st.shared.f32 [%6+8], %16;\n\t@pd st.shared.f32 [%7+8], %19;\n\t}"
                 ::"r"(sa), "r"(sb_), "r"(sc_), "r"(sd), "r"(sbase + sa), "r"(sbase + sb_), "r"(sbase + sc_),
                 "r"(sbase + sd), "f"(sc * Gax), "f"(sc * Gay), "f"(sc * Gaz), "f"(sc * Gbx), "f"(sc * Gby),
                 "f"(sc * Gbz), "f"(sc * Gcx), "f"(sc * Gcy), "f"(sc * Gcz), "f"(sc * Gdx), "f"(sc * Gdy),
                 "f"(sc * Gdz)
                 : "memory");
    if (degenerate) {
        if (oa < vfp_b) deg_add(narrow, deg, oa / 12);
        if (ob < vfp_b) deg_add(narrow, deg, ob / 12);
        if (oc < vfp_b) deg_add(narrow, deg, oc / 12);
        if (od < vfp_b) deg_add(narrow, deg, od / 12);
    }
}

// The fast kernel's tet item: byte offsets from the 32-bit shared base sb (positions and slots share
// it: narrow layout), rest volume 6 V0 given; same arithmetic as tet_item_b.
// RV4: only bits 14-15 of the first field carry the 6 V0 index, so the other three position
// fields need at most one operation each
template <bool RV4>
__device__ __forceinline__ void tet_item_fast(int *deg, uint4 q, float rvi, float kv, unsigned vfp_b) {
    const unsigned oa = q.x & 0x3fffu;
    const unsigned ob = RV4 ? q.x >> 16 : (q.x >> 16) & 0x3fffu;
    const unsigned oc = RV4 ? q.y & 0xffffu : q.y & 0x3fffu;
    const unsigned od = RV4 ? q.y >> 16 : (q.y >> 16) & 0x3fffu;
    float ax, ay, az, bx, by, bz, cx, cy, cz, dx, dy, dz;
    lds3c(oa, ax, ay, az);
    lds3c(ob, bx, by, bz);
    lds3c(oc, cx, cy, cz);
    lds3c(od, dx, dy, dz);
    const float bax = bx - ax, bay = by - ay, baz = bz - az;
    const float cax = cx - ax, cay = cy - ay, caz = cz - az;
    const float dax = dx - ax, day = dy - ay, daz = dz - az;
    const float Gbx = __fmaf_rn(cay, daz, -caz * day);
    const float Gby = __fmaf_rn(caz, dax, -cax * daz);
    const float Gbz = __fmaf_rn(cax, day, -cay * dax);
    const float Gcx = __fmaf_rn(day, baz, -daz * bay);
    const float Gcy = __fmaf_rn(daz, bax, -dax * baz);
    const float Gcz = __fmaf_rn(dax, bay, -day * bax);
    const float Gdx = __fmaf_rn(bay, caz, -baz * cay);
    const float Gdy = __fmaf_rn(baz, cax, -bax * caz);
    const float Gdz = __fmaf_rn(bax, cay, -bay * cax);
    const float Gax = -(Gbx + Gcx + Gdx);
    const float Gay = -(Gby + Gcy + Gdy);
    const float Gaz = -(Gbz + Gcz + Gdz);
    const float c6 = __fmaf_rn(Gdz, daz, __fmaf_rn(Gdy, day, Gdx * dax)) - rvi;
    const float den = tet_den(Gax, Gay, Gaz, Gbx, Gby, Gbz, Gcx, Gcy, Gcz, Gdx, Gdy, Gdz);
    const bool degenerate = !(den > 3.6e-17f);                  // sum|grad|^2 <= 1e-18
    const float sc = degenerate ? 0.0f : (-kv * c6) * rcp_ftz(den);
    // 0xffff: pinned corner, its stores predicated off.  One asm block with the four corners'
    // stores interleaved: ptxas keeps them predicated (per-corner blocks were turned into
    // BSSY / BRA / BSYNC regions, 3 extra instructions per corner)
    asm volatile("{\n\t.reg .pred pa, pb, pc, pd;\n\t"
                 "setp.ne.u32 pa, %0, 65535;\n\tsetp.ne.u32 pb, %1, 65535;\n\t"
                 "setp.ne.u32 pc, %2, 65535;\n\tsetp.ne.u32 pd, %3, 65535;\n\t"
                 "@pa st.shared.f32 [%0+%16], %4;\n\t@pb st.shared.f32 [%1+%16], %7;\n\t"
                 "@pc st.shared.f32 [%2+%16], %10;\n\t@pd st.shared.f32 [%3+%16], %13;\n\t"
                 "@pa st.shared.f32 [%0+%17], %5;\n\t@pb st.shared.f32 [%1+%17], %8;\n\t"
                 "@pc st.shared.f32 [%2+%17], %11;\n\t@pd st.shared.f32 [%3+%17], %14;\n\t"
                 "@pa st.shared.f32 [%0+%18], %6;\n\t@pb st.shared.f32 [%1+%18], %9;\n\t"
                 "@pc st.shared.f32 [%2+%18], %12;\n\t@pd st.shared.f32 [%3+%18], %15;\n\t}"
                 ::"r"(q.z & 0xffffu), "r"(q.z >> 16), "r"(q.w & 0xffffu), "r"(q.w >> 16),
                 "f"(sc * Gax), "f"(sc * Gay), "f"(sc * Gaz), "f"(sc * Gbx), "f"(sc * Gby), "f"(sc * Gbz),
                 "f"(sc * Gcx), "f"(sc * Gcy), "f"(sc * Gcz), "f"(sc * Gdx), "f"(sc * Gdy), "f"(sc * Gdz),
                 "n"(TS_SB), "n"(TS_SB + 4), "n"(TS_SB + 8)
                 : "memory");
    if (degenerate) {
        if (oa < vfp_b) deg_add(1, deg, oa / 12);
        if (ob < vfp_b) deg_add(1, deg, ob / 12);
        if (oc < vfp_b) deg_add(1, deg, oc / 12);
        if (od < vfp_b) deg_add(1, deg, od / 12);
    }
}

// The fast kernel's share of one warp's tet items [wb, wb + 32 j) (the stream is padded by a CTA's
// worth of items: the prefetch needs no clamp).  RV4: at most 4 distinct 6 V0 values, whose
// dictionary index sits in bits 14-15 of the first position field alone.
template <bool RV4>
__device__ __forceinline__ void p1_tets_fast(const TsDevProg &P, int *deg, int begin, int wb, int we, float kv) {
    const int lane = threadIdx.x & 31;
    const unsigned vfp_b = 12u * (unsigned)P.Vf_pad;
    const uint4 *ip = P.tet_c + begin + wb + lane;
    uint4 nq = __ldg(ip);
#pragma unroll kTetUnroll
    for (int i = wb + lane; i < we; i += 32) {
        const uint4 q = nq;
        ip += 32;
        nq = __ldg(ip);
        const unsigned ri = RV4 ? ((q.x >> 14) & 3u)
                                : (((q.x >> 14) & 3u) | ((q.x >> 28) & 12u) | ((q.y >> 10) & 48u) | ((q.y >> 24) & 192u));
        tet_item_fast<RV4>(deg, q, lds1c(TS_TAB_OFF + 4 * TS_TAB_CAP + 4 * ri), kv, vfp_b);
    }
}

template <typename Real, bool FAST = false>
__device__ __forceinline__ void p1_tets(const TsDevProg &P, const Smem<Real> &m, int begin, int wb, int we, Real kv) {
    // this warp's contiguous range [wb, we) of the chunk's items, lane l takes wb + l, wb + l + 32, ...
    const Real *rv = reinterpret_cast<const Real *>(P.tet_rv) + begin;
    const int vfp = P.Vf_pad;
    const int lane = threadIdx.x & 31;
    if constexpr (sizeof(Real) == 4) {
        if (FAST || P.boff) {   // byte-offset stream, padded by a CTA's worth of items: unclamped prefetch
            const uint4 *it = P.tet_c + begin;
            // narrow: slot fields are offsets from the position base too (FAST: a constant address)
            const char *pb = FAST ? smem_base() : reinterpret_cast<const char *>(m.pos);
            char *sb = FAST ? smem_base() : reinterpret_cast<char *>(P.narrow ? m.pos : m.slot);
            uint4 nq = __ldg(it + wb + lane);
            if (FAST || P.rvdict) {   // rest volume from the stream's spare bits + a tiny (L1-resident) table
                for (int i = wb + lane; i < we; i += 32) {
                    const uint4 q = nq;
                    nq = __ldg(it + i + 32);
                    const unsigned ri = ((q.x >> 14) & 3u) | ((q.x >> 28) & 12u) | ((q.y >> 10) & 48u) |
                                        ((q.y >> 24) & 192u);
                    // all four slots absent: an idle lane of the bank schedule (or four pinned corners);
                    // the fast kernel runs it anyway: its stores are predicated off and its corners
                    // are not free vertices (the compiler points idle lanes past Vf_pad)
                    if (FAST || (q.z & q.w) != 0xffffffffu)
                        tet_item_b(pb, sb, m.deg, m.narrow, q,
                                   FAST ? smem_tab(TS_TAB_OFF + 4 * TS_TAB_CAP)[ri] : __ldg(P.rvtab + ri), kv,
                                   12u * (unsigned)vfp, 0x3fffu);
                }
                return;
            }
            float nrv = __ldg(rv + wb + lane);
            for (int i = wb + lane; i < we; i += 32) {
                const uint4 q = nq;
                const float rvi = nrv;
                nq = __ldg(it + i + 32);
                nrv = __ldg(rv + i + 32);
                if ((q.z & q.w) != 0xffffffffu)   // idle lane of the bank schedule
                    tet_item_b(pb, sb, m.deg, m.narrow, q, rvi, kv, 12u * (unsigned)vfp, 0xffffu);
            }
            return;
        }
    }
    if (wb >= we) return;
    if (P.compact) {
        const uint4 *it = P.tet_c + begin;
        uint4 nq = make_uint4(0, 0, 0, 0);
        Real nrv = 0;
        if (wb + lane < we) { nq = __ldg(it + wb + lane); nrv = rv[wb + lane]; }
        for (int i = wb + lane; i < we; i += 32) {
            const uint4 q = nq;
            const Real rvi = nrv;
            { const int j = min(i + 32, we - 1); nq = __ldg(it + j); nrv = rv[j]; }
            const int4 id = make_int4(q.x & 0xffff, q.x >> 16, q.y & 0xffff, q.y >> 16);
            auto s16 = [](unsigned v) { return v == 0xffffu ? -1 : (int)v; };   // 0xffff: no slot
            const int4 sl = make_int4(s16(q.z & 0xffff), s16(q.z >> 16), s16(q.w & 0xffff), s16(q.w >> 16));
            if ((q.z & q.w) != 0xffffffffu) tet_item<Real>(m, id, sl, rvi, kv, vfp);
        }
        return;
    }
    const int4 *idx = P.tet_idx + begin;
    const int4 *slot = P.tet_slot + begin;
    int4 nid = make_int4(0, 0, 0, 0), nsl = make_int4(0, 0, 0, 0);
    Real nrv = 0;
    if (wb + lane < we) { nid = __ldg(idx + wb + lane); nsl = __ldg(slot + wb + lane); nrv = rv[wb + lane]; }
    for (int i = wb + lane; i < we; i += 32) {
        const int4 id = nid;
        const int4 sl = nsl;
        const Real rvi = nrv;
        {
            const int j = min(i + 32, we - 1);
            nid = __ldg(idx + j); nsl = __ldg(slot + j); nrv = rv[j];
        }
        if ((sl.x & sl.y & sl.z & sl.w) != -1) tet_item<Real>(m, id, sl, rvi, kv, vfp);   // all -1: idle lane
    }
}

// One volume constraint: correction vectors for its four vertices into their slots.
template <typename Real>
__device__ __forceinline__ void tet_item(const Smem<Real> &m, int4 id, int4 sl, Real rvi, Real kv, int vfp) {
    {
        const Real ax = m.X(id.x), ay = m.Y(id.x), az = m.Z(id.x);
        const Real bax = m.X(id.y) - ax, bay = m.Y(id.y) - ay, baz = m.Z(id.y) - az;
        const Real cax = m.X(id.z) - ax, cay = m.Y(id.z) - ay, caz = m.Z(id.z) - az;
        const Real dax = m.X(id.w) - ax, day = m.Y(id.w) - ay, daz = m.Z(id.w) - az;
        bool degenerate;
        if constexpr (sizeof(Real) == 8) {
            // exact build: ts_lane_tets, _kernels.pyx:165-208
            const Real gbx = (cay * daz - caz * day) / 6.0;
            const Real gby = (caz * dax - cax * daz) / 6.0;
            const Real gbz = (cax * day - cay * dax) / 6.0;
            const Real gcx = (day * baz - daz * bay) / 6.0;
            const Real gcy = (daz * bax - dax * baz) / 6.0;
            const Real gcz = (dax * bay - day * bax) / 6.0;
            const Real gdx = (bay * caz - baz * cay) / 6.0;
            const Real gdy = (baz * cax - bax * caz) / 6.0;
            const Real gdz = (bax * cay - bay * cax) / 6.0;
            const Real gax = -(gbx + gcx + gdx);
            const Real gay = -(gby + gcy + gdy);
            const Real gaz = -(gbz + gcz + gdz);
            const Real cval = (gdx * dax + gdy * day + gdz * daz) - rvi;
            const Real denom = gax * gax + gay * gay + gaz * gaz
                             + gbx * gbx + gby * gby + gbz * gbz
                             + gcx * gcx + gcy * gcy + gcz * gcz
                             + gdx * gdx + gdy * gdy + gdz * gdz;
            const Real mm = (Real)0.5 + copysign((Real)0.5, denom - (Real)1e-18);
            const Real sc = -mm * kv * cval / (denom + ((Real)1 - mm));
            put_slot(m, sl.x, sc, gax, gay, gaz);   // -1: pinned corner, no slot
            put_slot(m, sl.y, sc, gbx, gby, gbz);
            put_slot(m, sl.z, sc, gcx, gcy, gcz);
            put_slot(m, sl.w, sc, gdx, gdy, gdz);
            degenerate = mm == (Real)0;
        } else {
            // fp32 build on unscaled cross products G = 6 grad (rv holds 6 V0):
            //   s grad_i = -kv (G_d . da - 6 V0) / sum|G|^2  G_i
            const float Gbx = __fmaf_rn(cay, daz, -caz * day);
            const float Gby = __fmaf_rn(caz, dax, -cax * daz);
            const float Gbz = __fmaf_rn(cax, day, -cay * dax);
            const float Gcx = __fmaf_rn(day, baz, -daz * bay);
            const float Gcy = __fmaf_rn(daz, bax, -dax * baz);
            const float Gcz = __fmaf_rn(dax, bay, -day * bax);
            const float Gdx = __fmaf_rn(bay, caz, -baz * cay);
            const float Gdy = __fmaf_rn(baz, cax, -bax * caz);
            const float Gdz = __fmaf_rn(bax, cay, -bay * cax);
            const float Gax = -(Gbx + Gcx + Gdx);
            const float Gay = -(Gby + Gcy + Gdy);
            const float Gaz = -(Gbz + Gcz + Gdz);
            const float c6 = __fmaf_rn(Gdz, daz, __fmaf_rn(Gdy, day, Gdx * dax)) - rvi;
            const float den = tet_den(Gax, Gay, Gaz, Gbx, Gby, Gbz, Gcx, Gcy, Gcz, Gdx, Gdy, Gdz);
            degenerate = !(den > 3.6e-17f);                  // sum|grad|^2 <= 1e-18
            const float sc = degenerate ? 0.0f : (-kv * c6) * rcp_ftz(den);
            put_slot(m, sl.x, sc, Gax, Gay, Gaz);
            put_slot(m, sl.y, sc, Gbx, Gby, Gbz);
            put_slot(m, sl.z, sc, Gcx, Gcy, Gcz);
            put_slot(m, sl.w, sc, Gdx, Gdy, Gdz);
        }
        if (degenerate) {
            if (id.x < vfp) deg_add(m.narrow, m.deg, id.x);
            if (id.y < vfp) deg_add(m.narrow, m.deg, id.y);
            if (id.z < vfp) deg_add(m.narrow, m.deg, id.z);
            if (id.w < vfp) deg_add(m.narrow, m.deg, id.w);
        }
    }
}

template <typename Real>
__device__ void p1_atts(const TsDevProg &P, const Smem<Real> &m, int begin, int count) {
    using V4 = typename R4<Real>::T;
    const int4 *idx = P.att_idx + begin;
    const int4 *slot = P.att_slot + begin;
    const V4 *par = reinterpret_cast<const V4 *>(P.att_par) + begin;
    const V4 *anc = reinterpret_cast<const V4 *>(P.att_anchor) + begin;
    for (int i = threadIdx.x; i < count; i += blockDim.x) {
        const int4 id = idx[i];
        const int4 sl = slot[i];
        const V4 pr = par[i];   // rest, k, wv, wc
        const V4 an = anc[i];   // ax, ay, az, is_face
        const bool face = an.w != (Real)0;
        Real cx, cy, cz;
        if (face) {
            cx = (m.X(id.y) + m.X(id.z) + m.X(id.w)) / (Real)3;
            cy = (m.Y(id.y) + m.Y(id.z) + m.Y(id.w)) / (Real)3;
            cz = (m.Z(id.y) + m.Z(id.z) + m.Z(id.w)) / (Real)3;
        } else { cx = an.x; cy = an.y; cz = an.z; }
        const Real wsum = pr.z + pr.w;
        const Real dx = m.X(id.x) - cx, dy = m.Y(id.x) - cy, dz = m.Z(id.x) - cz;
        const Real dist = sqrt(dx * dx + dy * dy + dz * dz);
        const Real mm = dist > (Real)1e-12 ? (Real)1 : (Real)0;
        const Real scale = mm * pr.y * (dist - pr.x) / (dist * wsum + ((Real)1 - mm));
        const Real ca = -pr.z * scale;
        put_slot(m, sl.x, ca, dx, dy, dz);
        if (face) {
            const Real cb = pr.w * scale / (Real)3;
            put_slot(m, sl.y, cb, dx, dy, dz);
            put_slot(m, sl.z, cb, dx, dy, dz);
            put_slot(m, sl.w, cb, dx, dy, dz);
        }
        if (mm == (Real)0) {
            if (sl.x >= 0) deg_add(m.narrow, m.deg, id.x);
            if (face) {
                if (sl.y >= 0) deg_add(m.narrow, m.deg, id.y);
                if (sl.z >= 0) deg_add(m.narrow, m.deg, id.z);
                if (sl.w >= 0) deg_add(m.narrow, m.deg, id.w);
            }
        }
    }
}

// ---------------------------------------------------------------------------
// owner-gathered distance constraints (edge_gather programs)
// ---------------------------------------------------------------------------
// Free vertex p (owner lane `lane`, own predicted position (px, py, pz)) adds the
// corrections of its live incident edges, in edge-index order, to (ax, ay, az).
// fp64: -(w_p scale) (x_p - x_q) with the reference's scale expression
// (ts_lane_edges, _kernels.pyx:121-136) -- bitwise the reference's per-endpoint
// term, see compiler.cpp; fp32: -coef (1 - rest / dist) (x_p - x_q) with FMAs.
template <typename Real, bool FAST = false, bool HOIST = FAST, bool STAB = FAST, bool PIPE = FAST>
__device__ __forceinline__ void owner_edges(const TsDevProg &P, const Smem<Real> &m, int p, int lane, Real px,
                                            Real py, Real pz, Real ks, Real &ax, Real &ay, Real &az, int &ndeg,
                                            int ev_h = 0, int rb_h = 0) {
    const int ev = HOIST ? ev_h : P.evalence[p];            // HOIST: read once, before the substep loop
    const int rb = HOIST ? rb_h : P.eregion[p >> 5] + lane;
    if constexpr (sizeof(Real) == 8) {
        const int4 *rec = reinterpret_cast<const int4 *>(P.einc) + rb;
        const double *wst = reinterpret_cast<const double *>(P.w);
        const double wp = wst[p];
        for (int k = 0; k < ev; ++k) {
            const int4 q = __ldg(rec + 32 * k);
            const int nb = q.x & 0x7fffffff;
            const double rl = __hiloint2double(q.w, q.z);
            const double wq = __ldg(wst + nb);
            const double dx = px - m.X(nb), dy = py - m.Y(nb), dz = pz - m.Z(nb);
            const double dist = sqrt(dx * dx + dy * dy + dz * dz);
            const double mm = 0.5 + copysign(0.5, dist - 1e-12);
            const double scale = mm * ks * (dist - rl) / (dist * (wp + wq) + (1.0 - mm));
            const double c = -(wp * scale);
            ax = ax + c * dx; ay = ay + c * dy; az = az + c * dz;
            ndeg += mm == 0.0;
        }
    } else if (FAST || P.einc_bytes == 4) {
        // 4-byte records: {neighbour byte offset | pair byte offset << 16}, pair = {rest length, -k_s w_p /
        // (w_p + w_q)} (pair 0 = {0, 0}: a null record of the compiler's conflict-free rounds, whose
        // term is exactly zero)
        const unsigned *rec = reinterpret_cast<const unsigned *>(P.einc) + rb;
        // PIPE (the fast kernel): the loop runs without the degenerate-edge select / count (|d| <= 1e-12 never happens in
        // a live simulation); it tracks the smallest |d|^2 instead and, when an edge was degenerate,
        // this vertex's edges are summed again with the exact rule below -- same result either way
        // (a NaN |d|^2 leaves NaN sums on both paths).  The edges are summed from zero and added at
        // the end: the edges come first in every vertex's sum, so the accumulators are +0 here and
        // the result is bitwise the in-place sum (no saved copies live across the loop)
        float ex = 0.0f, ey = 0.0f, ez = 0.0f;
        float d2min = 3.0e38f;
        // neighbour position and {rest, coefficient} pair of a record (FAST: constant shared
        // addresses; STAB, the edges kernel: the pair table's shared copy; else through L1)
        auto fetch = [&](unsigned r, float &qx, float &qy, float &qz, float2 &rc) {
            if constexpr (FAST) {
                rc = lds2c(TS_TAB_OFF + (r >> 16));
                lds3c(r & 0xffffu, qx, qy, qz);
            } else {
                rc = STAB ? lds2c(TS_TAB_OFF + (r >> 16))
                          : __ldg(reinterpret_cast<const float2 *>(reinterpret_cast<const char *>(P.rltab) +
                                                                    (r >> 16)));
                const float *nq = reinterpret_cast<const float *>(reinterpret_cast<const char *>(m.pos) + (r & 0xffffu));
                qx = nq[0]; qy = nq[1]; qz = nq[2];
            }
        };
        if constexpr (PIPE) {
            // software-pipelined: record k + 2 and the shared operands of record k + 1 are in flight
            // while record k's term is computed (the shared loads no longer wait behind the previous
            // term's arithmetic).  Loads past a lane's last record read a neighbouring lane's record
            // row or a zero padding row -- in-bounds offsets, results unused.
            unsigned qn = __ldg(rec + 32);
            float nx, ny, nz;
            float2 nrc;
            fetch(__ldg(rec), nx, ny, nz, nrc);
#pragma unroll kEdgeUnroll
            for (int k = 0; k < ev; ++k) {
                const float qx = nx, qy = ny, qz = nz;
                const float2 rc = nrc;
                fetch(qn, nx, ny, nz, nrc);
                qn = __ldg(rec + 32 * (k + 2));
                const float dx = px - qx, dy = py - qy, dz = pz - qz;
                const float d2 = __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, dx * dx));
                const float c = rc.y * __fmaf_rn(-rc.x, rsqrt_ftz(d2), 1.0f);
                d2min = fminf(d2min, d2);
                ex = __fmaf_rn(c, dx, ex); ey = __fmaf_rn(c, dy, ey); ez = __fmaf_rn(c, dz, ez);
            }
        }
        // the exact rule: every edge of the other kernels (measured faster there than the pipelined
        // loop -- the edges kernel is latency-bound), and a FAST vertex with a degenerate edge
        auto exact = [&](float &sx, float &sy, float &sz) {
            unsigned q = __ldg(rec);
            for (int k = 0; k < ev; ++k) {
                const unsigned cur = q;
                q = __ldg(rec + 32 * (k + 1));
                float qx, qy, qz;
                float2 rc;
                fetch(cur, qx, qy, qz, rc);
                const float dx = px - qx, dy = py - qy, dz = pz - qz;
                const float d2 = __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, dx * dx));
                const bool degenerate = !(d2 >= 1e-24f);
                const float c = rc.y * (degenerate ? 0.0f : __fmaf_rn(-rc.x, rsqrt_ftz(d2), 1.0f));
                sx = __fmaf_rn(c, dx, sx); sy = __fmaf_rn(c, dy, sy); sz = __fmaf_rn(c, dz, sz);
                ndeg += degenerate;
            }
        };
        if constexpr (PIPE) {
            if (d2min < 1e-24f) {
                ex = ey = ez = 0.0f;
                exact(ex, ey, ez);
            }
            ax += ex; ay += ey; az += ez;
        } else {
            exact(ax, ay, az);
        }
    } else if (P.einc_bytes == 8 && P.boff) {
        // byte-offset records, padded by one row: the prefetch of record k + 1 needs no clamp
        const uint2 *rec = reinterpret_cast<const uint2 *>(P.einc) + rb;
        const char *pb = reinterpret_cast<const char *>(m.pos);
        const float hks = 0.5f * ks;
        uint2 q = __ldg(rec);
        for (int k = 0; k < ev; ++k) {
            const uint2 cur = q;
            q = __ldg(rec + 32 * (k + 1));
            const unsigned nb = cur.x & 0x7fffffffu;
            const float rl = __uint_as_float(cur.y);
            const float *nq = reinterpret_cast<const float *>(pb + nb);
            const float dx = px - nq[0], dy = py - nq[1], dz = pz - nq[2];
            const float d2 = __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, dx * dx));
            const bool degenerate = !(d2 >= 1e-24f);
            const float f = degenerate ? 0.0f : __fmaf_rn(-rl, rsqrt_ftz(d2), 1.0f);
            const float c = -((int)cur.x < 0 ? ks : hks) * f;
            ax = __fmaf_rn(c, dx, ax); ay = __fmaf_rn(c, dy, ay); az = __fmaf_rn(c, dz, az);
            ndeg += degenerate;
        }
    } else if (P.einc_bytes == 8) {
        // uniform free mass: coef = ks w / (w + w) = ks / 2, or ks when the neighbour is pinned
        // (record bit 31)
        const uint2 *rec = reinterpret_cast<const uint2 *>(P.einc) + rb;
        const float hks = 0.5f * ks;   // == TsParams::hks_f
        uint2 q = ev > 0 ? __ldg(rec) : make_uint2(0, 0);
        for (int k = 0; k < ev; ++k) {
            const uint2 cur = q;
            q = __ldg(rec + 32 * min(k + 1, ev - 1));    // next record, branch-free prefetch
            const int nb = (int)(cur.x & 0x7fffffffu);
            const float rl = __uint_as_float(cur.y);
            const float dx = px - m.X(nb), dy = py - m.Y(nb), dz = pz - m.Z(nb);
            const float d2 = __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, dx * dx));
            const bool degenerate = !(d2 >= 1e-24f);
            const float f = degenerate ? 0.0f : __fmaf_rn(-rl, rsqrt_ftz(d2), 1.0f);
            const float c = -((int)cur.x < 0 ? ks : hks) * f;
            ax = __fmaf_rn(c, dx, ax); ay = __fmaf_rn(c, dy, ay); az = __fmaf_rn(c, dz, az);
            ndeg += degenerate;
        }
    } else {
        const int4 *rec = reinterpret_cast<const int4 *>(P.einc) + rb;
        for (int k = 0; k < ev; ++k) {
            const int4 q = __ldg(rec + 32 * k);
            const int nb = q.x & 0x7fffffff;
            const float coef = __int_as_float(q.y), rl = __int_as_float(q.z);
            const float dx = px - m.X(nb), dy = py - m.Y(nb), dz = pz - m.Z(nb);
            const float d2 = __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, dx * dx));
            const bool degenerate = !(d2 >= 1e-24f);
            const float f = degenerate ? 0.0f : __fmaf_rn(-rl, rsqrt_ftz(d2), 1.0f);
            const float c = -coef * f;
            ax = __fmaf_rn(c, dx, ax); ay = __fmaf_rn(c, dy, ay); az = __fmaf_rn(c, dz, az);
            ndeg += degenerate;
        }
    }
}

// tool command + grasp release + capsule rows for one env (thread 0), tool.py:307-378
static __device__ __forceinline__ void env_command(const TsDevProg &P, const TsParams &S, const TsLaunch &L,
                                                   int64_t env, TsCmd &sc) {
    const int mode = L.mode;
    Pose p;
    const bool has_tool = L.axis != nullptr;
    if (has_tool) {
        for (int c = 0; c < 3; ++c) { p.ax[c] = L.axis[3 * env + c]; p.jw[c] = L.jaw[3 * env + c]; }
        p.reach = L.reach[env]; p.clamp = L.clamp[env];
    }
    bool clipped = false, rejected = false;
    if (mode & TS_M_CMD_ACTIONS) {
        double tgt[3];
        for (int c = 0; c < 3; ++c) {
            double a = L.actions_f32 ? (double)reinterpret_cast<const float *>(L.actions)[3 * env + c]
                                     : reinterpret_cast<const double *>(L.actions)[3 * env + c];
            a = a > 1.0 ? 1.0 : (a < -1.0 ? -1.0 : a);   // np.clip(actions, -1, 1)
            tgt[c] = (S.rcm[c] + p.reach * p.ax[c]) + a * S.action_scale;
        }
        apply_command(S, p, tgt, S.held_angle, clipped, rejected);
    } else if (mode & TS_M_CMD_TARGETS) {
        double tgt[3] = {L.targets[3 * env], L.targets[3 * env + 1], L.targets[3 * env + 2]};
        apply_command(S, p, tgt, L.angles ? L.angles[env] : p.clamp, clipped, rejected);
    } else if (mode & TS_M_CMD_OVERRIDE) {
        for (int c = 0; c < 3; ++c) { p.ax[c] = L.ovr_axis[3 * env + c]; p.jw[c] = L.ovr_jaw[3 * env + c]; }
        p.reach = L.ovr_reach[env]; p.clamp = L.ovr_clamp[env];
        clipped = L.ovr_clipped ? L.ovr_clipped[env] != 0 : false;
    }
    sc.clipped = clipped; sc.rejected = rejected;
    sc.pre_done = 0; sc.dist = 0.0;
    if (mode & TS_M_ENV) {
        // env.py:167-174: success and the step limit are known before the physics runs;
        // only the divergence flag is added by the step kernel
        double rel[3];
        for (int c = 0; c < 3; ++c) rel[c] = (S.rcm[c] + p.reach * p.ax[c]) - S.target[c];
        // np.einsum("nq,nq->n") association on the reference hosts: (r0^2 + r2^2) + r1^2
        const double l = sqrt((rel[0] * rel[0] + rel[2] * rel[2]) + rel[1] * rel[1]);
        sc.dist = l;
        sc.pre_done = (l < S.success_thr) || (L.steps[env] + 1 >= S.max_steps);
    }
    int64_t gv = -1;
    if (mode & TS_M_EXT_GRASP) {
        gv = L.ext_gv[env];
        for (int c = 0; c < 3; ++c) sc.drag[c] = L.ext_drag[3 * env + c];
    } else if (has_tool) {
        gv = L.grasp_vertex[env];
        for (int c = 0; c < 3; ++c) sc.drag[c] = S.rcm[c] + p.reach * p.ax[c];
    } else {
        for (int c = 0; c < 3; ++c) sc.drag[c] = 0.0;   // plugin detect_contacts: no tool, no drag
    }
    sc.need_search = 0;
    if (mode & TS_M_GRASP) {
        if (p.clamp >= 3.0) {            // GRASP_ENGAGE_DEG, tool.py:23, 374-378
            if (gv >= 0) { L.grasped[env * P.V + gv] = 0; gv = -1; }
        } else if (gv < 0) {
            sc.need_search = 1;
        }
    }
    sc.gv = (int)gv;
    sc.pose = p;
    if (mode & TS_M_DETECT_ONLY) {
        for (int r = 0; r < 3; ++r) for (int k = 0; k < 7; ++k) sc.caps[r][k] = L.ext_caps[(env * 3 + r) * 7 + k];
    } else if (mode & TS_M_CONTACTS) {
        capsule_rows(S, p, sc.caps);
    }
    sc.any_bad = 0; sc.n_contacts = 0;
}

// reward / done / auto-reset / obs for one env (thread 0, fp64), env.py:160-197
static __device__ __forceinline__ void env_epilogue(const TsParams &S, const TsLaunch &L, int64_t env,
                                                    const TsCmd &sc) {
    const int mode = L.mode;
    const int any_bad = sc.any_bad;
    Pose p = sc.pose;
    const int64_t gv_new = sc.gv;
    int done = 0;
    if (mode & TS_M_ENV) {
        double drag[3];
        for (int c = 0; c < 3; ++c) drag[c] = S.rcm[c] + p.reach * p.ax[c];
        const double l = sc.dist;
        const bool success = l < S.success_thr;
        const double lp = L.l_prev[env];
        const double reward = S.reward_scale * (S.w_l * l + S.w_d * (l - lp) + S.w_s * (success ? 1.0 : 0.0));
        const int64_t steps = L.steps[env] + 1;
        const double ret = L.ep_return[env] + reward;
        const bool div = any_bad != 0;
        const bool term = success && !div;
        const bool trunc = !term && (steps >= S.max_steps || div);
        done = term || trunc;
        if (L.reward) L.reward[env] = reward;
        if (L.terminated) L.terminated[env] = term;
        if (L.truncated) L.truncated[env] = trunc;
        if (L.distance) L.distance[env] = l;
        if (L.success) L.success[env] = success;
        if (L.diverged) L.diverged[env] = div;
        if (L.clipped) L.clipped[env] = sc.clipped;
        if (L.contacts) L.contacts[env] = sc.n_contacts;
        if (L.ret_out) L.ret_out[env] = ret;
        if (L.len_out) L.len_out[env] = steps;
        if (L.done_mask) L.done_mask[env] = done;
        double o[6];
        for (int c = 0; c < 3; ++c) { o[c] = 2.0 * (drag[c] - S.lo[c]) / (S.hi[c] - S.lo[c]) - 1.0; o[3 + c] = S.target_obs[c]; }
        if (L.final_obs) {
            for (int c = 0; c < 6; ++c) {
                const double val = done ? o[c] : 0.0;
                if (L.obs_f64) reinterpret_cast<double *>(L.final_obs)[6 * env + c] = val;
                else reinterpret_cast<float *>(L.final_obs)[6 * env + c] = (float)val;
            }
        }
        if (done) {
            for (int c = 0; c < 3; ++c) { p.ax[c] = S.start_axis[c]; p.jw[c] = S.start_jaw[c]; }
            p.reach = S.start_reach; p.clamp = S.start_clamp;
            for (int c = 0; c < 3; ++c) o[c] = 2.0 * ((S.rcm[c] + p.reach * p.ax[c]) - S.lo[c]) / (S.hi[c] - S.lo[c]) - 1.0;
            L.steps[env] = 0; L.ep_return[env] = 0.0; L.l_prev[env] = S.start_distance;
        } else {
            L.steps[env] = steps; L.ep_return[env] = ret; L.l_prev[env] = l;
        }
        if (L.obs) {
            for (int c = 0; c < 6; ++c) {
                if (L.obs_f64) reinterpret_cast<double *>(L.obs)[6 * env + c] = o[c];
                else reinterpret_cast<float *>(L.obs)[6 * env + c] = (float)o[c];
            }
        }
    } else {
        if (L.diverged) L.diverged[env] = any_bad != 0;
        if (L.clipped) L.clipped[env] = sc.clipped;
        if (L.rejected) L.rejected[env] = sc.rejected;
        if (L.contacts) L.contacts[env] = sc.n_contacts;
    }
    if (L.axis != nullptr && !(mode & TS_M_DETECT_ONLY) && !(mode & TS_M_EXT_GRASP)) {
        for (int c = 0; c < 3; ++c) { L.axis[3 * env + c] = p.ax[c]; L.jaw[3 * env + c] = p.jw[c]; }
        L.reach[env] = p.reach; L.clamp[env] = p.clamp;
        L.grasp_vertex[env] = done ? -1 : gv_new;
    }
}

// per-env stages, one thread per environment
static __global__ void __launch_bounds__(128) cmd_kernel(const __grid_constant__ TsDevProg P,
                                                  const __grid_constant__ TsParams S,
                                                  const __grid_constant__ TsLaunch L) {
    if (blockIdx.x == 0 && P.pf_base && !(S.ablate & 512)) {
        // the step kernel that follows reads the whole program every substep: start its L2 fill
        // now (bulk prefetch, 16 KB per request, fire and forget) -- after an L2 flush the
        // first substep of a small batch otherwise waits on HBM for every program line
        const char *b = reinterpret_cast<const char *>(P.pf_base);
        for (int64_t off = 16384 * (int64_t)threadIdx.x; off < P.pf_bytes; off += 16384 * (int64_t)blockDim.x) {
            const unsigned n = (unsigned)min((int64_t)16384, P.pf_bytes - off);
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(b + off), "r"(n) : "memory");
        }
    }
    // launched with programmatic dependent launch: the prefetch above overlaps the stream's previous
    // kernel (e.g. the action producer); its outputs are read only after this wait
    pdl_wait();
    // the step kernel may launch now (it reads the state and the action-check flag before its own
    // pdl_wait: both are final once this kernel's predecessors are)
    pdl_trigger();
    if ((L.mode & TS_M_CHECK_ACTIONS) && *L.bad_flag) return;   // deferred ValidationError
    for (int64_t env = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; env < L.n_env;
         env += (int64_t)gridDim.x * blockDim.x)
        env_command(P, S, L, env, L.cmd[env]);
}

static __global__ void __launch_bounds__(128) epilogue_kernel(const __grid_constant__ TsDevProg P,
                                                       const __grid_constant__ TsParams S,
                                                       const __grid_constant__ TsLaunch L) {
    pdl_wait();      // every step-kernel result of this step is visible after this
    if ((L.mode & TS_M_CHECK_ACTIONS) && *L.bad_flag) return;
    for (int64_t env = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; env < L.n_env;
         env += (int64_t)gridDim.x * blockDim.x)
        env_epilogue(S, L, env, L.cmd[env]);
}

// ---------------------------------------------------------------------------
// thread-block cluster primitives (large-mesh mode: one cluster of K CTAs per env)
// ---------------------------------------------------------------------------
namespace cl {
__device__ __forceinline__ unsigned rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ unsigned cluster_id() {
    unsigned r;
    asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
    return r;
}
__device__ __forceinline__ unsigned n_clusters() {
    unsigned r;
    asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
    return r;
}
// all threads of all CTAs of the cluster; release/acquire orders the DSMEM traffic around it
__device__ __forceinline__ void sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t saddr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
// the same shared-memory offset in CTA `r` of the cluster
__device__ __forceinline__ uint32_t map(uint32_t a, unsigned r) {
    uint32_t o;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r));
    return o;
}
__device__ __forceinline__ void st(uint32_t a, float v) { asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory"); }
__device__ __forceinline__ void st(uint32_t a, double v) { asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory"); }
__device__ __forceinline__ void st(uint32_t a, int v) { asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(a), "r"(v) : "memory"); }
template <typename T> __device__ __forceinline__ T ld(uint32_t a);
template <> __device__ __forceinline__ float ld<float>(uint32_t a) {
    float v;
    asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(a) : "memory");
    return v;
}
template <> __device__ __forceinline__ double ld<double>(uint32_t a) {
    double v;
    asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
    return v;
}
template <> __device__ __forceinline__ int ld<int>(uint32_t a) {
    int v;
    asm volatile("ld.shared::cluster.s32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
template <> __device__ __forceinline__ unsigned ld<unsigned>(uint32_t a) {
    unsigned v;
    asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
}  // namespace cl

// Cluster parts: push owned free vertex p's position (x, y, z) into the halo copies other CTAs
// keep of it, in their buffer at the same shared-memory offset as `buf` here.
template <typename Real>
__device__ __forceinline__ void halo_send(const TsDevProg &P, const Real *buf, int p, Real x, Real y, Real z) {
    const int k1 = P.send_off[p + 1];
    for (int k = P.send_off[p]; k < k1; ++k) {
        const int sd = P.send[k];
        const uint32_t a = cl::map(cl::saddr(buf + 3 * (sd & 0xfffff)), (unsigned)sd >> 20);
        cl::st(a, x); cl::st(a + sizeof(Real), y); cl::st(a + 2 * sizeof(Real), z);
    }
}

// ---------------------------------------------------------------------------
// the fused step of one environment
// ---------------------------------------------------------------------------
// CL = false: this CTA owns the whole env.  CL = true: this CTA is rank `rank` of the env's
// cluster (program P = progs[rank]); it owns part of the vertices and keeps a halo of the rest
// current over DSMEM; grasp search, contacts and the divergence flag are cluster-wide.
template <typename Real, int VPT, bool CL, bool EO = false, bool FAST = false>
__device__ __forceinline__ void step_env(const TsDevProg &P, const TsDevProg *progs, const TsParams &S,
                                         const TsLaunch &L, Smem<Real> &m, int64_t env, unsigned rank) {
    Scal &sc = *m.sc;
    const int t = threadIdx.x;
    const int B = blockDim.x;
    const int lane = t & 31;
    const int mode = L.mode;
    const Real h = prm<Real>(S.h, S.h_f), damp = prm<Real>(S.damp, S.damp_f);
    const Real inv_h = prm<Real>(1.0 / S.h, S.inv_h_f);   // fp32 build: v += d * (1/h)
    const Real gx = prm<Real>(S.g[0], S.g_f[0]), gy = prm<Real>(S.g[1], S.g_f[1]), gz = prm<Real>(S.g[2], S.g_f[2]);
    const Real ks = prm<Real>(S.ks, S.ks_f), kv = prm<Real>(S.kv, S.kv_f);
    const Real *wst = reinterpret_cast<const Real *>(P.w);
    const Real *rest = reinterpret_cast<const Real *>(P.rest);
    const int K = CL ? P.cluster_k : 1;

    Real *xg = reinterpret_cast<Real *>(L.x) + env * (int64_t)P.V * 3;
    Real *vg = reinterpret_cast<Real *>(L.v) + env * (int64_t)P.V * 3;

    // FAST (one chunk): the per-vertex program words are substep-invariant -> registers, loaded first
    // so their (after an L2 flush, HBM) latency overlaps the state load and the command kernel
    int h_base[VPT], h_val[VPT], h_pre[VPT], h_cnt[VPT], h_ev[VPT], h_rb[VPT];
    int h_tb = 0, h_wb = 0, h_we = 0;   // FAST: the chunk's tet base and this warp's range
    // cluster parts (a few warps per CTA, latency-bound): the substep-invariant per-vertex words
    // in registers too -- counts and edge rows always, chunk 0's slot rows when it is the only one
    // (also the fp64 one-vertex-per-thread kernels: one CTA at 1-2 per SM, latency-bound; not the fp64
    // cluster kernels, out of registers already)
    constexpr bool HC = (CL && sizeof(Real) == 4) || (!CL && !FAST && sizeof(Real) == 8 && VPT == 1 && !EO) ||
                       (EO && sizeof(Real) == 4);   // the edges kernel: counts and edge rows
    const bool hc1 = HC && P.n_chunks == 1;
    if constexpr (HC) {
        const TsChunk ch0 = P.chunks[0];
#pragma unroll
        for (int r = 0; r < VPT; ++r) {
            const int p = max(0, min(r * B + t, P.Vf - 1));
            h_cnt[r] = P.static_cnt[p];
            h_ev[r] = P.edge_gather ? P.evalence[p] : 0;
            h_rb[r] = P.edge_gather ? P.eregion[p >> 5] + lane : 0;
            h_base[r] = hc1 ? P.region[ch0.region_off + (p >> 5)] + lane : 0;
            h_val[r] = hc1 ? P.valence[ch0.val_off + p] : 0;
            h_pre[r] = hc1 ? min(h_val[r], P.gsplit[p]) : 0;
        }
    }
    if constexpr (FAST) {
        const TsChunk ch0 = P.chunks[0];
        h_tb = ch0.tet_begin;
        h_wb = P.wsplit[t >> 5];
        h_we = P.wsplit[(t >> 5) + 1];
#pragma unroll
        for (int r = 0; r < VPT; ++r) {
            const int p = max(0, min(r * B + t, P.Vf - 1));   // rows past Vf are never used
            h_base[r] = 12 * (P.Vstore + P.region[ch0.region_off + (p >> 5)] + lane);   // bytes from smem_base
            h_val[r] = P.valence[ch0.val_off + p];
            h_pre[r] = min(h_val[r], P.gsplit[p]);
            h_cnt[r] = P.static_cnt[p];
            h_ev[r] = P.evalence[p];
            h_rb[r] = P.eregion[p >> 5] + lane;
        }
    }
    // ---- A. the state load, then the env's command block (cmd_kernel) ---
    // state -> shared (storage order) / registers: the command kernel does not write x / v, so
    // under programmatic dependent launch this overlaps the command kernel's tail
    for (int p = t; p < P.Vstore; p += B) {
        const int o = P.s2o[p];
        Real a = 0, b = 0, c = 0;
        // state is read once per env-step: streaming loads keep L1 for the program streams
        if (o >= 0) { a = __ldcs(xg + 3 * o); b = __ldcs(xg + 3 * o + 1); c = __ldcs(xg + 3 * o + 2); }
        m.X(p) = a; m.Y(p) = b; m.Z(p) = c;
        m.alt[3 * p] = a; m.alt[3 * p + 1] = b; m.alt[3 * p + 2] = c;   // pinned rows of the ping-pong
    }
    Real vx[VPT], vy[VPT], vz[VPT];
#pragma unroll
    for (int r = 0; r < VPT; ++r) {
        const int p = r * B + t;
        vx[r] = vy[r] = vz[r] = 0;
        if (p < P.Vf) {
            const int o = P.s2o[p];
            vx[r] = __ldcs(vg + 3 * o); vy[r] = __ldcs(vg + 3 * o + 1); vz[r] = __ldcs(vg + 3 * o + 2);
        }
    }
    for (int p = t; p < (P.narrow ? P.Vf_pad / 4 : P.Vf_pad); p += B) m.deg[p] = 0;
    if constexpr (FAST || EO) {   // dictionary tables -> shared memory (read by every tet / edge of every substep)
        float *tab = const_cast<float *>(smem_tab(TS_TAB_OFF));
        for (int i = t; i < 2 * TS_TAB_CAP; i += B) {
            const int j = i - TS_TAB_CAP;
            // [edge pairs {rest, coef} | 6 V0 values]
            tab[i] = i < TS_TAB_CAP ? (i < 2 * P.n_rltab ? __ldg(P.rltab + i) : 0.0f) : (j < P.n_rvtab ? __ldg(P.rvtab + j) : 0.0f);
        }
    }
    for (int i = t; i < P.cbits_words; i += B) m.cbits[i] = 0u;
    pdl_wait();   // the command blocks (and the grasp flags the command kernel released) are ready
    TsCmd &cmd = L.cmd[env];
    if (t < 24) {
        const double *src = t < 21 ? &cmd.caps[0][0] + t : cmd.drag + (t - 21);
        (&sc.caps[0][0])[t] = *src;            // caps[21] and drag[3] are contiguous in Scal too
    } else if (t == 24) {
        sc.gv_orig = cmd.gv; sc.need_search = cmd.need_search; sc.n_contacts = 0;
    }
    if constexpr (CL) cl::sync();   // every CTA holds its halo before anyone pushes into it
    else __syncthreads();

    if (mode & (TS_M_CONTACTS | TS_M_DETECT_ONLY)) {
        if (t < 3) make_cap<Real>(sc.caps[t], m.caps[t]);
        __syncthreads();
    }
    // ---- B. grasp search: nearest free vertex (tool.py:380-389) ------
    if (sc.need_search && !(S.ablate & 16)) {
        double bk = INFINITY;
        int bi = 0x7fffffff;
        for (int p = t; p < P.Vf; p += B) {
            const double r0 = (double)m.X(p) - sc.drag[0];
            const double r1 = (double)m.Y(p) - sc.drag[1];
            const double r2 = (double)m.Z(p) - sc.drag[2];
            double d2 = r0 * r0 + r1 * r1 + r2 * r2;
            if (isnan(d2)) d2 = -INFINITY;      // numpy argmin returns the first NaN
            const int o = P.s2o[p];
            if (d2 < bk || (d2 == bk && o < bi)) { bk = d2; bi = o; }
        }
        for (int off = 16; off > 0; off >>= 1) {
            const double ok = __shfl_xor_sync(0xffffffffu, bk, off);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
            if (ok < bk || (ok == bk && oi < bi)) { bk = ok; bi = oi; }
        }
        if (lane == 0) { sc.red_key[t >> 5] = bk; sc.red_idx[t >> 5] = bi; }
        __syncthreads();
        if (t == 0) {
            for (int wi = 1; wi < (B >> 5); ++wi) {
                if (sc.red_key[wi] < bk || (sc.red_key[wi] == bk && sc.red_idx[wi] < bi)) {
                    bk = sc.red_key[wi]; bi = sc.red_idx[wi];
                }
            }
            if constexpr (CL) {   // cluster-wide argmin: every part's winner to rank 0
                cl::st(cl::map(cl::saddr(&sc.cl_key[rank]), 0), bk);
                cl::st(cl::map(cl::saddr(&sc.cl_idx[rank]), 0), bi);
            }
        }
        if constexpr (CL) {
            cl::sync();
            if (t == 0) {
                for (int r = 0; r < K; ++r) {
                    const double ok = cl::ld<double>(cl::map(cl::saddr(&sc.cl_key[r]), 0));
                    const int oi = cl::ld<int>(cl::map(cl::saddr(&sc.cl_idx[r]), 0));
                    if (r == 0 || ok < bk || (ok == bk && oi < bi)) { bk = ok; bi = oi; }
                }
            }
        }
        if (t == 0) {
            if (bi != 0x7fffffff && bk != -INFINITY && bk <= S.grasp_r2) {
                sc.gv_orig = bi;
                if (rank == 0) L.grasped[env * P.V + bi] = 1;
            }
        }
        __syncthreads();
    }
    // grasp vertex in storage order (any vertex; pinned ones are never applied)
    const int gvs = sc.gv_orig >= 0 ? P.o2s[sc.gv_orig] : -1;

    // ---- C. substeps ---------------------------------------------------
    if ((mode & TS_M_SUBSTEPS) && !(S.ablate & 64)) {
        Real xr[VPT], yr[VPT], zr[VPT], accx[VPT], accy[VPT], accz[VPT];
        int ndeg[VPT], gcnt[VPT];
#pragma unroll
        for (int r = 0; r < VPT; ++r) {
            const int p = r * B + t;
            accx[r] = accy[r] = accz[r] = 0; ndeg[r] = 0; gcnt[r] = 0;
            xr[r] = yr[r] = zr[r] = 0;
            if (p < P.Vf) {
                // predict for substep 0 (ts_lane_predict, _kernels.pyx:63-87)
                vx[r] += h * gx; xr[r] = m.X(p) + h * vx[r];
                vy[r] += h * gy; yr[r] = m.Y(p) + h * vy[r];
                vz[r] += h * gz; zr[r] = m.Z(p) + h * vz[r];
                m.X(p) = xr[r]; m.Y(p) = yr[r]; m.Z(p) = zr[r];
                if constexpr (CL) halo_send<Real>(P, m.pos, p, xr[r], yr[r], zr[r]);
            }
        }
        if constexpr (CL) cl::sync();
        else __syncthreads();
        const double d0 = sc.drag[0], d1 = sc.drag[1], d2 = sc.drag[2];
        // grasp contribution of owner slot r: after the vertex's edges (_kernels.pyx:283-298)
        auto add_grasp = [&](int r) {
            const int p = r * B + t;
            if (p < P.Vf && p == gvs) {
                const Real dx = (Real)(d0 - (double)xr[r]);
                const Real dy = (Real)(d1 - (double)yr[r]);
                const Real dz = (Real)(d2 - (double)zr[r]);
                const Real dist = sqrt(dx * dx + dy * dy + dz * dz);
                if (!(dist <= (Real)1e-12)) { accx[r] += dx; accy[r] += dy; accz[r] += dz; gcnt[r] = 1; }
            }
        };
        for (int s = 0; s < S.substeps; ++s) {
            if constexpr (!EO) for (int c = 0; c < (FAST ? 1 : P.n_chunks); ++c) {
                const TsChunk ch = P.chunks[c];
                // owner-gathered edges need only the position snapshot: they run in phase 1 of the
                // first chunk, next to this warp's share of the tets (the compiler sized the shares so
                // that edges + tets take about the same time in every warp); they still come first in
                // each vertex's sum, the reference order
                if (P.edge_gather && c == 0 && !(S.ablate & 4)) {
#pragma unroll
                    for (int r = 0; r < VPT; ++r) {
                        const int p = r * B + t;
                        if (p < P.Vf)
                            owner_edges<Real, FAST, FAST || HC>(P, m, p, lane, xr[r], yr[r], zr[r], ks, accx[r],
                                                                accy[r], accz[r], ndeg[r], h_ev[r], h_rb[r]);
                    }
                }
                // phase 1: every kind of the chunk, no barrier in between (disjoint slots)
                if (!FAST && ch.edge_count) p1_edges<Real>(P, m, ch.edge_begin, ch.edge_count, ks);
                if (!FAST && ch.att_count) p1_atts<Real>(P, m, ch.att_begin, ch.att_count);
                if ((FAST || ch.tet_count) && !(S.ablate & 1)) {
                    if constexpr (FAST) {
                        if (P.n_rvtab <= 4) p1_tets_fast<true>(P, m.deg, h_tb, h_wb, h_we, kv);
                        else p1_tets_fast<false>(P, m.deg, h_tb, h_wb, h_we, kv);
                    } else {
                        const int *ws = P.wsplit + c * (B / 32 + 1) + (t >> 5);
                        p1_tets<Real, FAST>(P, m, ch.tet_begin, ws[0], ws[1], kv);
                    }
                }
                __syncthreads();
                // phase 2: owner gathers its slots in reference order
                const bool gchunk = FAST || c == P.grasp_chunk;
#pragma unroll
                for (int r = 0; r < VPT; ++r) {
                    const int p = r * B + t;
                    if (p < P.Vf) {
                        const int base = FAST ? 0 : hc1 ? h_base[r] : P.region[ch.region_off + (p >> 5)] + lane;
                        const int val0 = FAST || hc1 ? h_val[r] : P.valence[ch.val_off + p];
                        const int val = (S.ablate & 2) ? 0 : ((S.ablate & 128) ? min(val0, 12) : val0);
                        const int pre = (FAST || hc1) && !(S.ablate & 130) ? h_pre[r]
                                        : gchunk ? min(val, P.gsplit[p]) : val;
                        Real ax = accx[r], ay = accy[r], az = accz[r];
                        // slot k of this vertex (FAST: a byte offset from the constant shared base)
                        auto add_slot = [&](int k) {
                            if constexpr (FAST) {
                                float qx, qy, qz;
                                lds3c(h_base[r] + 384 * k, qx, qy, qz);
                                ax += qx; ay += qy; az += qz;
                            } else {
                                const int sidx = base + 32 * k;
                                ax += m.SX(sidx); ay += m.SY(sidx); az += m.SZ(sidx);
                            }
                        };
#pragma unroll kSlotUnroll
                        for (int k = 0; k < pre; ++k) add_slot(k);
                        if (gchunk) {
                            accx[r] = ax; accy[r] = ay; accz[r] = az;
                            add_grasp(r);
                            ax = accx[r]; ay = accy[r]; az = accz[r];
                            for (int k = pre; k < val; ++k) add_slot(k);
                        }
                        accx[r] = ax; accy[r] = ay; accz[r] = az;
                        ndeg[r] += deg_take(FAST ? 1 : m.narrow, m.deg, p);
                    }
                }
                if (!FAST && c + 1 < P.n_chunks) __syncthreads();   // slots are reused by the next chunk
            }
            if (!FAST && P.grasp_chunk == P.n_chunks) {
#pragma unroll
                for (int r = 0; r < VPT; ++r) {
                    const int p = r * B + t;
                    if (P.edge_gather && P.n_chunks == 0 && p < P.Vf)   // distance constraints only
                        owner_edges<Real, false, HC, EO>(P, m, p, lane, xr[r], yr[r], zr[r], ks, accx[r],
                                                         accy[r], accz[r], ndeg[r], h_ev[r], h_rb[r]);
                    add_grasp(r);
                }
            }
            // apply (ts_lane_apply, _kernels.pyx:213-244) + next predict
#pragma unroll
            for (int r = 0; r < VPT; ++r) {
                const int p = r * B + t;
                if (p < P.Vf) {
                    const int cnt = (FAST || HC ? h_cnt[r] : P.static_cnt[p]) - ndeg[r] + gcnt[r];
                    if constexpr (sizeof(Real) == 8) {
                        const Real n = (Real)cnt;
                        const Real mm = (Real)0.5 + copysign((Real)0.5, n - (Real)0.5);
                        const Real inv = mm / (n + ((Real)1 - mm));
                        const Real e0 = accx[r] * inv, e1 = accy[r] * inv, e2 = accz[r] * inv;
                        xr[r] += e0; vx[r] += e0 / h;
                        yr[r] += e1; vy[r] += e1 / h;
                        zr[r] += e2; vz[r] += e2 / h;
                    } else {
                        const float inv = cnt > 0 ? rcp_ftz((float)cnt) : 0.0f;
                        const float e0 = accx[r] * inv, e1 = accy[r] * inv, e2 = accz[r] * inv;
                        xr[r] += e0; vx[r] = __fmaf_rn(e0, inv_h, vx[r]);
                        yr[r] += e1; vy[r] = __fmaf_rn(e1, inv_h, vy[r]);
                        zr[r] += e2; vz[r] = __fmaf_rn(e2, inv_h, vz[r]);
                    }
                    if (damp != (Real)1) { vx[r] *= damp; vy[r] *= damp; vz[r] *= damp; }
                    if (s + 1 < S.substeps) {
                        vx[r] += h * gx; xr[r] += h * vx[r];
                        vy[r] += h * gy; yr[r] += h * vy[r];
                        vz[r] += h * gz; zr[r] += h * vz[r];
                    }
                    // ping-pong when other owners may still read this substep's snapshot (distance-only
                    // gather in this phase, cluster halos); narrow programs write in place (alt == pos)
                    Real *dst = m.alt + 3 * p;
                    dst[0] = xr[r]; dst[1] = yr[r]; dst[2] = zr[r];
                    if constexpr (CL) halo_send<Real>(P, m.alt, p, xr[r], yr[r], zr[r]);
                    accx[r] = accy[r] = accz[r] = 0; ndeg[r] = 0; gcnt[r] = 0;
                }
            }
            if constexpr (CL) cl::sync();
            else __syncthreads();
            if (!FAST && P.edge_gather) {
                Real *cur = m.pos;
                m.pos = m.alt;
                m.alt = cur;
            }
        }
    }

    // ---- D. contacts ---------------------------------------------------
    if ((mode & (TS_M_CONTACTS | TS_M_DETECT_ONLY)) && (CL || P.F > 0) && !(S.ablate & 8)) {
        Cap<Real> *C = m.caps;   // built by threads 0..2 before the substeps
        Real *rec = m.slot;   // 3F records x 7 reals (the slot buffer is free now)
        // union of the three capsule boxes: one test rejects almost every face
        Real ulo[3], uhi[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            ulo[k] = cmin(cmin(C[0].lo[k], C[1].lo[k]), C[2].lo[k]);
            uhi[k] = cmax(cmax(C[0].hi[k], C[1].hi[k]), C[2].hi[k]);
        }
        for (int f = t; f < P.F; f += B) {
            const int ia = P.faces[3 * f], ib = P.faces[3 * f + 1], ic = P.faces[3 * f + 2];
            const Real pa[3] = {m.X(ia), m.Y(ia), m.Z(ia)};
            const Real pb[3] = {m.X(ib), m.Y(ib), m.Z(ib)};
            const Real pc[3] = {m.X(ic), m.Y(ic), m.Z(ic)};
            Real tlo[3], thi[3];
            bool any = true;
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                tlo[k] = cmin(cmin(pa[k], pb[k]), pc[k]);
                thi[k] = cmax(cmax(pa[k], pb[k]), pc[k]);
                any = any && !(thi[k] < ulo[k] || tlo[k] > uhi[k]);
            }
            if (!any) continue;
#pragma unroll
            for (int ci = 0; ci < 3; ++ci) {
                bool skip = false;
                for (int k = 0; k < 3; ++k)
                    if (thi[k] < C[ci].lo[k] || tlo[k] > C[ci].hi[k]) { skip = true; break; }
                if (skip) continue;
                Real dir[3], bary[3];
                const Real sd = witness<Real>(C[ci], pa, pb, pc, S.contact_iters, dir, bary);
                if (sd < (Real)0) {
                    const int key = ci * P.F + f;
                    Real *q = rec + 7 * key;
                    q[0] = -sd; q[1] = dir[0]; q[2] = dir[1]; q[3] = dir[2];
                    q[4] = bary[0]; q[5] = bary[1]; q[6] = bary[2];
                    atomicOr(&m.cbits[key >> 5], 1u << (key & 31));
                }
            }
        }
        __syncthreads();
        if constexpr (!CL) {
            if (t < 32) {
                // warp 0 finds the non-empty words (usually none); lane 0 walks them in order
                int count = 0;
                for (int wb = 0; wb < P.cbits_words; wb += 32) {
                  const unsigned word = wb + t < P.cbits_words ? m.cbits[wb + t] : 0u;
                  unsigned nz = __ballot_sync(0xffffffffu, word != 0u);
                  while (nz) {
                    const int l = __ffs(nz) - 1;
                    nz &= nz - 1;
                    unsigned bits = __shfl_sync(0xffffffffu, word, l);
                    const int wi = wb + l;
                    if (t == 0) while (bits) {
                        const int b = __ffs(bits) - 1;
                        bits &= bits - 1;
                        const int key = wi * 32 + b;
                        const int ci = key / P.F, f = key - ci * P.F;
                        const Real *q = rec + 7 * key;
                        if (mode & TS_M_DETECT_ONLY) {
                            const int64_t row = env * 3 * (int64_t)P.F + count;
                            L.det_face[row] = P.face_gid[f]; L.det_cap[row] = ci; L.det_depth[row] = (double)q[0];
                            for (int k = 0; k < 3; ++k) { L.det_dir[3 * row + k] = (double)q[1 + k]; L.det_bary[3 * row + k] = (double)q[4 + k]; }
                        } else {
                            // collision.resolve_contact_arrays, sequential in emission order
                            const Real b0 = q[4], b1 = q[5], b2 = q[6];
                            const Real bb = fused_sq3<Real>(b0, b1, b2);
                            if (bb > (Real)0) {
                                const Real sc_ = (Real)S.k_contact * q[0] / bb;
                                const Real px = sc_ * q[1], py = sc_ * q[2], pz = sc_ * q[3];
                                const Real bj[3] = {b0, b1, b2};
                                for (int j = 0; j < 3; ++j) {
                                    const int vs = P.faces[3 * f + j];
                                    if (wst[vs] > (Real)0) {
                                        m.X(vs) += bj[j] * px; m.Y(vs) += bj[j] * py; m.Z(vs) += bj[j] * pz;
                                    }
                                }
                            }
                        }
                        ++count;
                    }
                  }
                }
                if (t == 0) {
                    sc.n_contacts = count;
                    if (mode & TS_M_DETECT_ONLY) L.det_count[env] = count;
                }
            }
            __syncthreads();
        } else {
            // every part lists its contact keys in (capsule, local face) order -- local faces are
            // ascending global faces -- into its (now free) degenerate-counter array
            if (t == 0) {
                int n = 0;
                for (int wi = 0; wi < P.cbits_words; ++wi) {
                    unsigned bits = m.cbits[wi];
                    while (bits && n < P.Vf_pad) {
                        const int b = __ffs(bits) - 1;
                        bits &= bits - 1;
                        m.deg[n++] = wi * 32 + b;
                    }
                }
                sc.n_list = n;
            }
            cl::sync();
            // rank 0 merges the K lists in emission order (capsule-major, global face minor) and
            // applies the push-outs sequentially to the owners' positions (collision.py:55-73)
            if (rank == 0 && t == 0) {
                int count = 0;
                int head[TS_MAX_CLUSTER], nl[TS_MAX_CLUSTER];
                for (int r = 0; r < K; ++r) {
                    head[r] = 0;
                    nl[r] = cl::ld<int>(cl::map(cl::saddr(&sc.n_list), r));
                }
                for (int ci = 0; ci < 3; ++ci) {
                    while (true) {
                        int best_r = -1, best_g = 0x7fffffff, best_f = 0;
                        for (int r = 0; r < K; ++r) {
                            if (head[r] >= nl[r]) continue;
                            const TsDevProg &Q = progs[r];
                            const int key = cl::ld<int>(cl::map(cl::saddr(&m.deg[head[r]]), r));
                            const int kc = key / Q.F;
                            if (kc != ci) continue;
                            const int f = key - kc * Q.F;
                            const int g = Q.face_gid[f];
                            if (g < best_g) { best_g = g; best_r = r; best_f = f; }
                        }
                        if (best_r < 0) break;
                        const TsDevProg &Q = progs[best_r];
                        const int key = ci * Q.F + best_f;
                        const uint32_t qa = cl::map(cl::saddr(rec + 7 * key), best_r);
                        Real q[7];
                        for (int k = 0; k < 7; ++k) q[k] = cl::ld<Real>(qa + k * sizeof(Real));
                        if (mode & TS_M_DETECT_ONLY) {
                            const int64_t row = env * 3 * (int64_t)S.n_face + count;
                            L.det_face[row] = best_g; L.det_cap[row] = ci; L.det_depth[row] = (double)q[0];
                            for (int k = 0; k < 3; ++k) { L.det_dir[3 * row + k] = (double)q[1 + k]; L.det_bary[3 * row + k] = (double)q[4 + k]; }
                        } else {
                            const Real b0 = q[4], b1 = q[5], b2 = q[6];
                            const Real bb = fused_sq3<Real>(b0, b1, b2);
                            if (bb > (Real)0) {
                                const Real sc_ = (Real)S.k_contact * q[0] / bb;
                                const Real px = sc_ * q[1], py = sc_ * q[2], pz = sc_ * q[3];
                                const Real bj[3] = {b0, b1, b2};
                                for (int j = 0; j < 3; ++j) {
                                    const int ow = Q.face_own[3 * best_f + j];
                                    if (ow < 0) continue;   // pinned
                                    const uint32_t a = cl::map(cl::saddr(m.pos + 3 * (ow & 0xfffff)), (unsigned)ow >> 20);
                                    cl::st(a, cl::ld<Real>(a) + bj[j] * px);
                                    cl::st(a + sizeof(Real), cl::ld<Real>(a + sizeof(Real)) + bj[j] * py);
                                    cl::st(a + 2 * sizeof(Real), cl::ld<Real>(a + 2 * sizeof(Real)) + bj[j] * pz);
                                }
                            }
                        }
                        ++head[best_r];
                        ++count;
                    }
                }
                sc.n_contacts = count;
                if (mode & TS_M_DETECT_ONLY) L.det_count[env] = count;
            }
            cl::sync();
        }
    }

    // ---- E. divergence guard (solver.py:357-359) ----------------------
    int bad = 0;
    for (int p = t; p < P.Vown; p += B)
        bad |= !(isfinite(m.X(p)) && isfinite(m.Y(p)) && isfinite(m.Z(p)));
    int any_bad = __syncthreads_or(bad);
    if constexpr (CL) {
        if (t == 0) cl::st(cl::map(cl::saddr(&sc.cl_flag[rank]), 0), any_bad);
        cl::sync();
        if (t == 0) {
            int a = 0;
            for (int r = 0; r < K; ++r) a |= cl::ld<int>(cl::map(cl::saddr(&sc.cl_flag[r]), 0));
            sc.any_bad = a;
        }
        __syncthreads();
        any_bad = sc.any_bad;
    }

    // ---- F. hand the step's results to the epilogue kernel -------------
    // done = terminated || truncated = success || steps >= max || diverged (env.py:173-175)
    if (t == 0 && rank == 0) {
        cmd.gv = sc.gv_orig; cmd.any_bad = any_bad; cmd.n_contacts = sc.n_contacts;
    }
    const bool done_env = (mode & TS_M_ENV) && (cmd.pre_done || any_bad);

    // ---- G. write back (owned vertices) ----------------------------------
    if (!(mode & TS_M_DETECT_ONLY)) {
        const bool done = done_env;
        if (done)
            for (int i = t * K + (int)rank; i < P.V; i += B * K) L.grasped[env * P.V + i] = 0;
#pragma unroll
        for (int r = 0; r < VPT; ++r) {
            const int p = r * B + t;
            if (p < P.Vf) {
                const int o = P.s2o[p];
                if (done) {
                    xg[3 * o] = rest[3 * o]; xg[3 * o + 1] = rest[3 * o + 1]; xg[3 * o + 2] = rest[3 * o + 2];
                    vg[3 * o] = 0; vg[3 * o + 1] = 0; vg[3 * o + 2] = 0;
                } else {
                    xg[3 * o] = m.X(p); xg[3 * o + 1] = m.Y(p); xg[3 * o + 2] = m.Z(p);
                    vg[3 * o] = vx[r]; vg[3 * o + 1] = vy[r]; vg[3 * o + 2] = vz[r];
                }
            }
        }
        for (int p = P.Vf_pad + t; p < P.Vown; p += B) {
            const int o = P.s2o[p];
            if (o < 0) continue;
            if (done) { xg[3 * o] = rest[3 * o]; xg[3 * o + 1] = rest[3 * o + 1]; xg[3 * o + 2] = rest[3 * o + 2]; }
            else if (mode & TS_M_CONTACTS) { xg[3 * o] = m.X(p); xg[3 * o + 1] = m.Y(p); xg[3 * o + 2] = m.Z(p); }
            if (mode & TS_M_SUBSTEPS || done) { vg[3 * o] = 0; vg[3 * o + 1] = 0; vg[3 * o + 2] = 0; }
        }
    }
    if constexpr (CL) cl::sync();   // no CTA of the cluster still reads this one's shared memory
    else __syncthreads();           // shared scalars are reused by the next environment
}

template <typename Real, int VPT>
__global__ void __launch_bounds__(TS_STEP_MAXT, sizeof(Real) == 4 ? TS_STEP_MINB : 1) step_kernel(const __grid_constant__ TsDevProg P,
                                                   const __grid_constant__ TsParams S,
                                                   const __grid_constant__ TsLaunch L) {
    pdl_trigger();   // the epilogue may launch early; it waits for this grid before reading
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem<Real> m = carve<Real>(P, smem_raw);
    if ((L.mode & TS_M_CHECK_ACTIONS) && *L.bad_flag) return;   // deferred ValidationError: no state change
    for (int64_t env = blockIdx.x; env < L.n_env; env += gridDim.x)
        step_env<Real, VPT, false>(P, nullptr, S, L, m, env, 0);
}

// The fp64 validation build of a one-vertex-per-thread program of at most 320 threads: two CTAs per
// SM (at most 102 registers; two fp64 reach CTAs fit the shared memory) instead of one.
template <typename Real>
__global__ void __launch_bounds__(320, 2) step2_kernel(const __grid_constant__ TsDevProg P,
                                                   const __grid_constant__ TsParams S,
                                                   const __grid_constant__ TsLaunch L) {
    pdl_trigger();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem<Real> m = carve<Real>(P, smem_raw);
    if ((L.mode & TS_M_CHECK_ACTIONS) && *L.bad_flag) return;
    for (int64_t env = blockIdx.x; env < L.n_env; env += gridDim.x)
        step_env<Real, 1, false>(P, nullptr, S, L, m, env, 0);
}

// The reach-scene shape (fp32, one CTA, one chunk, owner-gathered edges in 4-byte records, byte-offset
// tet stream with dictionary-coded volumes, no attachments, narrow layout): every layout test resolved
// at compile time.  ts_fast_program() is the host-side test.
template <typename Real>
__global__ void __launch_bounds__(TS_STEP_MAXT, TS_STEP_MINB) fast_step_kernel(const __grid_constant__ TsDevProg P,
                                                                              const __grid_constant__ TsParams S,
                                                                              const __grid_constant__ TsLaunch L) {
    pdl_trigger();   // the epilogue may launch early; it waits for this grid before reading
    extern __shared__ __align__(16) unsigned char smem_raw[];
    if (smem_u32(0) != TS_SMEM_WINDOW) __trap();   // constant shared addresses (lds3c): never silently wrong
    Smem<Real> m = carve<Real>(P, smem_raw);
    if ((L.mode & TS_M_CHECK_ACTIONS) && *L.bad_flag) return;
    for (int64_t env = blockIdx.x; env < L.n_env; env += gridDim.x)
        step_env<Real, 1, false, false, true>(P, nullptr, S, L, m, env, 0);
}

// Distance-constraint-only programs (no chunks: SURVEY §8(d) config 2): the same step with the slot
// machinery compiled out (measured 0.101 vs 0.124 ms/step at 1024 envs; more CTAs per SM at fewer
// registers were slower: 0.118-0.123 ms, profiles/r01i/negative_results.txt).
template <typename Real>
__global__ void __launch_bounds__(TS_EDGES_MAXT, TS_EDGES_MINB) edges_step_kernel(const __grid_constant__ TsDevProg P,
                                                            const __grid_constant__ TsParams S,
                                                            const __grid_constant__ TsLaunch L) {
    pdl_trigger();   // the epilogue may launch early; it waits for this grid before reading
    extern __shared__ __align__(16) unsigned char smem_raw[];
    if (smem_u32(0) != TS_SMEM_WINDOW) __trap();   // constant shared addresses (lds2c): never silently wrong
    Smem<Real> m = carve<Real>(P, smem_raw);
    if ((L.mode & TS_M_CHECK_ACTIONS) && *L.bad_flag) return;
    for (int64_t env = blockIdx.x; env < L.n_env; env += gridDim.x)
        step_env<Real, 1, false, true>(P, nullptr, S, L, m, env, 0);
}

// Large-mesh mode: a thread-block cluster of K CTAs per environment (grid = K x clusters).
template <typename Real, int VPT>
__global__ void __launch_bounds__(512, 1) cluster_step_kernel(const TsDevProg *__restrict__ progs,
                                                              const __grid_constant__ TsParams S,
                                                              const __grid_constant__ TsLaunch L) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const unsigned rank = cl::rank();
    const TsDevProg &P = progs[rank];
    Smem<Real> m = carve<Real>(P, smem_raw);
    if ((L.mode & TS_M_CHECK_ACTIONS) && *L.bad_flag) return;   // the same verdict in every CTA
    for (int64_t env = cl::cluster_id(); env < L.n_env; env += cl::n_clusters())
        step_env<Real, VPT, true>(P, progs, S, L, m, env, rank);
}

// ---------------------------------------------------------------------------
// reset / observe (EnvBatch.reset, env.py:123-142) -- one thread per (env, vertex)
// ---------------------------------------------------------------------------
template <typename Real>
__global__ void reset_kernel(const TsDevProg P, const TsParams S, const TsLaunch L, const uint8_t *mask,
                             int observe_only) {
    const int64_t n = L.n_env;
    const int64_t V = P.V;
    const Real *rest = reinterpret_cast<const Real *>(P.rest);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * V; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t env = i / V, vtx = i - env * V;
        const bool sel = !observe_only && (mask == nullptr || mask[env] != 0);
        if (sel) {
            Real *x = reinterpret_cast<Real *>(L.x) + 3 * i;
            Real *v = reinterpret_cast<Real *>(L.v) + 3 * i;
            x[0] = rest[3 * vtx]; x[1] = rest[3 * vtx + 1]; x[2] = rest[3 * vtx + 2];
            v[0] = 0; v[1] = 0; v[2] = 0;
            L.grasped[i] = 0;
        }
        if (vtx == 0) {
            if (sel) {
                for (int c = 0; c < 3; ++c) { L.axis[3 * env + c] = S.start_axis[c]; L.jaw[3 * env + c] = S.start_jaw[c]; }
                L.reach[env] = S.start_reach; L.clamp[env] = S.start_clamp;
                L.grasp_vertex[env] = -1;
                if (L.steps) L.steps[env] = 0;
                if (L.ep_return) L.ep_return[env] = 0.0;
                if (L.l_prev) L.l_prev[env] = S.start_distance;
            }
            if (L.obs) {
                double ax[3], reach;
                if (sel) { for (int c = 0; c < 3; ++c) ax[c] = S.start_axis[c]; reach = S.start_reach; }
                else { for (int c = 0; c < 3; ++c) ax[c] = L.axis[3 * env + c]; reach = L.reach[env]; }
                for (int c = 0; c < 6; ++c) {
                    const double val = c < 3 ? 2.0 * ((S.rcm[c] + reach * ax[c]) - S.lo[c]) / (S.hi[c] - S.lo[c]) - 1.0
                                             : S.target_obs[c - 3];
                    if (L.obs_f64) reinterpret_cast<double *>(L.obs)[6 * env + c] = val;
                    else reinterpret_cast<float *>(L.obs)[6 * env + c] = (float)val;
                }
            }
        }
    }
}

}  // namespace tsk

// launch `fn` normally, or with programmatic stream serialization (PDL) so that it may start while
// the stream's previous kernel finishes (the kernel calls pdl_wait before consuming its results)
template <typename... Args>
static cudaError_t ts_launch_pdl(void (*fn)(Args...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                                 bool pdl, const TsDevProg &P, const TsParams &S, const TsLaunch &L) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = pdl ? attr : nullptr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, fn, P, S, L);
}

// ---------------------------------------------------------------------------
// launchers (instantiated per precision in step_f32.cu / step_f64.cu)
// ---------------------------------------------------------------------------
template <typename Real>
cudaError_t ts_launch_step(const TsDevProg &P, const TsParams &S, const TsLaunch &L, int grid, int smem,
                           cudaStream_t stream, bool pdl) {
    void (*fn)(const TsDevProg, const TsParams, const TsLaunch) = nullptr;
    if constexpr (sizeof(Real) == 4) {   // shape-specialised fp32 kernels
        if (ts_use_fast_kernel(P, S.ablate)) fn = tsk::fast_step_kernel<Real>;
        else if (ts_use_edges_kernel(P)) fn = tsk::edges_step_kernel<Real>;
    } else {
        if (P.VPT == 1 && P.B <= 320 && !(S.ablate & 2048)) fn = tsk::step2_kernel<Real>;
    }
    if (!fn) switch (P.VPT) {
        case 1: fn = tsk::step_kernel<Real, 1>; break;
        case 2: fn = tsk::step_kernel<Real, 2>; break;
        case 4: fn = tsk::step_kernel<Real, 4>; break;
        case 8: fn = tsk::step_kernel<Real, 8>; break;
        default:
            if (P.VPT == 3) fn = tsk::step_kernel<Real, 4>;
            else if (P.VPT <= 8) fn = tsk::step_kernel<Real, 8>;
            else return cudaErrorInvalidValue;
    }
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    return ts_launch_pdl(fn, dim3((unsigned)grid), dim3((unsigned)P.B), (size_t)smem, stream, pdl, P, S, L);
}

template <typename Real>
cudaError_t ts_launch_cluster_step(const TsDevProg *parts, int VPT, int K, int B, const TsParams &S,
                                   const TsLaunch &L, int n_clusters, int smem, cudaStream_t stream) {
    void (*fn)(const TsDevProg *, const TsParams, const TsLaunch) = nullptr;
    if (VPT <= 1) fn = tsk::cluster_step_kernel<Real, 1>;
    else if (VPT <= 2) fn = tsk::cluster_step_kernel<Real, 2>;
    else if (VPT <= 4) fn = tsk::cluster_step_kernel<Real, 4>;
    else return cudaErrorInvalidValue;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    if (K > 8) {
        e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(n_clusters * K), 1, 1);
    cfg.blockDim = dim3((unsigned)B, 1, 1);
    cfg.dynamicSmemBytes = (size_t)smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)K;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, fn, parts, S, L);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

template <typename Real>
cudaError_t ts_launch_reset(const TsDevProg &P, const TsParams &S, const TsLaunch &L, const uint8_t *mask,
                            int observe_only, cudaStream_t stream) {
    const int64_t total = L.n_env * (int64_t)(P.V > 0 ? P.V : 1);
    int grid = (int)((total + 255) / 256);
    if (grid > 65535 * 4) grid = 65535 * 4;
    if (grid < 1) grid = 1;
    tsk::reset_kernel<Real><<<grid, 256, 0, stream>>>(P, S, L, mask, observe_only);
    return cudaGetLastError();
}

#ifdef TS_DEFINE_SCALAR_KERNELS
static int scalar_grid(int64_t n) {
    int64_t g = (n + 127) / 128;
    return (int)(g < 1 ? 1 : (g > 65535 ? 65535 : g));
}

cudaError_t ts_launch_cmd(const TsDevProg &P, const TsParams &S, const TsLaunch &L, cudaStream_t stream,
                          bool pdl) {
    cudaError_t e = ts_launch_pdl(tsk::cmd_kernel, dim3((unsigned)scalar_grid(L.n_env)), dim3(128), 0, stream, pdl,
                                  P, S, L);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

cudaError_t ts_launch_epilogue(const TsDevProg &P, const TsParams &S, const TsLaunch &L, cudaStream_t stream,
                               bool pdl) {
    return ts_launch_pdl(tsk::epilogue_kernel, dim3((unsigned)scalar_grid(L.n_env)), dim3(128), 0, stream, pdl,
                         P, S, L);
}
#endif
