/*
 * ts_oracle.c -- CPU restatement of the reference's native kernels.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path may link or call
 * this file; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg use it, and only as the checker.
 *
 * What is restated (reference = /root/reference/pkg, tissuesim 0.1.0):
 *   tso_run_substeps      <- backends/_kernels.pyx:260-352 (_lane_substeps),
 *                            ts_lane_predict 63-87, ts_lane_clear 89-100,
 *                            ts_lane_edges 102-139, grasp 283-298,
 *                            attachments 300-349, ts_lane_tets 141-211,
 *                            ts_lane_apply 213-244, damping 592
 *   tso_detect_contacts   <- backends/_kernels.pyx:797-947
 *                            (_cap_sd 732, _cap_sd_grad 750, _simplex3 778)
 *   tso_resolve_contacts  <- collision.py:55-73 (numpy semantics, see b2 note)
 *
 * Arithmetic contract: fp64, IEEE, compiled with -ffp-contract=off (as the
 * reference is, pkg/setup.py:20), and every expression keeps the reference's
 * association so the results are bitwise identical to the compiled backend.
 * The reference's env-minor "lane" layout only vectorises identical per-lane
 * arithmetic across environments, so a per-environment loop reproduces it.
 *
 * Cython's min()/max() on C doubles compile to (b < a ? b : a) and
 * (b > a ? b : a); cy_min/cy_max reproduce that (it only matters for -0.0).
 *
 * Parity pin: tests/test_oracle.py checks this file bitwise against the
 * reference built by oracle/build_ref.sh and against tests/golden/.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

#define TSO_EPS_LEN 1e-12
#define TSO_EPS_GRAD 1e-18

static inline double cy_min(double a, double b) { return (b < a) ? b : a; }
static inline double cy_max(double a, double b) { return (b > a) ? b : a; }

/* ---------------------------------------------------------------------- */
/* solver substeps                                                          */
/* ---------------------------------------------------------------------- */

typedef struct {
    int n_vert;
    const double *w;
    int n_edge; const int32_t *edges; const double *rest_len; double ks;
    int n_tet; const int32_t *tets; const double *rest_vol; double kv;
    int n_att; const int32_t *att_vertex; const int32_t *att_faces;
    const uint8_t *att_is_face; const double *att_anchor;
    const double *att_rest; const double *att_k;
    double gx, gy, gz, h, damp;
    int substeps;
} tso_solver;

/* accumulate a correction into vertex i of one environment */
static inline void acc_add(double *acc, int i, double cx, double cy, double cz) {
    acc[3 * i] += cx;
    acc[3 * i + 1] += cy;
    acc[3 * i + 2] += cz;
}

static void substeps_one_env(const tso_solver *S, double *x, double *v,
                             int64_t grasp_vertex, const double *drag,
                             double *acc, double *cnt) {
    const int nv = S->n_vert;
    for (int s = 0; s < S->substeps; ++s) {
        /* predict: kick + drift, pinned vertices get zero velocity */
        for (int i = 0; i < nv; ++i) {
            double *xi = x + 3 * i, *vi = v + 3 * i;
            if (S->w[i] > 0.0) {
                vi[0] += S->h * S->gx; xi[0] += S->h * vi[0];
                vi[1] += S->h * S->gy; xi[1] += S->h * vi[1];
                vi[2] += S->h * S->gz; xi[2] += S->h * vi[2];
            } else {
                vi[0] = 0.0; vi[1] = 0.0; vi[2] = 0.0;
            }
        }
        memset(acc, 0, sizeof(double) * 3 * (size_t)nv);
        memset(cnt, 0, sizeof(double) * (size_t)nv);

        /* distance constraints, index order */
        for (int e = 0; e < S->n_edge; ++e) {
            const int a = S->edges[2 * e], b = S->edges[2 * e + 1];
            const double wa = S->w[a], wb = S->w[b];
            const double wsum = wa + wb;
            if (wsum <= 0.0) continue;
            const double dx = x[3 * a] - x[3 * b];
            const double dy = x[3 * a + 1] - x[3 * b + 1];
            const double dz = x[3 * a + 2] - x[3 * b + 2];
            const double dist = sqrt(dx * dx + dy * dy + dz * dz);
            const double m = 0.5 + copysign(0.5, dist - TSO_EPS_LEN);
            const double scale = m * S->ks * (dist - S->rest_len[e]) / (dist * wsum + (1.0 - m));
            const double ca = -wa * scale;
            const double cb = wb * scale;
            acc_add(acc, a, ca * dx, ca * dy, ca * dz);
            acc_add(acc, b, cb * dx, cb * dy, cb * dz);
            cnt[a] += m;
            cnt[b] += m;
        }

        /* grasp: full pull of one vertex toward the kinematic drag point */
        if (grasp_vertex >= 0) {
            const int64_t g = grasp_vertex;
            const double dx = drag[0] - x[3 * g];
            const double dy = drag[1] - x[3 * g + 1];
            const double dz = drag[2] - x[3 * g + 2];
            const double dist = sqrt(dx * dx + dy * dy + dz * dz);
            if (!(dist <= TSO_EPS_LEN)) {
                acc[3 * g] += dx; acc[3 * g + 1] += dy; acc[3 * g + 2] += dz;
                cnt[g] += 1.0;
            }
        }

        /* attachments: vertex vs face centroid or static anchor */
        for (int t = 0; t < S->n_att; ++t) {
            const int vtx = S->att_vertex[t];
            const int f0 = S->att_faces[3 * t], f1 = S->att_faces[3 * t + 1], f2 = S->att_faces[3 * t + 2];
            const int is_face = S->att_is_face[t] != 0;
            const double wv = S->w[vtx];
            const double wc = is_face ? (S->w[f0] + S->w[f1] + S->w[f2]) / 3.0 : 0.0;
            const double wsum = wv + wc;
            if (wsum <= 0.0) continue;
            double cx, cy, cz;
            if (is_face) {
                cx = (x[3 * f0] + x[3 * f1] + x[3 * f2]) / 3.0;
                cy = (x[3 * f0 + 1] + x[3 * f1 + 1] + x[3 * f2 + 1]) / 3.0;
                cz = (x[3 * f0 + 2] + x[3 * f1 + 2] + x[3 * f2 + 2]) / 3.0;
            } else {
                cx = S->att_anchor[3 * t]; cy = S->att_anchor[3 * t + 1]; cz = S->att_anchor[3 * t + 2];
            }
            const double dx = x[3 * vtx] - cx;
            const double dy = x[3 * vtx + 1] - cy;
            const double dz = x[3 * vtx + 2] - cz;
            const double dist = sqrt(dx * dx + dy * dy + dz * dz);
            const double m = dist > TSO_EPS_LEN ? 1.0 : 0.0;
            const double scale = m * S->att_k[t] * (dist - S->att_rest[t]) / (dist * wsum + (1.0 - m));
            const double ca = -wv * scale;
            acc_add(acc, vtx, ca * dx, ca * dy, ca * dz);
            cnt[vtx] += m;
            if (is_face) {
                const double cb = wc * scale / 3.0;
                acc_add(acc, f0, cb * dx, cb * dy, cb * dz);
                acc_add(acc, f1, cb * dx, cb * dy, cb * dz);
                acc_add(acc, f2, cb * dx, cb * dy, cb * dz);
                cnt[f0] += m; cnt[f1] += m; cnt[f2] += m;
            }
        }

        /* volume constraints, index order; analytic gradients */
        for (int t = 0; t < S->n_tet; ++t) {
            const int ia = S->tets[4 * t], ib = S->tets[4 * t + 1];
            const int ic = S->tets[4 * t + 2], id = S->tets[4 * t + 3];
            const double *pa = x + 3 * ia, *pb = x + 3 * ib, *pc = x + 3 * ic, *pd = x + 3 * id;
            const double bax = pb[0] - pa[0], bay = pb[1] - pa[1], baz = pb[2] - pa[2];
            const double cax = pc[0] - pa[0], cay = pc[1] - pa[1], caz = pc[2] - pa[2];
            const double dax = pd[0] - pa[0], day = pd[1] - pa[1], daz = pd[2] - pa[2];
            /* grad_b = (c-a)x(d-a)/6, grad_c = (d-a)x(b-a)/6, grad_d = (b-a)x(c-a)/6 */
            const double gbx = (cay * daz - caz * day) / 6.0;
            const double gby = (caz * dax - cax * daz) / 6.0;
            const double gbz = (cax * day - cay * dax) / 6.0;
            const double gcx = (day * baz - daz * bay) / 6.0;
            const double gcy = (daz * bax - dax * baz) / 6.0;
            const double gcz = (dax * bay - day * bax) / 6.0;
            const double gdx = (bay * caz - baz * cay) / 6.0;
            const double gdy = (baz * cax - bax * caz) / 6.0;
            const double gdz = (bax * cay - bay * cax) / 6.0;
            const double gax = -(gbx + gcx + gdx);
            const double gay = -(gby + gcy + gdy);
            const double gaz = -(gbz + gcz + gdz);
            const double cval = (gdx * dax + gdy * day + gdz * daz) - S->rest_vol[t];
            const double denom = gax * gax + gay * gay + gaz * gaz
                               + gbx * gbx + gby * gby + gbz * gbz
                               + gcx * gcx + gcy * gcy + gcz * gcz
                               + gdx * gdx + gdy * gdy + gdz * gdz;
            const double m = 0.5 + copysign(0.5, denom - TSO_EPS_GRAD);
            const double sc = -m * S->kv * cval / (denom + (1.0 - m));
            acc_add(acc, ia, sc * gax, sc * gay, sc * gaz);
            acc_add(acc, ib, sc * gbx, sc * gby, sc * gbz);
            acc_add(acc, ic, sc * gcx, sc * gcy, sc * gcz);
            acc_add(acc, id, sc * gdx, sc * gdy, sc * gdz);
            cnt[ia] += m; cnt[ib] += m; cnt[ic] += m; cnt[id] += m;
        }

        /* average, commit, delta-velocity update, damping */
        for (int i = 0; i < nv; ++i) {
            double *xi = x + 3 * i, *vi = v + 3 * i;
            if (S->w[i] > 0.0) {
                const double n = cnt[i];
                const double m = 0.5 + copysign(0.5, n - 0.5);
                const double inv = m / (n + (1.0 - m));
                const double d0 = acc[3 * i] * inv;
                const double d1 = acc[3 * i + 1] * inv;
                const double d2 = acc[3 * i + 2] * inv;
                xi[0] += d0; vi[0] += d0 / S->h;
                xi[1] += d1; vi[1] += d1 / S->h;
                xi[2] += d2; vi[2] += d2 / S->h;
            }
            if (S->damp != 1.0) {
                vi[0] *= S->damp; vi[1] *= S->damp; vi[2] *= S->damp;
            }
        }
    }
}

/* Same argument set as the reference plugin entry run_substeps
 * (_kernels.pyx:577-585) minus the python-only scratch/threads/mode;
 * x, v are (n_env, n_vert, 3) C-contiguous and updated in place.
 * acc/cnt are caller scratch of n_vert*3 and n_vert doubles. */
void tso_run_substeps(int n_env, int n_vert, double *x, double *v, const double *w,
                      int n_edge, const int32_t *edges, const double *rest_len, double ks,
                      int n_tet, const int32_t *tets, const double *rest_vol, double kv,
                      int n_att, const int32_t *att_vertex, const int32_t *att_faces,
                      const uint8_t *att_is_face, const double *att_anchor,
                      const double *att_rest, const double *att_k,
                      const int64_t *grasp_vertex, const double *drag_points,
                      const double *g, double h, int substeps, double damping,
                      double *acc, double *cnt) {
    tso_solver S;
    S.n_vert = n_vert; S.w = w;
    S.n_edge = n_edge; S.edges = edges; S.rest_len = rest_len; S.ks = ks;
    S.n_tet = n_tet; S.tets = tets; S.rest_vol = rest_vol; S.kv = kv;
    S.n_att = n_att; S.att_vertex = att_vertex; S.att_faces = att_faces;
    S.att_is_face = att_is_face; S.att_anchor = att_anchor; S.att_rest = att_rest; S.att_k = att_k;
    S.gx = g[0]; S.gy = g[1]; S.gz = g[2]; S.h = h; S.substeps = substeps;
    /* damping factor, _kernels.pyx:592: 1 when damping == 0, else max(0, 1 - damping*h) */
    S.damp = (damping == 0.0) ? 1.0 : cy_max(0.0, 1.0 - damping * h);
    if (n_env <= 0 || n_vert <= 0) return;
    for (int e = 0; e < n_env; ++e) {
        substeps_one_env(&S, x + (size_t)e * n_vert * 3, v + (size_t)e * n_vert * 3,
                         grasp_vertex[e], drag_points + 3 * e, acc, cnt);
    }
}

/* ---------------------------------------------------------------------- */
/* capsule SDF contact detection                                           */
/* ---------------------------------------------------------------------- */

typedef struct { double p0[3], seg[3], dd, radius, fb[3]; } tso_capsule;

static double cap_sd(const tso_capsule *c, double px, double py, double pz) {
    double t = ((px - c->p0[0]) * c->seg[0] + (py - c->p0[1]) * c->seg[1]
                + (pz - c->p0[2]) * c->seg[2]) / c->dd;
    if (t < 0.0) t = 0.0;
    else if (t > 1.0) t = 1.0;
    const double dx = px - (c->p0[0] + t * c->seg[0]);
    const double dy = py - (c->p0[1] + t * c->seg[1]);
    const double dz = pz - (c->p0[2] + t * c->seg[2]);
    return sqrt(dx * dx + dy * dy + dz * dz) - c->radius;
}

static double cap_sd_grad(const tso_capsule *c, double px, double py, double pz, double *grad) {
    double t = ((px - c->p0[0]) * c->seg[0] + (py - c->p0[1]) * c->seg[1]
                + (pz - c->p0[2]) * c->seg[2]) / c->dd;
    if (t < 0.0) t = 0.0;
    else if (t > 1.0) t = 1.0;
    const double dx = px - (c->p0[0] + t * c->seg[0]);
    const double dy = py - (c->p0[1] + t * c->seg[1]);
    const double dz = pz - (c->p0[2] + t * c->seg[2]);
    const double norm = sqrt(dx * dx + dy * dy + dz * dz);
    if (norm > TSO_EPS_LEN) {
        grad[0] = dx / norm; grad[1] = dy / norm; grad[2] = dz / norm;
    } else {
        grad[0] = c->fb[0]; grad[1] = c->fb[1]; grad[2] = c->fb[2];
    }
    return norm - c->radius;
}

/* Euclidean projection onto the 2-simplex, sorted-threshold form (_kernels.pyx:778-794) */
static void simplex3(double *b) {
    double u0 = b[0], u1 = b[1], u2 = b[2], tmp, theta;
    if (u0 < u1) { tmp = u0; u0 = u1; u1 = tmp; }
    if (u1 < u2) { tmp = u1; u1 = u2; u2 = tmp; }
    if (u0 < u1) { tmp = u0; u0 = u1; u1 = tmp; }
    if (u2 - (u0 + u1 + u2 - 1.0) / 3.0 > 0.0) theta = (u0 + u1 + u2 - 1.0) / 3.0;
    else if (u1 - (u0 + u1 - 1.0) / 2.0 > 0.0) theta = (u0 + u1 - 1.0) / 2.0;
    else theta = u0 - 1.0;
    b[0] = cy_max(b[0] - theta, 0.0);
    b[1] = cy_max(b[1] - theta, 0.0);
    b[2] = cy_max(b[2] - theta, 0.0);
}

static void bary_point(const double *b, const double *pa, const double *pb, const double *pc, double *out) {
    out[0] = b[0] * pa[0] + b[1] * pb[0] + b[2] * pc[0];
    out[1] = b[0] * pa[1] + b[1] * pb[1] + b[2] * pc[1];
    out[2] = b[0] * pa[2] + b[1] * pb[2] + b[2] * pc[2];
}

/* Returns the number of contact rows written (capsule-major, face-minor).
 * Output arrays must hold n_face*n_cap rows. */
int tso_detect_contacts(const double *pos, int n_face, const int32_t *faces,
                        int n_cap, const double *caps, int iters,
                        int32_t *out_face, int32_t *out_cap, double *out_depth,
                        double *out_dir, double *out_bary) {
    int count = 0;
    if (n_face == 0 || n_cap == 0) return 0;
    for (int ci = 0; ci < n_cap; ++ci) {
        const double *row = caps + 7 * ci;
        tso_capsule C;
        double lo[3], hi[3];
        for (int k = 0; k < 3; ++k) { C.p0[k] = row[k]; C.seg[k] = row[3 + k] - row[k]; }
        C.radius = row[6];
        C.dd = C.seg[0] * C.seg[0] + C.seg[1] * C.seg[1] + C.seg[2] * C.seg[2];
        if (C.dd <= 0.0) C.dd = 1.0;
        /* axis-perpendicular fallback: seg x ex, or seg x ey when seg is along ex */
        C.fb[0] = 0.0; C.fb[1] = C.seg[2]; C.fb[2] = -C.seg[1];
        double fn = C.fb[0] * C.fb[0] + C.fb[1] * C.fb[1] + C.fb[2] * C.fb[2];
        if (fn < 1e-20) {
            C.fb[0] = -C.seg[2]; C.fb[1] = 0.0; C.fb[2] = C.seg[0];
            fn = C.fb[0] * C.fb[0] + C.fb[1] * C.fb[1] + C.fb[2] * C.fb[2];
        }
        fn = sqrt(fn);
        if (fn > 0.0) { C.fb[0] /= fn; C.fb[1] /= fn; C.fb[2] /= fn; }
        for (int k = 0; k < 3; ++k) {
            lo[k] = cy_min(row[k], row[3 + k]) - C.radius;
            hi[k] = cy_max(row[k], row[3 + k]) + C.radius;
        }

        for (int f = 0; f < n_face; ++f) {
            const double *pa = pos + 3 * faces[3 * f];
            const double *pb = pos + 3 * faces[3 * f + 1];
            const double *pc = pos + 3 * faces[3 * f + 2];
            int skip = 0;
            for (int k = 0; k < 3; ++k) {
                const double tlo = cy_min(cy_min(pa[k], pb[k]), pc[k]);
                const double thi = cy_max(cy_max(pa[k], pb[k]), pc[k]);
                if (thi < lo[k] || tlo > hi[k]) { skip = 1; break; }
            }
            if (skip) continue;

            const double s0 = cap_sd(&C, pa[0], pa[1], pa[2]);
            const double s1 = cap_sd(&C, pb[0], pb[1], pb[2]);
            const double s2 = cap_sd(&C, pc[0], pc[1], pc[2]);
            int vbest = 0;
            double best_sd = s0;
            if (s1 < best_sd) { vbest = 1; best_sd = s1; }
            if (s2 < best_sd) { vbest = 2; best_sd = s2; }

            double bary[3] = {vbest == 0 ? 1.0 : 0.0, vbest == 1 ? 1.0 : 0.0, vbest == 2 ? 1.0 : 0.0};
            double pt[3], grad[3], gb[3];
            double step = 0.5;
            for (int it = 0; it < iters; ++it) {
                bary_point(bary, pa, pb, pc, pt);
                cap_sd_grad(&C, pt[0], pt[1], pt[2], grad);
                gb[0] = grad[0] * pa[0] + grad[1] * pa[1] + grad[2] * pa[2];
                gb[1] = grad[0] * pb[0] + grad[1] * pb[1] + grad[2] * pb[2];
                gb[2] = grad[0] * pc[0] + grad[1] * pc[1] + grad[2] * pc[2];
                const double mean_g = (gb[0] + gb[1] + gb[2]) / 3.0;
                gb[0] -= mean_g; gb[1] -= mean_g; gb[2] -= mean_g;
                const double mag = cy_max(cy_max(fabs(gb[0]), fabs(gb[1])), fabs(gb[2]));
                bary[0] -= step * gb[0] / (mag + 1e-30);
                bary[1] -= step * gb[1] / (mag + 1e-30);
                bary[2] -= step * gb[2] / (mag + 1e-30);
                simplex3(bary);
                step *= 0.7;
            }
            bary_point(bary, pa, pb, pc, pt);
            double sd = cap_sd_grad(&C, pt[0], pt[1], pt[2], grad);
            if (sd > best_sd) {
                bary[0] = vbest == 0 ? 1.0 : 0.0;
                bary[1] = vbest == 1 ? 1.0 : 0.0;
                bary[2] = vbest == 2 ? 1.0 : 0.0;
                bary_point(bary, pa, pb, pc, pt);
                sd = cap_sd_grad(&C, pt[0], pt[1], pt[2], grad);
            }
            if (sd < 0.0) {
                out_face[count] = f;
                out_cap[count] = ci;
                out_depth[count] = -sd;
                for (int k = 0; k < 3; ++k) {
                    out_dir[3 * count + k] = grad[k];
                    out_bary[3 * count + k] = bary[k];
                }
                ++count;
            }
        }
    }
    return count;
}

/* Sequential push-out in emission order (collision.py:55-73).
 * b2 follows numpy's `b @ b` for a length-3 float64 vector, which on the
 * reference hosts dispatches to OpenBLAS ddot and evaluates as the fused
 * chain fma(b2, b2, fma(b1, b1, b0*b0)) (pinned by tests/test_oracle.py). */
void tso_resolve_contacts(double *pos, const double *w, const int32_t *faces,
                          int n_contact, const int32_t *face_idx, const double *depth,
                          const double *dir, const double *bary, double k_c) {
    for (int k = 0; k < n_contact; ++k) {
        const int32_t *verts = faces + 3 * face_idx[k];
        const double *b = bary + 3 * k;
        const double b2 = fma(b[2], b[2], fma(b[1], b[1], b[0] * b[0]));
        if (b2 <= 0.0) continue;
        const double s = k_c * depth[k] / b2;
        const double push[3] = {s * dir[3 * k], s * dir[3 * k + 1], s * dir[3 * k + 2]};
        for (int j = 0; j < 3; ++j) {
            if (w[verts[j]] > 0.0) {
                double *p = pos + 3 * verts[j];
                p[0] += b[j] * push[0];
                p[1] += b[j] * push[1];
                p[2] += b[j] * push[2];
            }
        }
    }
}
