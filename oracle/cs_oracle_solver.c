/* ORACLE — test infrastructure only (tests/, __graft_entry__.smoke(), bench.py's CPU legs).
 *
 * Plain-C restatement of the reference's contact solver:
 *   ContactConstraints.build     contactsim/dynamics/solver.py:105-141 (+ _normal_velocity :166-171)
 *   gauss_seidel_sweeps          contactsim/dynamics/_kernels.py:54-115
 *   ContactConstraints.body_wrenches  solver.py:154-163
 * Compiled with -ffp-contract=off: numba's kernel has no FMA contraction. The numpy
 * products in build() go through OpenBLAS; their rounding is written out explicitly:
 *   3-term dots (ddot / np.linalg.norm):          fma chain from the first product (G3)
 *   (6,) @ (6,6) (cblas dgemv, OpenBLAS dgemv_n):  og_gemv6 below
 *   (6,) @ (6,) (ddot):                           fma chain from the first product
 * pinned bit for bit against the reference's own outputs (tests/golden/solver.npz,
 * made by tests/golden/make_solver_golden.py). */
#include <math.h>
#include <stdint.h>

static inline double G3s(double a0, double a1, double a2, double b0, double b1, double b2) {
    return fma(a2, b2, fma(a1, b1, a0 * b0));
}

/* math3d.py:143-152 */
static void sv_tangent_basis(const double *n, double *t1, double *t2) {
    double a[3];
    if (fabs(n[0]) < 0.57735) { a[0] = 1.0; a[1] = 0.0; a[2] = 0.0; }
    else { a[0] = 0.0; a[1] = 1.0; a[2] = 0.0; }
    double d = G3s(a[0], a[1], a[2], n[0], n[1], n[2]);
    for (int k = 0; k < 3; ++k) a[k] = a[k] - n[k] * d;
    double nn = sqrt(G3s(a[0], a[1], a[2], a[0], a[1], a[2]));
    for (int k = 0; k < 3; ++k) t1[k] = a[k] / nn;
    t2[0] = n[1] * t1[2] - n[2] * t1[1];
    t2[1] = n[2] * t1[0] - n[0] * t1[2];
    t2[2] = n[0] * t1[1] - n[1] * t1[0];
}

/* x @ W for x (6,), W (6,6) row-major: numpy hands it to cblas_dgemv, which runs
 * OpenBLAS's dgemv_n over the transposed view. Its 4-row vector block pairs the
 * products (1,0) and (5,4) and fuses the rest; the two leftover rows are a plain
 * fma chain (measured: tests/golden/make_solver_golden.py probes). */
static void og_gemv6(const double *x, const double *W, double *y) {
    for (int j = 0; j < 4; ++j) {
        double t = fma(x[0], W[0 * 6 + j], x[1] * W[1 * 6 + j]);
        t = fma(x[2], W[2 * 6 + j], t);
        t = fma(x[3], W[3 * 6 + j], t);
        double u = fma(x[4], W[4 * 6 + j], x[5] * W[5 * 6 + j]);
        y[j] = t + u;
    }
    for (int j = 4; j < 6; ++j) {
        double t = x[0] * W[j];
        for (int i = 1; i < 6; ++i) t = fma(x[i], W[i * 6 + j], t);
        y[j] = t;
    }
}

static double og_dot6(const double *a, const double *b) {
    double t = a[0] * b[0];
    for (int i = 1; i < 6; ++i) t = fma(a[i], b[i], t);
    return t;
}

/* ga @ W @ ga with ga = [d, r x d] (solver.py:128-131) */
static double og_quad(const double *d, const double *r, const double *W) {
    double g[6], v[6];
    g[0] = d[0]; g[1] = d[1]; g[2] = d[2];
    g[3] = r[1] * d[2] - r[2] * d[1];
    g[4] = r[2] * d[0] - r[0] * d[2];
    g[5] = r[0] * d[1] - r[1] * d[0];
    og_gemv6(g, W, v);
    return og_dot6(v, g);
}

/* solver.py:105-141 for one system: m rows in sweep order, nb bodies. */
void og_constraints_build(int64_t m, const int64_t *body_a, const int64_t *body_b, const double *point,
                          const double *normal, const double *depth, const double *restitution, const double *slop,
                          const double *ref, const double *w_mat, const double *vel, double h, double bias_factor,
                          double *ra, double *rb, double *tan1, double *tan2, double *kn, double *kt1, double *kt2,
                          double *bias_target, double *restitution_target) {
    for (int64_t c = 0; c < m; ++c) {
        const int64_t ia = body_a[c], ib = body_b[c];
        const double *p = point + 3 * c, *n = normal + 3 * c;
        double *a = ra + 3 * c, *b = rb + 3 * c, *t1 = tan1 + 3 * c, *t2 = tan2 + 3 * c;
        for (int k = 0; k < 3; ++k) {
            a[k] = p[k] - ref[3 * ia + k];
            b[k] = p[k] - ref[3 * ib + k];
        }
        sv_tangent_basis(n, t1, t2);
        const double *dirs[3] = {n, t1, t2};
        double *outs[3] = {kn + c, kt1 + c, kt2 + c};
        for (int q = 0; q < 3; ++q) {
            const double k = og_quad(dirs[q], a, w_mat + 36 * ia) + og_quad(dirs[q], b, w_mat + 36 * ib);
            *outs[q] = k > 1e-12 ? 1.0 / k : 0.0;
        }
        const double dep = depth[c], s = slop[c];
        double bt = 0.0;
        if (dep > s) bt = bias_factor * (dep - s) / h;
        else if (dep < 0.0) bt = dep / h;
        bias_target[c] = bt;
        /* _normal_velocity (solver.py:166-171) */
        const double *vb = vel + 6 * ib, *va = vel + 6 * ia;
        const double ub0 = vb[0] + (vb[4] * b[2] - vb[5] * b[1]);
        const double ub1 = vb[1] + (vb[5] * b[0] - vb[3] * b[2]);
        const double ub2 = vb[2] + (vb[3] * b[1] - vb[4] * b[0]);
        const double ua0 = va[0] + (va[4] * a[2] - va[5] * a[1]);
        const double ua1 = va[1] + (va[5] * a[0] - va[3] * a[2]);
        const double ua2 = va[2] + (va[3] * a[1] - va[4] * a[0]);
        const double vn0 = G3s(ub0 - ua0, ub1 - ua1, ub2 - ua2, n[0], n[1], n[2]);
        const double neg = -vn0;
        const double v_impact = (0.0 > neg) ? 0.0 : neg; /* Python max(-vn0, 0.0) */
        const double e = v_impact > 0.5 ? restitution[c] : 0.0;
        restitution_target[c] = e * v_impact;
    }
}

/* _kernels.py:16-37 */
static void og_apply_impulse(const double *w_mat, double *vel, double *imp, int64_t body, double jx, double jy,
                             double jz, double rx, double ry, double rz, double sign) {
    const double gx = jx * sign, gy = jy * sign, gz = jz * sign;
    const double tx = (ry * jz - rz * jy) * sign;
    const double ty = (rz * jx - rx * jz) * sign;
    const double tz = (rx * jy - ry * jx) * sign;
    const double *W = w_mat + 36 * body;
    for (int k = 0; k < 6; ++k)
        vel[6 * body + k] += W[6 * k] * gx + W[6 * k + 1] * gy + W[6 * k + 2] * gz + W[6 * k + 3] * tx +
                             W[6 * k + 4] * ty + W[6 * k + 5] * tz;
    imp[6 * body] += gx; imp[6 * body + 1] += gy; imp[6 * body + 2] += gz;
    imp[6 * body + 3] += tx; imp[6 * body + 4] += ty; imp[6 * body + 5] += tz;
}

/* _kernels.py:40-49 */
static double og_rel_vel(const double *vel, int64_t ia, int64_t ib, const double *ra, const double *rb, double dx,
                         double dy, double dz) {
    const double *vb = vel + 6 * ib, *va = vel + 6 * ia;
    const double ubx = vb[0] + vb[4] * rb[2] - vb[5] * rb[1];
    const double uby = vb[1] + vb[5] * rb[0] - vb[3] * rb[2];
    const double ubz = vb[2] + vb[3] * rb[1] - vb[4] * rb[0];
    const double uax = va[0] + va[4] * ra[2] - va[5] * ra[1];
    const double uay = va[1] + va[5] * ra[0] - va[3] * ra[2];
    const double uaz = va[2] + va[3] * ra[1] - va[4] * ra[0];
    return (ubx - uax) * dx + (uby - uay) * dy + (ubz - uaz) * dz;
}

/* _kernels.py:52-115 */
void og_gauss_seidel_sweeps(int64_t iters, const double *w_mat, double *vel, double *imp, int64_t m,
                            const int64_t *body_a, const int64_t *body_b, const double *ra, const double *rb,
                            const double *nrm, const double *tan1, const double *tan2, const double *kn,
                            const double *kt1, const double *kt2, const double *target_vn, const double *mu,
                            double *lam_n, double *lam_t1, double *lam_t2, int with_friction) {
    for (int64_t it = 0; it < iters; ++it) {
        for (int64_t c = 0; c < m; ++c) {
            const int64_t ia = body_a[c], ib = body_b[c];
            const double *a = ra + 3 * c, *b = rb + 3 * c;
            const double nx = nrm[3 * c], ny = nrm[3 * c + 1], nz = nrm[3 * c + 2];
            if (kn[c] > 0.0) {
                const double vn = og_rel_vel(vel, ia, ib, a, b, nx, ny, nz);
                double dl = kn[c] * (target_vn[c] - vn);
                double new_l = lam_n[c] + dl;
                if (new_l < 0.0) new_l = 0.0;
                dl = new_l - lam_n[c];
                lam_n[c] = new_l;
                if (dl != 0.0) {
                    og_apply_impulse(w_mat, vel, imp, ib, dl * nx, dl * ny, dl * nz, b[0], b[1], b[2], 1.0);
                    og_apply_impulse(w_mat, vel, imp, ia, dl * nx, dl * ny, dl * nz, a[0], a[1], a[2], -1.0);
                }
            }
            if (with_friction && mu[c] > 0.0 && lam_n[c] > 0.0) {
                const double t1x = tan1[3 * c], t1y = tan1[3 * c + 1], t1z = tan1[3 * c + 2];
                const double t2x = tan2[3 * c], t2y = tan2[3 * c + 1], t2z = tan2[3 * c + 2];
                double d1 = 0.0, d2 = 0.0;
                if (kt1[c] > 0.0) d1 = -kt1[c] * og_rel_vel(vel, ia, ib, a, b, t1x, t1y, t1z);
                if (kt2[c] > 0.0) d2 = -kt2[c] * og_rel_vel(vel, ia, ib, a, b, t2x, t2y, t2z);
                double new1 = lam_t1[c] + d1, new2 = lam_t2[c] + d2;
                const double limit = mu[c] * lam_n[c];
                const double mag = sqrt(new1 * new1 + new2 * new2);
                if (mag > limit) {
                    const double scale = limit / mag;
                    new1 *= scale;
                    new2 *= scale;
                }
                d1 = new1 - lam_t1[c];
                d2 = new2 - lam_t2[c];
                lam_t1[c] = new1;
                lam_t2[c] = new2;
                if (d1 != 0.0 || d2 != 0.0) {
                    const double jx = d1 * t1x + d2 * t2x, jy = d1 * t1y + d2 * t2y, jz = d1 * t1z + d2 * t2z;
                    og_apply_impulse(w_mat, vel, imp, ib, jx, jy, jz, b[0], b[1], b[2], 1.0);
                    og_apply_impulse(w_mat, vel, imp, ia, jx, jy, jz, a[0], a[1], a[2], -1.0);
                }
            }
        }
    }
}

/* solver.py:154-163: out (nb, 6), zero-initialised by the caller */
void og_body_wrenches(int64_t m, const int64_t *body_a, const int64_t *body_b, const double *ra, const double *rb,
                      const double *nrm, const double *tan1, const double *tan2, const double *lam_n,
                      const double *lam_vel, const double *lam_t1, const double *lam_t2, double h, double *out) {
    for (int64_t c = 0; c < m; ++c) {
        const double lam = lam_n[c] + lam_vel[c];
        double j[3];
        for (int k = 0; k < 3; ++k) j[k] = (lam * nrm[3 * c + k] + lam_t1[c] * tan1[3 * c + k]) + lam_t2[c] * tan2[3 * c + k];
        const double *a = ra + 3 * c, *b = rb + 3 * c;
        const double cb[3] = {b[1] * j[2] - b[2] * j[1], b[2] * j[0] - b[0] * j[2], b[0] * j[1] - b[1] * j[0]};
        const double ca[3] = {a[1] * j[2] - a[2] * j[1], a[2] * j[0] - a[0] * j[2], a[0] * j[1] - a[1] * j[0]};
        double *ob = out + 6 * body_b[c], *oa = out + 6 * body_a[c];
        for (int k = 0; k < 3; ++k) {
            ob[k] += j[k] / h;
            ob[3 + k] += cb[k] / h;
            oa[k] -= j[k] / h;
            oa[3 + k] -= ca[k] / h;
        }
    }
}
