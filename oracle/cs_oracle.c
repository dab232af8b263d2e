/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, single-file CPU restatement of the reference's contact hot path
 * (contactsim, /root/reference/pkg/src/contactsim). Only tests/, the smoke()
 * entry and bench.py's cpu_baseline / --impl reference leg may load it, and
 * only as the CHECKER or the timed CPU baseline. The product path
 * (paper_2205_03532_b200/) never links or calls it.
 *
 * Parity is pinned: tests/test_oracle.py checks this file bit-for-bit against
 * golden vectors produced by running the reference itself
 * (tests/golden/make_golden.py).
 *
 * Arithmetic contract (compile with -ffp-contract=off):
 *  - numba kernels (sdf/_kernels.py, contacts/_kernels.py) are compiled by
 *    numba/LLVM without fast-math: IEEE double, no FMA contraction, IEEE div/sqrt.
 *  - numpy `@` / np.dot route through OpenBLAS (SkylakeX kernels in the build
 *    container). Measured there, the 3-term dot products round as
 *      gemm / ddot(n=3) / F-contiguous gemv : G3 = fma(a2,b2, fma(a1,b1, a0*b0))
 *      C-contiguous (m>=2, 3) @ (3,) gemv   : V3 = fma(a2,b2, fma(a0,b0, a1*b1))
 *    and the length-n ddot / pairwise sums as restated in og_ddot*, og_pairwise.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define G3(a0, a1, a2, b0, b1, b2) fma((a2), (b2), fma((a1), (b1), (a0) * (b0)))
#define V3(a0, a1, a2, b0, b1, b2) fma((a2), (b2), fma((a0), (b0), (a1) * (b1)))

typedef struct {
    const float *v;
    int64_t nx, ny, nz;
    double ox, oy, oz, voxel;
} og_grid;

/* ------------------------------------------------------------------ SDF sampling */

/* sdf/_kernels.py:253-292 */
static inline double og_trilinear(const og_grid *g, double gx, double gy, double gz) {
    int64_t x0 = (int64_t)floor(gx), y0 = (int64_t)floor(gy), z0 = (int64_t)floor(gz);
    if (x0 < 0) x0 = 0;
    if (x0 > g->nx - 2) x0 = g->nx - 2;
    if (y0 < 0) y0 = 0;
    if (y0 > g->ny - 2) y0 = g->ny - 2;
    if (z0 < 0) z0 = 0;
    if (z0 > g->nz - 2) z0 = g->nz - 2;
    double fx = gx - (double)x0, fy = gy - (double)y0, fz = gz - (double)z0;
    int64_t base = x0 + g->nx * (y0 + g->ny * z0);
    int64_t sy = g->nx, sz = g->nx * g->ny;
    const float *v = g->v;
    double c000 = v[base], c100 = v[base + 1], c010 = v[base + sy], c110 = v[base + 1 + sy];
    double c001 = v[base + sz], c101 = v[base + 1 + sz], c011 = v[base + sy + sz], c111 = v[base + 1 + sy + sz];
    double c00 = c000 * (1.0 - fx) + c100 * fx;
    double c10 = c010 * (1.0 - fx) + c110 * fx;
    double c01 = c001 * (1.0 - fx) + c101 * fx;
    double c11 = c011 * (1.0 - fx) + c111 * fx;
    double c0 = c00 * (1.0 - fy) + c10 * fy;
    double c1 = c01 * (1.0 - fy) + c11 * fy;
    return c0 * (1.0 - fz) + c1 * fz;
}

static inline double og_minf(double a, double b) { return b < a ? b : a; }
static inline double og_maxf(double a, double b) { return b > a ? b : a; }

/* sdf/_kernels.py:295-309 */
double og_sample(const og_grid *g, double px, double py, double pz) {
    double gx = (px - g->ox) / g->voxel;
    double gy = (py - g->oy) / g->voxel;
    double gz = (pz - g->oz) / g->voxel;
    double cx = og_minf(og_maxf(gx, 0.0), (double)g->nx - 1.0);
    double cy = og_minf(og_maxf(gy, 0.0), (double)g->ny - 1.0);
    double cz = og_minf(og_maxf(gz, 0.0), (double)g->nz - 1.0);
    double dx = gx - cx, dy = gy - cy, dz = gz - cz;
    double outside = sqrt(dx * dx + dy * dy + dz * dz) * g->voxel;
    return og_trilinear(g, cx, cy, cz) + outside;
}

/* sdf/_kernels.py:312-327 */
void og_gradient(const og_grid *g, double px, double py, double pz, double *gx, double *gy, double *gz) {
    double h = g->voxel, h2 = 2.0 * g->voxel;
    *gx = (og_sample(g, px + h, py, pz) - og_sample(g, px - h, py, pz)) / h2;
    *gy = (og_sample(g, px, py + h, pz) - og_sample(g, px, py - h, pz)) / h2;
    *gz = (og_sample(g, px, py, pz + h) - og_sample(g, px, py, pz - h)) / h2;
}

/* sdf/_kernels.py:20-61 (Ericson) */
static void og_closest(double ax, double ay, double az, double bx, double by, double bz, double cx, double cy,
                       double cz, double px, double py, double pz, double *qx, double *qy, double *qz) {
    double abx = bx - ax, aby = by - ay, abz = bz - az;
    double acx = cx - ax, acy = cy - ay, acz = cz - az;
    double apx = px - ax, apy = py - ay, apz = pz - az;
    double d1 = abx * apx + aby * apy + abz * apz;
    double d2 = acx * apx + acy * apy + acz * apz;
    if (d1 <= 0.0 && d2 <= 0.0) { *qx = ax; *qy = ay; *qz = az; return; }
    double bpx = px - bx, bpy = py - by, bpz = pz - bz;
    double d3 = abx * bpx + aby * bpy + abz * bpz;
    double d4 = acx * bpx + acy * bpy + acz * bpz;
    if (d3 >= 0.0 && d4 <= d3) { *qx = bx; *qy = by; *qz = bz; return; }
    double vc = d1 * d4 - d3 * d2;
    if (vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0) {
        double v = d1 / (d1 - d3);
        *qx = ax + v * abx; *qy = ay + v * aby; *qz = az + v * abz; return;
    }
    double cpx = px - cx, cpy = py - cy, cpz = pz - cz;
    double d5 = abx * cpx + aby * cpy + abz * cpz;
    double d6 = acx * cpx + acy * cpy + acz * cpz;
    if (d6 >= 0.0 && d5 <= d6) { *qx = cx; *qy = cy; *qz = cz; return; }
    double vb = d5 * d2 - d1 * d6;
    if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) {
        double w = d2 / (d2 - d6);
        *qx = ax + w * acx; *qy = ay + w * acy; *qz = az + w * acz; return;
    }
    double va = d3 * d6 - d5 * d4;
    if (va <= 0.0 && (d4 - d3) >= 0.0 && (d5 - d6) >= 0.0) {
        double w = (d4 - d3) / ((d4 - d3) + (d5 - d6));
        *qx = bx + w * (cx - bx); *qy = by + w * (cy - by); *qz = bz + w * (cz - bz); return;
    }
    double denom = 1.0 / (va + vb + vc);
    double v = vb * denom, w = vc * denom;
    *qx = ax + abx * v + acx * w;
    *qy = ay + aby * v + acy * w;
    *qz = az + abz * v + acz * w;
}

/* contacts/_kernels.py:11-87 — one face. Returns 0 if pruned (outputs untouched). */
static int og_face(const og_grid *g, const double *t, double cd, int max_iters, double tol, double *op, double *ophi,
                   double *og, uint8_t *ofound) {
    double ax = t[0], ay = t[1], az = t[2], bx = t[3], by = t[4], bz = t[5], cx = t[6], cy = t[7], cz = t[8];
    double phi_a = og_sample(g, ax, ay, az);
    double phi_b = og_sample(g, bx, by, bz);
    double phi_c = og_sample(g, cx, cy, cz);
    double e0 = sqrt((bx - ax) * (bx - ax) + (by - ay) * (by - ay) + (bz - az) * (bz - az));
    double e1 = sqrt((cx - bx) * (cx - bx) + (cy - by) * (cy - by) + (cz - bz) * (cz - bz));
    double e2 = sqrt((ax - cx) * (ax - cx) + (ay - cy) * (ay - cy) + (az - cz) * (az - cz));
    double diam = og_maxf(e0, og_maxf(e1, e2));
    double phi_min = og_minf(phi_a, og_minf(phi_b, phi_c));
    if (phi_min - diam > cd) { *ofound = 0; return 0; }
    double gxc = (ax + bx + cx) / 3.0, gyc = (ay + by + cy) / 3.0, gzc = (az + bz + cz) / 3.0;
    double phi_cen = og_sample(g, gxc, gyc, gzc);
    double px = gxc, py = gyc, pz = gzc, phi = phi_cen;
    if (phi_a < phi) { px = ax; py = ay; pz = az; phi = phi_a; }
    if (phi_b < phi) { px = bx; py = by; pz = bz; phi = phi_b; }
    if (phi_c < phi) { px = cx; py = cy; pz = cz; phi = phi_c; }
    double alpha = g->voxel;
    for (int it = 0; it < max_iters; ++it) {
        double grx, gry, grz;
        og_gradient(g, px, py, pz, &grx, &gry, &grz);
        double gnorm = sqrt(grx * grx + gry * gry + grz * grz);
        if (gnorm < 1e-12) break;
        grx /= gnorm; gry /= gnorm; grz /= gnorm;
        double moved = 0.0;
        for (int bt = 0; bt < 4; ++bt) {
            double qx, qy, qz;
            og_closest(ax, ay, az, bx, by, bz, cx, cy, cz, px - alpha * grx, py - alpha * gry, pz - alpha * grz,
                       &qx, &qy, &qz);
            double phi_new = og_sample(g, qx, qy, qz);
            if (phi_new < phi) {
                moved = sqrt((qx - px) * (qx - px) + (qy - py) * (qy - py) + (qz - pz) * (qz - pz));
                px = qx; py = qy; pz = qz; phi = phi_new;
                alpha = og_minf(alpha * 1.5, 4.0 * g->voxel);
                break;
            }
            alpha *= 0.5;
        }
        if (moved < tol) break;
    }
    op[0] = px; op[1] = py; op[2] = pz;
    *ophi = phi;
    double grx, gry, grz;
    og_gradient(g, px, py, pz, &grx, &gry, &grz);
    og[0] = grx; og[1] = gry; og[2] = grz;
    *ofound = (phi <= cd) ? 1 : 0;
    return 1;
}

/* numba face_contacts drop-in: same argument list (contacts/_kernels.py:12-17). */
void og_face_contacts(const float *values, int64_t nx, int64_t ny, int64_t nz, double ox, double oy, double oz,
                      double voxel, const double *tri_verts, int64_t m, double cd, int max_iters, double tol,
                      double *out_point, double *out_phi, double *out_grad, uint8_t *out_found) {
    og_grid g = {values, nx, ny, nz, ox, oy, oz, voxel};
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t t = 0; t < m; ++t)
        og_face(&g, tri_verts + 9 * t, cd, max_iters, tol, out_point + 3 * t, out_phi + t, out_grad + 3 * t,
                out_found + t);
}

void og_sample_batch(const float *values, int64_t nx, int64_t ny, int64_t nz, double ox, double oy, double oz,
                     double voxel, const double *pts, int64_t n, double *out) {
    og_grid g = {values, nx, ny, nz, ox, oy, oz, voxel};
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) out[i] = og_sample(&g, pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]);
}

void og_gradient_batch(const float *values, int64_t nx, int64_t ny, int64_t nz, double ox, double oy, double oz,
                       double voxel, const double *pts, int64_t n, double *out) {
    og_grid g = {values, nx, ny, nz, ox, oy, oz, voxel};
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i)
        og_gradient(&g, pts[3 * i], pts[3 * i + 1], pts[3 * i + 2], out + 3 * i, out + 3 * i + 1, out + 3 * i + 2);
}

/* ------------------------------------------------------------------ poses (math3d.py) */

/* math3d.py:45-53 */
void og_quat_to_matrix(const double *q, double *R) {
    double w = q[0], x = q[1], y = q[2], z = q[3];
    R[0] = 1.0 - 2.0 * (y * y + z * z);
    R[1] = 2.0 * (x * y - w * z);
    R[2] = 2.0 * (x * z + w * y);
    R[3] = 2.0 * (x * y + w * z);
    R[4] = 1.0 - 2.0 * (x * x + z * z);
    R[5] = 2.0 * (y * z - w * x);
    R[6] = 2.0 * (x * z - w * y);
    R[7] = 2.0 * (y * z + w * x);
    R[8] = 1.0 - 2.0 * (x * x + y * y);
}

/* to_grid = sdf_pose.inverse().compose(mesh_pose) (generation.py:70; math3d.py:174-179).
 * pose7 = (px, py, pz, qw, qx, qy, qz) as Transform.from_pose consumes it. */
void og_to_grid(const double *sdf7, const double *mesh7, double *R, double *t) {
    double Rs[9], Rm[9];
    og_quat_to_matrix(sdf7 + 3, Rs);
    og_quat_to_matrix(mesh7 + 3, Rm);
    const double *ts = sdf7, *tm = mesh7;
    double ti[3];
    for (int i = 0; i < 3; ++i) /* (-rt) @ ts, rt F-contiguous -> gemv_n pattern G3 */
        ti[i] = G3(-Rs[0 * 3 + i], -Rs[1 * 3 + i], -Rs[2 * 3 + i], ts[0], ts[1], ts[2]);
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) /* rt @ Rm: gemm */
            R[i * 3 + j] = G3(Rs[0 * 3 + i], Rs[1 * 3 + i], Rs[2 * 3 + i], Rm[0 * 3 + j], Rm[1 * 3 + j], Rm[2 * 3 + j]);
    for (int i = 0; i < 3; ++i) /* rt @ tm + ti */
        t[i] = G3(Rs[0 * 3 + i], Rs[1 * 3 + i], Rs[2 * 3 + i], tm[0], tm[1], tm[2]) + ti[i];
}

/* points @ R.T + t for n points (Transform.apply, math3d.py:168-169) */
static void og_apply(const double *R, const double *t, const double *p, int64_t n, double *out) {
    for (int64_t i = 0; i < n; ++i) {
        const double *a = p + 3 * i;
        for (int j = 0; j < 3; ++j) {
            const double *r = R + 3 * j;
            double d = (n >= 2) ? G3(a[0], a[1], a[2], r[0], r[1], r[2]) : V3(a[0], a[1], a[2], r[0], r[1], r[2]);
            out[3 * i + j] = d + t[j];
        }
    }
}

/* vectors @ R.T (normals to world) */
static void og_rotate(const double *R, const double *p, int64_t n, double *out) {
    for (int64_t i = 0; i < n; ++i) {
        const double *a = p + 3 * i;
        for (int j = 0; j < 3; ++j) {
            const double *r = R + 3 * j;
            out[3 * i + j] = (n >= 2) ? G3(a[0], a[1], a[2], r[0], r[1], r[2]) : V3(a[0], a[1], a[2], r[0], r[1], r[2]);
        }
    }
}

void og_tri_verts(const double *sdf7, const double *mesh7, const double *verts, int64_t nv, const int32_t *tris,
                  int64_t nt, double *out) {
    double R[9], t[3];
    og_to_grid(sdf7, mesh7, R, t);
    double *vg = (double *)malloc(sizeof(double) * 3 * (size_t)nv);
    og_apply(R, t, verts, nv, vg);
    for (int64_t f = 0; f < nt; ++f)
        for (int c = 0; c < 3; ++c)
            for (int k = 0; k < 3; ++k) out[9 * f + 3 * c + k] = vg[3 * (int64_t)tris[3 * f + c] + k];
    free(vg);
}

/* generate_contacts (generation.py:54-114) for one pair. Outputs sized nt.
 * Returns the number of candidates, or -1 on non-finite pose, -2 on cd < 0. */
int64_t og_generate_contacts(const float *values, int64_t nx, int64_t ny, int64_t nz, double ox, double oy, double oz,
                             double voxel, const double *aabb_lo, const double *aabb_hi, const double *verts,
                             int64_t nv, const int32_t *tris, int64_t nt, const double *sdf7, const double *mesh7,
                             double cd, double *points, double *normals, double *depths, int64_t *faces,
                             int threads_inner) {
    if (cd < 0.0) return -2;
    double Rs[9], Rm[9];
    og_quat_to_matrix(sdf7 + 3, Rs);
    og_quat_to_matrix(mesh7 + 3, Rm);
    for (int i = 0; i < 9; ++i)
        if (!isfinite(Rs[i]) || !isfinite(Rm[i])) return -1;
    for (int i = 0; i < 3; ++i)
        if (!isfinite(sdf7[i]) || !isfinite(mesh7[i])) return -1;
    double *tv = (double *)malloc(sizeof(double) * 9 * (size_t)(nt > 0 ? nt : 1));
    og_tri_verts(sdf7, mesh7, verts, nv, tris, nt, tv);
    double margin = cd + 2.0 * voxel;
    double hi_m[3], lo_m[3];
    for (int k = 0; k < 3; ++k) { hi_m[k] = aabb_hi[k] + margin; lo_m[k] = aabb_lo[k] - margin; }
    int64_t *ids = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nt > 0 ? nt : 1));
    int64_t m = 0;
    for (int64_t f = 0; f < nt; ++f) {
        const double *t = tv + 9 * f;
        int near = 1;
        for (int k = 0; k < 3; ++k) {
            double lo = og_minf(og_minf(t[k], t[3 + k]), t[6 + k]);
            double hi = og_maxf(og_maxf(t[k], t[3 + k]), t[6 + k]);
            if (!(lo <= hi_m[k] && hi >= lo_m[k])) near = 0;
        }
        if (near) ids[m++] = f;
    }
    og_grid g = {values, nx, ny, nz, ox, oy, oz, voxel};
    double *op = (double *)malloc(sizeof(double) * 3 * (size_t)(m > 0 ? m : 1));
    double *ophi = (double *)malloc(sizeof(double) * (size_t)(m > 0 ? m : 1));
    double *ogr = (double *)malloc(sizeof(double) * 3 * (size_t)(m > 0 ? m : 1));
    uint8_t *ofd = (uint8_t *)calloc((size_t)(m > 0 ? m : 1), 1);
    double tol = 0.1 * voxel;
#pragma omp parallel for schedule(dynamic, 256) if (threads_inner)
    for (int64_t i = 0; i < m; ++i)
        og_face(&g, tv + 9 * ids[i], cd, 12, tol, op + 3 * i, ophi + i, ogr + 3 * i, ofd + i);
    int64_t c = 0;
    for (int64_t i = 0; i < m; ++i) {
        if (!ofd[i]) continue;
        memcpy(points + 3 * c, op + 3 * i, 3 * sizeof(double));
        double gx = ogr[3 * i], gy = ogr[3 * i + 1], gz = ogr[3 * i + 2];
        double nrm = sqrt(gx * gx + gy * gy + gz * gz); /* add.reduce over 3: ((x2+y2)+z2) */
        if (nrm < 1e-12) { gx = 0.0; gy = 0.0; gz = 1.0; nrm = 1.0; }
        normals[3 * c] = gx / nrm; normals[3 * c + 1] = gy / nrm; normals[3 * c + 2] = gz / nrm;
        depths[c] = -ophi[i];
        faces[c] = ids[i];
        ++c;
    }
    /* world frame: n @ Rs.T ; Rs p + ts */
    double *tmp = (double *)malloc(sizeof(double) * 3 * (size_t)(c > 0 ? c : 1));
    og_rotate(Rs, normals, c, tmp);
    memcpy(normals, tmp, sizeof(double) * 3 * (size_t)c);
    og_apply(Rs, sdf7, points, c, tmp);
    memcpy(points, tmp, sizeof(double) * 3 * (size_t)c);
    free(tmp); free(op); free(ophi); free(ogr); free(ofd); free(ids); free(tv);
    return c;
}

/* ------------------------------------------------------------------ reduction helpers */

/* numpy add.reduce over a contiguous 1-D float64 array: 0 + pairwise (umath loops). */
static double og_pw(const double *a, int64_t n) {
    if (n < 8) {
        double r = 0.0;
        for (int64_t i = 0; i < n; ++i) r += a[i];
        return r;
    } else if (n <= 128) {
        double r[8];
        for (int j = 0; j < 8; ++j) r[j] = a[j];
        int64_t i;
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; ++j) r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; ++i) res += a[i];
        return res;
    } else {
        int64_t n2 = n / 2;
        n2 -= n2 % 8;
        return og_pw(a, n2) + og_pw(a + n2, n - n2);
    }
}
double og_sum(const double *a, int64_t n) { return 0.0 + og_pw(a, n); }

/* OpenBLAS ddot, strided x (inc_x != 1) path: used for np.dot(poly[:,0], roll(poly[:,1]))
 * x stride 2 (a column of an (H,2) array), y contiguous. */
static double og_ddot_x2(int64_t n, const double *x, const double *y) {
    double t1 = 0.0, t2 = 0.0;
    int64_t i = 0, n1 = n & -4;
    while (i < n1) {
        double m3 = y[i + 2] * x[2 * (i + 2)];
        double m4 = y[i + 3] * x[2 * (i + 3)];
        t1 = t1 + fma(y[i], x[2 * i], m3);
        t2 = t2 + fma(y[i + 1], x[2 * (i + 1)], m4);
        i += 4;
    }
    while (i < n) { t1 = fma(y[i], x[2 * i], t1); ++i; }
    return t1 + t2;
}

/* math3d.py:143-152 */
static void og_tangent_basis(const double *n, double *t1, double *t2) {
    double a[3];
    if (fabs(n[0]) < 0.57735) { a[0] = 1.0; a[1] = 0.0; a[2] = 0.0; }
    else { a[0] = 0.0; a[1] = 1.0; a[2] = 0.0; }
    double d = G3(a[0], a[1], a[2], n[0], n[1], n[2]);
    for (int k = 0; k < 3; ++k) a[k] = a[k] - n[k] * d;
    double nn = sqrt(G3(a[0], a[1], a[2], a[0], a[1], a[2]));
    for (int k = 0; k < 3; ++k) t1[k] = a[k] / nn;
    t2[0] = n[1] * t1[2] - n[2] * t1[1];
    t2[1] = n[2] * t1[0] - n[0] * t1[2];
    t2[2] = n[0] * t1[1] - n[1] * t1[0];
}

typedef struct { double u, v; int64_t pos; } og_uv;
static int og_nan_last_cmp(double x, double y) {
    const int xn = isnan(x), yn = isnan(y);
    if (xn || yn) return xn - yn;
    return (x < y) ? -1 : (x > y);
}

static int og_uv_cmp(const void *pa, const void *pb) {
    /* numpy's sort order per key: NaN after every number, NaNs equal to each other
     * (npy_sort's LT: a < b || (b != b && a == a)); lexsort is stable, so ties keep
     * their positions */
    const og_uv *a = (const og_uv *)pa, *b = (const og_uv *)pb;
    const int c = og_nan_last_cmp(a->u, b->u);
    if (c) return c;
    const int d = og_nan_last_cmp(a->v, b->v);
    if (d) return d;
    return (a->pos < b->pos) ? -1 : (a->pos > b->pos);
}

/* _project_2d + _monotone_hull (reduction.py:202-224). pts indexed via idx[0..n).
 * Writes hull positions (0..n-1 into idx) to hull; returns hull length. uv out (n x 2). */
static int64_t og_hull(const double *points, const int64_t *idx, int64_t n, const double *normal, int64_t *hull,
                       double *uvout, og_uv *scratch, int64_t *stack) {
    double t1[3], t2[3];
    og_tangent_basis(normal, t1, t2);
    for (int64_t i = 0; i < n; ++i) {
        const double *p = points + 3 * idx[i];
        double u = (n >= 2) ? V3(p[0], p[1], p[2], t1[0], t1[1], t1[2]) : G3(p[0], p[1], p[2], t1[0], t1[1], t1[2]);
        double v = (n >= 2) ? V3(p[0], p[1], p[2], t2[0], t2[1], t2[2]) : G3(p[0], p[1], p[2], t2[0], t2[1], t2[2]);
        uvout[2 * i] = u; uvout[2 * i + 1] = v;
        scratch[i].u = u; scratch[i].v = v; scratch[i].pos = i;
    }
    qsort(scratch, (size_t)n, sizeof(og_uv), og_uv_cmp);
#define CROSS(o, a, b) ((uvout[2 * (a)] - uvout[2 * (o)]) * (uvout[2 * (b) + 1] - uvout[2 * (o) + 1]) - \
                        (uvout[2 * (a) + 1] - uvout[2 * (o) + 1]) * (uvout[2 * (b)] - uvout[2 * (o)]))
    int64_t h = 0, top = 0;
    for (int64_t k = 0; k < n; ++k) {
        int64_t i = scratch[k].pos;
        while (top >= 2 && CROSS(stack[top - 2], stack[top - 1], i) <= 0) --top;
        stack[top++] = i;
    }
    for (int64_t k = 0; k + 1 < top; ++k) hull[h++] = stack[k];
    top = 0;
    for (int64_t k = n - 1; k >= 0; --k) {
        int64_t i = scratch[k].pos;
        while (top >= 2 && CROSS(stack[top - 2], stack[top - 1], i) <= 0) --top;
        stack[top++] = i;
    }
    for (int64_t k = 0; k + 1 < top; ++k) hull[h++] = stack[k];
#undef CROSS
    return h;
}

typedef struct {
    double *uv;
    og_uv *sc;
    int64_t *stack, *hull, *idx;
    double *x, *y;
} og_ws;

/* _hull_area (reduction.py:227-236) over points[idx[0..n)] */
static double og_hull_area(const double *points, const int64_t *idx, int64_t n, const double *normal, og_ws *w) {
    if (n < 3) return 0.0;
    int64_t h = og_hull(points, idx, n, normal, w->hull, w->uv, w->sc, w->stack);
    if (h < 3) return 0.0;
    /* poly = uv[hull] (H,2) C-contiguous; x = poly[:,0] (stride 2), y = poly[:,1] */
    double *poly = w->x, *ry = w->y;
    for (int64_t k = 0; k < h; ++k) { poly[2 * k] = w->uv[2 * w->hull[k]]; poly[2 * k + 1] = w->uv[2 * w->hull[k] + 1]; }
    for (int64_t k = 0; k < h; ++k) ry[k] = poly[2 * ((k + 1) % h) + 1]; /* roll(y, -1) */
    double d1 = og_ddot_x2(h, poly, ry);
    for (int64_t k = 0; k < h; ++k) ry[k] = poly[2 * ((k + 1) % h)];     /* roll(x, -1) */
    double d2 = og_ddot_x2(h, poly + 1, ry);
    return 0.5 * fabs(d1 - d2);
}

/* numpy argmax semantics: first max; NaN wins (first NaN). */
static int64_t og_argmax(const double *a, const int64_t *idx, int64_t n) {
    int64_t best = 0;
    double bv = a[idx ? idx[0] : 0];
    if (isnan(bv)) return 0;
    for (int64_t i = 1; i < n; ++i) {
        double v = a[idx ? idx[i] : i];
        if (isnan(v)) return i;
        if (v > bv) { bv = v; best = i; }
    }
    return best;
}

typedef struct {
    int max_patches, per_patch_cap;
    double cone, min_depth;
    int has_min_depth, batch_size;
} og_params;

typedef struct {
    const double *points, *normals, *depths;
    int64_t n;
} og_cands;

typedef struct {
    double normal[3];
    double max_depth;
} og_builder;

#define MERGE_COS 0.9961946980917455 /* float(np.cos(np.radians(5.0))) */

static double og_builder_area(const og_cands *c, const int32_t *label, int slot, const double *normal,
                              int64_t *tmpidx, og_ws *w) {
    int64_t m = 0;
    for (int64_t i = 0; i < c->n; ++i)
        if (label[i] == slot) tmpidx[m++] = i;
    return og_hull_area(c->points, tmpidx, m, normal, w);
}

/* reduce_contacts (reduction.py:45-75) with _assign_to_existing / _add_patch / _fold_members.
 * Membership is kept as a label per candidate (-1 = none); order inside a patch never
 * matters downstream (finalize sorts; hull area depends only on the point set). */
static int og_reduce_labels(const og_cands *c, const og_params *p, int32_t *label, og_builder *B, og_ws *w,
                            int64_t *order, int64_t *unassigned, double *cosb, int64_t *tmpidx) {
    const double *N = c->normals, *D = c->depths;
    int64_t n_order = 0;
    for (int64_t i = 0; i < c->n; ++i) {
        label[i] = -1;
        if (!p->has_min_depth || D[i] >= p->min_depth) order[n_order++] = i;
    }
    int P = 0;
    const int32_t PENDING = -2;
    for (int64_t start = 0; start < n_order; start += p->batch_size) {
        int64_t bsz = n_order - start < p->batch_size ? n_order - start : p->batch_size;
        const int64_t *batch = order + start;
        int64_t nu = 0;
        /* _assign_to_existing: cos = normals[batch] @ reps.T ; argmax ; >= cone */
        if (P == 0) {
            for (int64_t k = 0; k < bsz; ++k) unassigned[nu++] = batch[k];
        } else {
            int gemm = (bsz >= 2 && P >= 2) || (bsz == 1 && P == 1);
            for (int64_t k = 0; k < bsz; ++k) {
                const double *a = N + 3 * batch[k];
                for (int q = 0; q < P; ++q) {
                    const double *b = B[q].normal;
                    cosb[q] = gemm ? G3(a[0], a[1], a[2], b[0], b[1], b[2]) : V3(a[0], a[1], a[2], b[0], b[1], b[2]);
                }
                int best = (int)og_argmax(cosb, NULL, P);
                double bc = cosb[best];
                if (bc >= p->cone) {
                    label[batch[k]] = best;
                    if (D[batch[k]] > B[best].max_depth) B[best].max_depth = D[batch[k]];
                } else {
                    unassigned[nu++] = batch[k];
                }
            }
        }
        while (nu > 0) {
            int64_t dp = og_argmax(D, unassigned, nu);
            int64_t seed = unassigned[dp];
            double sn[3] = {N[3 * seed], N[3 * seed + 1], N[3 * seed + 2]};
            double pmax = -INFINITY;
            int64_t keep = 0;
            for (int64_t k = 0; k < nu; ++k) {
                int64_t i = unassigned[k];
                const double *a = N + 3 * i;
                double cs = (nu >= 2) ? V3(a[0], a[1], a[2], sn[0], sn[1], sn[2]) : G3(a[0], a[1], a[2], sn[0], sn[1], sn[2]);
                if (cs >= p->cone || k == dp) {
                    label[i] = PENDING;
                    if (D[i] > pmax) pmax = D[i];
                } else {
                    unassigned[keep++] = i;
                }
            }
            nu = keep;
            /* _add_patch (reduction.py:91-126) */
            int best = -1, similar = 0;
            double bc = 0.0;
            if (P > 0) {
                for (int q = 0; q < P; ++q) {
                    const double *b = B[q].normal;
                    cosb[q] = (P >= 2) ? V3(b[0], b[1], b[2], sn[0], sn[1], sn[2]) : G3(b[0], b[1], b[2], sn[0], sn[1], sn[2]);
                }
                best = (int)og_argmax(cosb, NULL, P);
                bc = cosb[best];
                similar = bc >= p->cone;
            }
            if (similar && (bc >= MERGE_COS || P >= p->max_patches)) {
                if (pmax > B[best].max_depth) { B[best].normal[0] = sn[0]; B[best].normal[1] = sn[1]; B[best].normal[2] = sn[2]; }
                for (int64_t i = 0; i < c->n; ++i)
                    if (label[i] == PENDING) {
                        label[i] = best;
                        if (D[i] > B[best].max_depth) B[best].max_depth = D[i];
                    }
                continue;
            }
            if (P < p->max_patches) {
                B[P].normal[0] = sn[0]; B[P].normal[1] = sn[1]; B[P].normal[2] = sn[2];
                B[P].max_depth = pmax;
                for (int64_t i = 0; i < c->n; ++i)
                    if (label[i] == PENDING) label[i] = P;
                ++P;
                continue;
            }
            /* eviction */
            double gmax = B[0].max_depth;
            for (int q = 1; q < P; ++q) gmax = (B[q].max_depth > gmax || isnan(gmax)) ? B[q].max_depth : gmax;
            int victim = -1;
            int vprot = 0;
            double vdepth = 0, varea = 0;
            for (int q = 0; q < P; ++q) {
                int prot = B[q].max_depth >= gmax;
                double area = og_builder_area(c, label, q, B[q].normal, tmpidx, w);
                /* score = (0 if protected else 1, -max_depth, -area, -q); max wins */
                int better;
                if (victim < 0) better = 1;
                else {
                    int s0 = prot ? 0 : 1, v0 = vprot ? 0 : 1;
                    if (s0 != v0) better = s0 > v0;
                    else if (-B[q].max_depth != -vdepth) better = -B[q].max_depth > -vdepth;
                    else if (-area != -varea) better = -area > -varea;
                    else better = -q > -victim;
                }
                if (better) { victim = q; vprot = prot; vdepth = B[q].max_depth; varea = area; }
            }
            double parea = og_builder_area(c, label, PENDING, sn, tmpidx, w);
            int replace = (pmax > vdepth) || (pmax == vdepth && parea > varea);
            if (replace) {
                og_builder vb = B[victim];
                B[victim].normal[0] = sn[0]; B[victim].normal[1] = sn[1]; B[victim].normal[2] = sn[2];
                B[victim].max_depth = pmax;
                /* fold victim's members into nearest other (skip victim) */
                for (int q = 0; q < P; ++q) {
                    const double *b = B[q].normal;
                    cosb[q] = (P >= 2) ? V3(b[0], b[1], b[2], vb.normal[0], vb.normal[1], vb.normal[2])
                                       : G3(b[0], b[1], b[2], vb.normal[0], vb.normal[1], vb.normal[2]);
                }
                cosb[victim] = -INFINITY;
                int tgt = (int)og_argmax(cosb, NULL, P);
                for (int64_t i = 0; i < c->n; ++i) {
                    if (label[i] == victim) {
                        label[i] = tgt == victim ? -3 : tgt; /* -3: re-resolved below */
                        if (tgt != victim && D[i] > B[tgt].max_depth) B[tgt].max_depth = D[i];
                    }
                }
                for (int64_t i = 0; i < c->n; ++i) {
                    if (label[i] == PENDING) label[i] = victim;
                    else if (label[i] == -3) { label[i] = victim; if (D[i] > B[victim].max_depth) B[victim].max_depth = D[i]; }
                }
            } else {
                for (int q = 0; q < P; ++q) {
                    const double *b = B[q].normal;
                    cosb[q] = (P >= 2) ? V3(b[0], b[1], b[2], sn[0], sn[1], sn[2]) : G3(b[0], b[1], b[2], sn[0], sn[1], sn[2]);
                }
                int tgt = (int)og_argmax(cosb, NULL, P);
                for (int64_t i = 0; i < c->n; ++i)
                    if (label[i] == PENDING) {
                        label[i] = tgt;
                        if (D[i] > B[tgt].max_depth) B[tgt].max_depth = D[i];
                    }
            }
        }
    }
    return P;
}

/* numpy stable argsort of -depths (NaN last). */
static _Thread_local const double *og_sort_depths; /* per thread: envs run in parallel (OpenMP) */
static int og_negdepth_cmp(const void *pa, const void *pb) {
    int64_t a = *(const int64_t *)pa, b = *(const int64_t *)pb;
    double x = -og_sort_depths[a], y = -og_sort_depths[b];
    int xn = isnan(x), yn = isnan(y);
    if (xn != yn) return xn ? 1 : -1;
    if (!xn) {
        if (x < y) return -1;
        if (x > y) return 1;
    }
    return (a < b) ? -1 : (a > b);
}

/* _select_kept (reduction.py:172-199) over member arrays (local positions). Returns count. */
static int og_select_kept(const double *pts, const double *deps, int64_t n, const double *normal, int cap,
                          int64_t *chosen, og_ws *w, int64_t *tmp) {
    if (n <= cap) {
        for (int64_t i = 0; i < n; ++i) chosen[i] = i;
        return (int)n;
    }
    int64_t deepest = og_argmax(deps, NULL, n);
    int64_t nt = 0;
    for (int64_t i = 0; i < n; ++i)
        if (deps[i] >= 0.0) tmp[nt++] = i;
    if (nt < 3) { nt = n; for (int64_t i = 0; i < n; ++i) tmp[i] = i; }
    int64_t h = og_hull(pts, tmp, nt, normal, w->hull, w->uv, w->sc, w->stack);
    int64_t nh = 0;
    for (int64_t k = 0; k < h; ++k) {
        int64_t m = tmp[w->hull[k]];
        if (m != deepest) w->idx[nh++] = m;
    }
    int nc = 0;
    chosen[nc++] = deepest;
    if (nh <= cap - 1) {
        for (int64_t k = 0; k < nh; ++k) chosen[nc++] = w->idx[k];
        if (nc < cap) {
            for (int64_t i = 0; i < n; ++i) tmp[i] = i;
            og_sort_depths = deps;
            qsort(tmp, (size_t)n, sizeof(int64_t), og_negdepth_cmp);
            for (int64_t k = 0; k < n && nc < cap; ++k) {
                int in = 0;
                for (int j = 0; j < nc; ++j) if (chosen[j] == tmp[k]) { in = 1; break; }
                if (!in) chosen[nc++] = tmp[k];
            }
        }
    } else {
        double step = (double)nh / (double)(cap - 1);
        for (int k = 0; k < cap - 1; ++k) {
            int64_t pk = (int64_t)((double)k * step + 0.0);
            chosen[nc++] = w->idx[pk];
        }
    }
    return nc < cap ? nc : cap;
}

/* reduce_contacts end to end. Output layout (capacity N = max_patches, K = per_patch_cap):
 *   rep[N*3], nkept[N], kept[N*K] (candidate indices), member_offsets[N+1], members[n],
 *   wsum[N], wp[N*3], wn[N*3], wt[N*3], area[N], maxd[N].  Returns number of patches. */
int og_reduce_contacts(int64_t n, const double *points, const double *normals, const double *depths,
                       int max_patches, int per_patch_cap, double cone, double min_depth, int has_min_depth,
                       int batch_size, double *rep, int64_t *nkept, int64_t *kept, int64_t *member_offsets,
                       int64_t *members, double *wsum, double *wp, double *wn, double *wt, double *area, double *maxd) {
    member_offsets[0] = 0;
    if (n == 0) return 0;
    og_params p = {max_patches, per_patch_cap, cone, min_depth, has_min_depth, batch_size};
    og_cands c = {points, normals, depths, n};
    size_t nn = (size_t)n + 4;
    int32_t *label = (int32_t *)malloc(sizeof(int32_t) * nn);
    og_builder *B = (og_builder *)malloc(sizeof(og_builder) * (size_t)(max_patches + 1));
    int64_t *order = (int64_t *)malloc(sizeof(int64_t) * nn);
    int64_t *un = (int64_t *)malloc(sizeof(int64_t) * nn);
    int64_t *tmpidx = (int64_t *)malloc(sizeof(int64_t) * nn);
    int64_t *tmp2 = (int64_t *)malloc(sizeof(int64_t) * nn);
    double *cosb = (double *)malloc(sizeof(double) * (size_t)(max_patches + 1));
    og_ws w;
    w.uv = (double *)malloc(sizeof(double) * 2 * nn);
    w.sc = (og_uv *)malloc(sizeof(og_uv) * nn);
    w.stack = (int64_t *)malloc(sizeof(int64_t) * 2 * nn);
    w.hull = (int64_t *)malloc(sizeof(int64_t) * 2 * nn);
    w.idx = (int64_t *)malloc(sizeof(int64_t) * 2 * nn);
    w.x = (double *)malloc(sizeof(double) * 4 * nn);  /* the hull polygon (u, v): up to 2n - 2 vertices (NaN keys never pop) */
    w.y = (double *)malloc(sizeof(double) * 2 * nn);
    double *mp = (double *)malloc(sizeof(double) * 3 * nn);
    double *mn = (double *)malloc(sizeof(double) * 3 * nn);
    double *md = (double *)malloc(sizeof(double) * nn);
    double *wv = (double *)malloc(sizeof(double) * nn);
    int64_t *chosen = (int64_t *)malloc(sizeof(int64_t) * (size_t)(per_patch_cap + 1));

    int P = og_reduce_labels(&c, &p, label, B, &w, order, un, cosb, tmpidx);

    /* _finalize each builder in slot order (reduction.py:146-169) */
    int64_t off = 0;
    for (int q = 0; q < P; ++q) {
        int64_t m = 0;
        for (int64_t i = 0; i < n; ++i)
            if (label[i] == q) members[off + m++] = i;
        for (int64_t k = 0; k < m; ++k) {
            int64_t i = members[off + k];
            memcpy(mp + 3 * k, points + 3 * i, 3 * sizeof(double));
            memcpy(mn + 3 * k, normals + 3 * i, 3 * sizeof(double));
            md[k] = depths[i];
        }
        int nk = og_select_kept(mp, md, m, B[q].normal, per_patch_cap, chosen, &w, tmp2);
        nkept[q] = nk;
        for (int k = 0; k < per_patch_cap; ++k) kept[(int64_t)q * per_patch_cap + k] = k < nk ? members[off + chosen[k]] : -1;
        rep[3 * q] = B[q].normal[0]; rep[3 * q + 1] = B[q].normal[1]; rep[3 * q + 2] = B[q].normal[2];
        for (int64_t k = 0; k < m; ++k) wv[k] = md[k] > 0.0 ? md[k] : (md[k] <= 0.0 ? 0.0 : md[k]); /* np.maximum */
        wsum[q] = og_sum(wv, m);
        double sp[3] = {0, 0, 0}, sn[3] = {0, 0, 0}, st[3] = {0, 0, 0};
        for (int64_t k = 0; k < m; ++k) {
            const double *pp = mp + 3 * k, *np_ = mn + 3 * k;
            double t0 = (pp[1] * np_[2] - pp[2] * np_[1]) * wv[k];
            double t1 = (pp[2] * np_[0] - pp[0] * np_[2]) * wv[k];
            double t2 = (pp[0] * np_[1] - pp[1] * np_[0]) * wv[k];
            double a0 = pp[0] * wv[k], a1 = pp[1] * wv[k], a2 = pp[2] * wv[k];
            double b0 = np_[0] * wv[k], b1 = np_[1] * wv[k], b2 = np_[2] * wv[k];
            if (k == 0) {
                sp[0] = a0; sp[1] = a1; sp[2] = a2; sn[0] = b0; sn[1] = b1; sn[2] = b2; st[0] = t0; st[1] = t1; st[2] = t2;
            } else {
                sp[0] += a0; sp[1] += a1; sp[2] += a2; sn[0] += b0; sn[1] += b1; sn[2] += b2; st[0] += t0; st[1] += t1; st[2] += t2;
            }
        }
        for (int k = 0; k < 3; ++k) { wp[3 * q + k] = sp[k]; wn[3 * q + k] = sn[k]; wt[3 * q + k] = st[k]; }
        for (int64_t k = 0; k < m; ++k) tmpidx[k] = k;
        area[q] = og_hull_area(mp, tmpidx, m, B[q].normal, &w);
        double mx = md[0];
        for (int64_t k = 1; k < m; ++k) { if (isnan(md[k]) || isnan(mx)) { mx = NAN; } else if (md[k] > mx) mx = md[k]; }
        maxd[q] = mx;
        off += m;
        member_offsets[q + 1] = off;
    }
    free(label); free(B); free(order); free(un); free(tmpidx); free(tmp2); free(cosb);
    free(w.uv); free(w.sc); free(w.stack); free(w.hull); free(w.idx); free(w.x); free(w.y);
    free(mp); free(mn); free(md); free(wv); free(chosen);
    return P;
}

/* Batched CPU path (the timed CPU baseline): per env generate + reduce, exactly as
 * Scene._collect_contacts calls them (dynamics/scene.py:206-226). OpenMP over envs. */
typedef struct {
    int64_t n_cand, n_patch, n_kept;
    double max_depth;
} og_env_stats;

void og_collide_batched(int64_t E, const float *values, int64_t nx, int64_t ny, int64_t nz, double ox, double oy,
                        double oz, double voxel, const double *aabb_lo, const double *aabb_hi, const double *verts,
                        int64_t nv, const int32_t *tris, int64_t nt, const double *sdf7, const double *mesh7,
                        const double *cd, int max_patches, int per_patch_cap, double cone, int batch_size,
                        og_env_stats *stats) {
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t e = 0; e < E; ++e) {
        size_t cap = (size_t)(nt > 0 ? nt : 1);
        double *P = (double *)malloc(sizeof(double) * 3 * cap), *Nn = (double *)malloc(sizeof(double) * 3 * cap);
        double *D = (double *)malloc(sizeof(double) * cap);
        int64_t *F = (int64_t *)malloc(sizeof(int64_t) * cap);
        int64_t c = og_generate_contacts(values, nx, ny, nz, ox, oy, oz, voxel, aabb_lo, aabb_hi, verts, nv, tris, nt,
                                         sdf7 + 7 * e, mesh7 + 7 * e, cd[e], P, Nn, D, F, 0);
        int64_t np_ = 0, nk = 0;
        double mx = 0.0;
        if (c > 0) {
            size_t N = (size_t)max_patches, K = (size_t)per_patch_cap;
            double *rep = malloc(sizeof(double) * 3 * N), *ws = malloc(sizeof(double) * N), *wp = malloc(sizeof(double) * 3 * N);
            double *wn = malloc(sizeof(double) * 3 * N), *wt = malloc(sizeof(double) * 3 * N), *ar = malloc(sizeof(double) * N);
            double *md = malloc(sizeof(double) * N);
            int64_t *nkp = malloc(sizeof(int64_t) * N), *kept = malloc(sizeof(int64_t) * N * K);
            int64_t *moff = malloc(sizeof(int64_t) * (N + 1)), *mem = malloc(sizeof(int64_t) * (size_t)c);
            np_ = og_reduce_contacts(c, P, Nn, D, max_patches, per_patch_cap, cone, -cd[e], 1, batch_size, rep, nkp,
                                     kept, moff, mem, ws, wp, wn, wt, ar, md);
            for (int64_t q = 0; q < np_; ++q) {
                nk += nkp[q];
                for (int64_t k = 0; k < nkp[q]; ++k) {
                    double d = D[kept[q * K + k]];
                    if (d > mx) mx = d;
                }
            }
            free(rep); free(ws); free(wp); free(wn); free(wt); free(ar); free(md); free(nkp); free(kept); free(moff); free(mem);
        }
        stats[e].n_cand = c < 0 ? 0 : c;
        stats[e].n_patch = np_;
        stats[e].n_kept = nk;
        stats[e].max_depth = mx;
        free(P); free(Nn); free(D); free(F);
    }
}

int og_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* Per-env digest of EVERY output of generate + reduce (test infrastructure: the GPU
 * suite compares the batched collide's outputs of all envs against it). The stream
 * of 64-bit words of an env, in order:
 *   n_cand; points[3c], normals[3c], depths[c] (double bits), faces[c];
 *   n_patch; per patch: rep[3], nkept, kept candidate indices[nkept], n_members,
 *   members[n_members], wsum, wp[3], wn[3], wt[3], area, max_depth
 * and digest = sum_i (w_i ^ 0x9e3779b97f4a7c15) * (2 i + 1) mod 2^64 (tests/conftest.py:
 * env_digest computes the same from the GPU outputs). */
typedef struct {
    uint64_t h, i;
} og_dig;
static inline void og_dig_u(og_dig *d, uint64_t w) {
    d->h += (w ^ 0x9e3779b97f4a7c15ull) * (2 * d->i + 1);
    d->i++;
}
static inline void og_dig_d(og_dig *d, double x) {
    uint64_t w;
    memcpy(&w, &x, 8);
    og_dig_u(d, w);
}

void og_collide_digest(int64_t E, const float *values, int64_t nx, int64_t ny, int64_t nz, double ox, double oy,
                       double oz, double voxel, const double *aabb_lo, const double *aabb_hi, const double *verts,
                       int64_t nv, const int32_t *tris, int64_t nt, const double *sdf7, const double *mesh7,
                       const double *cd, int max_patches, int per_patch_cap, double cone, int batch_size,
                       uint64_t *digest) {
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t e = 0; e < E; ++e) {
        size_t cap = (size_t)(nt > 0 ? nt : 1);
        double *P = (double *)malloc(sizeof(double) * 3 * cap), *Nn = (double *)malloc(sizeof(double) * 3 * cap);
        double *D = (double *)malloc(sizeof(double) * cap);
        int64_t *F = (int64_t *)malloc(sizeof(int64_t) * cap);
        int64_t c = og_generate_contacts(values, nx, ny, nz, ox, oy, oz, voxel, aabb_lo, aabb_hi, verts, nv, tris, nt,
                                         sdf7 + 7 * e, mesh7 + 7 * e, cd[e], P, Nn, D, F, 0);
        if (c < 0) c = 0;
        og_dig d = {0, 0};
        og_dig_u(&d, (uint64_t)c);
        for (int64_t i = 0; i < 3 * c; ++i) og_dig_d(&d, P[i]);
        for (int64_t i = 0; i < 3 * c; ++i) og_dig_d(&d, Nn[i]);
        for (int64_t i = 0; i < c; ++i) og_dig_d(&d, D[i]);
        for (int64_t i = 0; i < c; ++i) og_dig_u(&d, (uint64_t)F[i]);
        int64_t np_ = 0;
        if (c > 0) {
            size_t N = (size_t)max_patches, K = (size_t)per_patch_cap;
            double *rep = malloc(sizeof(double) * 3 * N), *ws = malloc(sizeof(double) * N), *wp = malloc(sizeof(double) * 3 * N);
            double *wn = malloc(sizeof(double) * 3 * N), *wt = malloc(sizeof(double) * 3 * N), *ar = malloc(sizeof(double) * N);
            double *md = malloc(sizeof(double) * N);
            int64_t *nkp = malloc(sizeof(int64_t) * N), *kept = malloc(sizeof(int64_t) * N * K);
            int64_t *moff = malloc(sizeof(int64_t) * (N + 1)), *mem = malloc(sizeof(int64_t) * (size_t)c);
            np_ = og_reduce_contacts(c, P, Nn, D, max_patches, per_patch_cap, cone, -cd[e], 1, batch_size, rep, nkp,
                                     kept, moff, mem, ws, wp, wn, wt, ar, md);
            og_dig_u(&d, (uint64_t)np_);
            for (int64_t q = 0; q < np_; ++q) {
                for (int k = 0; k < 3; ++k) og_dig_d(&d, rep[3 * q + k]);
                og_dig_u(&d, (uint64_t)nkp[q]);
                for (int64_t k = 0; k < nkp[q]; ++k) og_dig_u(&d, (uint64_t)kept[q * K + k]);
                og_dig_u(&d, (uint64_t)(moff[q + 1] - moff[q]));
                for (int64_t k = moff[q]; k < moff[q + 1]; ++k) og_dig_u(&d, (uint64_t)mem[k]);
                og_dig_d(&d, ws[q]);
                for (int k = 0; k < 3; ++k) og_dig_d(&d, wp[3 * q + k]);
                for (int k = 0; k < 3; ++k) og_dig_d(&d, wn[3 * q + k]);
                for (int k = 0; k < 3; ++k) og_dig_d(&d, wt[3 * q + k]);
                og_dig_d(&d, ar[q]);
                og_dig_d(&d, md[q]);
            }
            free(rep); free(ws); free(wp); free(wn); free(wt); free(ar); free(md); free(nkp); free(kept); free(moff); free(mem);
        } else {
            og_dig_u(&d, 0);
        }
        digest[e] = d.h;
        free(P); free(Nn); free(D); free(F);
    }
}
