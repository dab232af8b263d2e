/* ORACLE — test infrastructure only (tests/, __graft_entry__.smoke(), bench.py's CPU legs).
 *
 * Plain-C restatement of the reference's broadphase:
 *   broadphase_pairs   contactsim/geometry/broadphase.py:25-68: sorted (id_a, id_b) tuples of
 *                      the pairs whose margin-inflated boxes overlap. Up to
 *                      SWEEP_THRESHOLD (64) bodies all three axes are tested both ways
 *                      (:47-52); above it sweep-and-prune along x (:55-68) tests, for k
 *                      before idx in the stable lo.x order, hi_k.x >= lo_idx.x and y/z
 *                      both ways. The two agree on valid boxes and differ on inverted
 *                      ones (lo.x > hi.x); both are reproduced.
 *   world AABB         dynamics/body.py:77-83 (mesh AABB corners through
 *                      Transform.from_pose(...).apply, math3d.py:45-53,164-169; the
 *                      (8,3) @ (3,3).T product is OpenBLAS dgemm: G3 per element)
 * pinned against tests/golden/broadphase.npz (made by tests/golden/make_broadphase_golden.py). */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

static void bp_quat(const double *q, double *R) {
    const double w = q[0], x = q[1], y = q[2], z = q[3];
    R[0] = 1.0 - 2.0 * (y * y + z * z); R[1] = 2.0 * (x * y - w * z); R[2] = 2.0 * (x * z + w * y);
    R[3] = 2.0 * (x * y + w * z); R[4] = 1.0 - 2.0 * (x * x + z * z); R[5] = 2.0 * (y * z - w * x);
    R[6] = 2.0 * (x * z - w * y); R[7] = 2.0 * (y * z + w * x); R[8] = 1.0 - 2.0 * (x * x + y * y);
}

/* numpy min/max reductions: NaN propagates */
static double bp_min(double a, double b) { return (isnan(a) || a < b) ? a : b; }
static double bp_max(double a, double b) { return (isnan(a) || a > b) ? a : b; }

void og_world_aabb(int64_t n, const double *mesh_lo, const double *mesh_hi, const double *pose7, double *lo,
                   double *hi) {
    for (int64_t i = 0; i < n; ++i) {
        double R[9];
        bp_quat(pose7 + 7 * i + 3, R);
        const double *t = pose7 + 7 * i, *ml = mesh_lo + 3 * i, *mh = mesh_hi + 3 * i;
        for (int c = 0; c < 8; ++c) {
            const double p[3] = {(c & 4) ? mh[0] : ml[0], (c & 2) ? mh[1] : ml[1], (c & 1) ? mh[2] : ml[2]};
            for (int j = 0; j < 3; ++j) {
                const double w = fma(p[2], R[3 * j + 2], fma(p[1], R[3 * j + 1], p[0] * R[3 * j])) + t[j];
                lo[3 * i + j] = c ? bp_min(lo[3 * i + j], w) : w;
                hi[3 * i + j] = c ? bp_max(hi[3 * i + j], w) : w;
            }
        }
    }
}

static const int64_t *bp_ids;
static int bp_cmp(const void *a, const void *b) {
    const int64_t x = bp_ids[*(const int64_t *)a], y = bp_ids[*(const int64_t *)b];
    return x < y ? -1 : x > y;
}
static const double *bp_lox;
static int bp_cmp_x(const void *a, const void *b) {  /* stable argsort of lo.x */
    const int64_t i = *(const int64_t *)a, j = *(const int64_t *)b;
    const double x = bp_lox[3 * i], y = bp_lox[3 * j];
    if (x < y) return -1;
    if (x > y) return 1;
    return i < j ? -1 : i > j;
}

/* One scene of n bodies; pairs out (cap 2 * n(n-1)/2), returns the pair count or -1 on a
 * non-finite box (the reference raises ValueError). ids must be unique. */
int64_t og_broadphase(int64_t n, const double *lo_in, const double *hi_in, const int64_t *ids, double margin,
                      int64_t *pairs) {
    if (n < 2) return 0;
    double *lo = malloc(sizeof(double) * 3 * n), *hi = malloc(sizeof(double) * 3 * n);
    int64_t *ord = malloc(sizeof(int64_t) * n), *xr = malloc(sizeof(int64_t) * n), *xo = malloc(sizeof(int64_t) * n);
    int bad = 0;
    for (int64_t i = 0; i < 3 * n; ++i) {
        lo[i] = lo_in[i] - margin;
        hi[i] = hi_in[i] + margin;
        bad |= !isfinite(lo[i]) || !isfinite(hi[i]);
    }
    int64_t np_ = -1;
    if (!bad) {
        for (int64_t i = 0; i < n; ++i) ord[i] = xo[i] = i;
        bp_ids = ids;
        qsort(ord, (size_t)n, sizeof(int64_t), bp_cmp);
        bp_lox = lo;
        qsort(xo, (size_t)n, sizeof(int64_t), bp_cmp_x);
        for (int64_t r = 0; r < n; ++r) xr[xo[r]] = r; /* rank in the sweep order */
        const int sweep = n > 64;
        np_ = 0;
        for (int64_t p = 0; p < n; ++p)
            for (int64_t q = p + 1; q < n; ++q) {
                const int64_t i = ord[p], j = ord[q];
                int ov = 1;
                if (sweep) {
                    const int64_t k0 = xr[i] < xr[j] ? i : j, k1 = xr[i] < xr[j] ? j : i; /* k0 swept first */
                    ov = hi[3 * k0] >= lo[3 * k1];
                    for (int k = 1; k < 3; ++k) ov &= lo[3 * k1 + k] <= hi[3 * k0 + k] && lo[3 * k0 + k] <= hi[3 * k1 + k];
                } else {
                    for (int k = 0; k < 3; ++k) ov &= lo[3 * i + k] <= hi[3 * j + k] && lo[3 * j + k] <= hi[3 * i + k];
                }
                if (ov) { pairs[2 * np_] = ids[i]; pairs[2 * np_ + 1] = ids[j]; ++np_; }
            }
    }
    free(lo); free(hi); free(ord); free(xr); free(xo);
    return np_;
}
