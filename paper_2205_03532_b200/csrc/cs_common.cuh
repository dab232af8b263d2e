// Shared device code for the contact path. Compiled with -fmad=false: plain
// double arithmetic is never contracted, so every expression rounds exactly like
// the reference's numba kernels; the reference's BLAS dot products are
// reproduced with explicit fma (G3 / V3 below).
//
// The SDF sampler is written for the B200 pipes rather than transliterated: it
// produces the reference's bits (sdf/_kernels.py:253-327) but
//   * divides by the voxel size with a reciprocal + two FMA corrections and an
//     exact remainder check (IEEE division only when the check cannot prove
//     correct rounding), instead of the MUFU + Newton IEEE division;
//   * clamps and floors grid coordinates with integer operations on the bit
//     pattern (no F2I / I2F on the XU pipe); the results are exact;
//   * skips the outside-distance term for samples inside the grid, where the
//     reference adds sqrt(0) * voxel == +0.0;
//   * reuses the per-axis work of the centre point across the six
//     central-difference samples.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/contactsim_b200.h"

namespace cs {

// 3-term dot products as the reference's OpenBLAS computes them (measured):
//   gemm, ddot(n=3), gemv on an F-contiguous matrix:  G3
//   gemv on a C-contiguous (m >= 2, 3) matrix:         V3
__device__ __forceinline__ double G3(double a0, double a1, double a2, double b0, double b1, double b2) {
    return __fma_rn(a2, b2, __fma_rn(a1, b1, __dmul_rn(a0, b0)));
}
__device__ __forceinline__ double V3(double a0, double a1, double a2, double b0, double b1, double b2) {
    return __fma_rn(a2, b2, __fma_rn(a0, b0, __dmul_rn(a1, b1)));
}

__host__ __device__ __forceinline__ void quat_to_matrix(const double *q, double *R) {
    // math3d.py:45-53, float64 scalar arithmetic
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

// Faces are processed in chunks of FACE_CHUNK consecutive triangles; each chunk
// carries the sorted list of the distinct vertices it references and, per face,
// the three corners as indices into that list (so a chunk samples every vertex once).
#ifndef FACE_CHUNK_DEF
#define FACE_CHUNK_DEF 256  // measured: 128 (4.41 ms) and 512 (4.62 ms) are not faster
#endif
constexpr int FACE_CHUNK = FACE_CHUNK_DEF;

struct MeshDesc {
    const double4 *verts;        // (x, y, z, 0)
    const int4 *tris;            // (a, b, c, 0)
    const int32_t *chunk_voff;   // [nchunks + 1] offsets into chunk_verts
    const int32_t *chunk_verts;  // distinct vertex ids per chunk, ascending
    const uint2 *face_loc;       // per face: (a_loc | b_loc << 16, c_loc) chunk-local corners
    int64_t nv, nt;
    int32_t nchunks, max_chunk_verts;
};

// Per-env transform state, computed on device from the poses.
struct EnvXf {
    double R[9];   // to_grid rotation
    double t[3];   // to_grid translation
    double Rs[9];  // sdf pose rotation (world epilogue)
    double ts[3];
    double cd, tol;
    double cull_lo[3], cull_hi[3];  // lo - margin, hi + margin
    int32_t status;                 // 0 ok, 1 non-finite pose, 2 cd < 0
    int32_t sdf, mesh;
    int32_t pad;
};

// Grid + everything the sampler derives from its scalars once.
template <class T>
struct GridT {
    const T *__restrict__ v;
    int nx, ny, nz;
    int sy, sz;
    double o[3];
    double voxel, rv;   // voxel, RN(1 / voxel)
    double h2, rh2;     // 2 voxel, RN(1 / (2 voxel))  (gradient denominator)
    double nm1[3];      // n - 1 (clamp bound, sdf/_kernels.py:302-304)
    double nm2[3];      // n - 2 (cell clamp, sdf/_kernels.py:261-270)
    int n2[3];
    // Cell-window minima (optional), for the exact face bound (sample_lower_bound):
    // cwin[l][c], c = cx + (nx - 1) (cy + (ny - 1) cz), l = 0..3: the minimum grid value
    // over the corners of the cells [c, c + 2^l - 1] per axis (the window is only read
    // inside the grid).
    const float *__restrict__ cwin;
    // Brick windows (optional), the cheap first pass of the same bound: bwin[t][b],
    // t = (wx - 1) + 2 (wy - 1) + 4 (wz - 1), w in {1, 2}: the minimum grid value over the
    // corners of the cells of bricks [b, b + w - 1] per axis (BRICK cells per brick edge).
    const float *__restrict__ bwin;
    int bnx, bny, bnz;
    // Absolute rounding margin of the bound: (max |value| over the grid) * 2^-40.
    double lbm;
    // The values as a 2D layered texture object (x, y, layer z), or 0: sample_axes then
    // gathers each z face of the cell's corners with one tld4 (CS_NO_TEX builds: __ldg).
    unsigned long long tex;
};

constexpr int BRICK = 2;  // cells per brick edge
#ifdef PREP_STATS
static __device__ unsigned long long g_bound_stat[4];  // brick passes, brick settled, cell passes, cell skipped
#define BOUND_STAT(i) atomicAdd(&g_bound_stat[i], 1ull)
#else
#define BOUND_STAT(i) ((void)0)
#endif
#ifndef CELL_SKIP
#define CELL_SKIP 1.5  // voxels (sample_lower_bound)
#endif
#ifndef CWIN_MAX_LOOKUPS
#define CWIN_MAX_LOOKUPS 12  // face boxes needing more window lookups skip the bound (measured: 8, 12, 16 -> prep 0.86, 0.87, 0.92 ms; descent 1.10, 1.03, 1.03 ms)
#endif
constexpr int CWIN_LEVELS = 4;  // window widths 1, 2, 4, 8 cells


template <class T>
__host__ __device__ inline GridT<T> make_grid(const T *v, int nx, int ny, int nz, double ox, double oy, double oz,
                                               double voxel) {
    GridT<T> g;
    g.v = v;
    g.nx = nx; g.ny = ny; g.nz = nz;
    g.sy = nx; g.sz = nx * ny;
    g.o[0] = ox; g.o[1] = oy; g.o[2] = oz;
    g.voxel = voxel;
    g.rv = 1.0 / voxel;
    g.h2 = 2.0 * voxel;
    g.rh2 = 1.0 / g.h2;
    g.nm1[0] = nx - 1.0; g.nm1[1] = ny - 1.0; g.nm1[2] = nz - 1.0;
    g.nm2[0] = nx - 2.0; g.nm2[1] = ny - 2.0; g.nm2[2] = nz - 2.0;
    g.n2[0] = nx - 2; g.n2[1] = ny - 2; g.n2[2] = nz - 2;
    g.cwin = nullptr;
    g.bwin = nullptr;
    g.tex = 0;
    g.lbm = 0.0;
    g.bnx = (nx - 2) / BRICK + 1; g.bny = (ny - 2) / BRICK + 1; g.bnz = (nz - 2) / BRICK + 1;
    return g;
}

using GridView = GridT<float>;  // per-pair drop-ins sample the caller's float32 grid

// The plan kernels sample the registered float32 values (the promotion to float64
// is exact). Measured against a float64 copy of the grid: half the gather bytes and
// L2 footprint, and faster despite the conversions (profiles/r1_*).
using PlanGrid = GridT<float>;

// Device SDF store entry.
struct SdfDesc {
    const float *values;     // the grid as registered (float32, x-fastest)
    int32_t nx, ny, nz, pad;
    double ox, oy, oz, voxel;
    double lo[3], hi[3];  // mesh AABB (grid.mesh_aabb)
    PlanGrid gp;          // the plan kernels' sampler view (values + brick minima)
};

__device__ __forceinline__ double dmin(double a, double b) { return b < a ? b : a; }
__device__ __forceinline__ double dmax(double a, double b) { return b > a ? b : a; }

// RN(a / b) for b >= 2^-900, given rb = RN(1 / b): one reciprocal multiply and a
// Markstein correction give a faithful q; the exact remainder r2 = a - q b (one FMA)
// then proves q is the correctly rounded quotient: for q normal and not a power of
// two, with 2^k <= |q| < 2^(k+1), q = RN(a / b) iff |a / b - q| < 2^(k-53) (division
// has no ties), i.e. |r2| < 2^k (b 2^-53). That threshold is a power of two times
// b 2^-53, exact whenever it is >= 2^-1000. Anything else (a power-of-two q, tiny or
// zero quotients, a failed proof) takes the IEEE division. Bit-identical to a / b.
// The IEEE division out of line: inlined, the compiler evaluates its fast path on
// every call and selects (if-conversion), which costs as much as the proof saves.
static __device__ __noinline__ double div_ieee(double a, double b) { return a / b; }

__device__ __forceinline__ double div_rn(double a, double b, double rb) {
    double q = a * rb;
    const double r = __fma_rn(-q, b, a);
    q = __fma_rn(r, rb, q);
    const double r2 = __fma_rn(-q, b, a);
    const int qh = __double2hiint(q);
    const double thr = __hiloint2double(qh & 0x7ff00000, 0) * (b * 0x1p-53);
    if (((qh & 0xfffff) | __double2loint(q)) != 0 && thr >= 0x1p-1000 && fabs(r2) < thr) return q;
    return div_ieee(a, b);
}

// x / 3.0 (the centroid, contacts/_kernels.py:40), correctly rounded via div_rn
__device__ __forceinline__ double div3(double x) { return div_rn(x, 3.0, 0x1.5555555555555p-2); }

// One axis of a sample (sdf/_kernels.py:299-308, 256-273): c = min(max(g, 0.0), n - 1.0)
// (numba's max/min keep -0.0), d = g - c (the outside-distance component),
// i = min(floor(c), n - 2), f = c - i.
struct Axis {
    double f, d;
    int i;
};

// For finite g (the contract: poses and vertices are validated finite):
//   * the lower clamp keeps numba's max(-0.0, 0.0) == -0.0 (a select, not DMNMX);
//   * the upper clamp is a select too (fmin costs four instructions on sm_100);
//   * d = g - c is +0.0 exactly when not clamped (no select);
//   * i = min(floor(c), n - 2) and f = c - i: only c == n - 1 is clamped, where the
//     reference's base cell n - 2 gives f = 1 (sdf/_kernels.py:261-270).
__device__ __forceinline__ Axis make_axis(double g, double nm1, double nm2, int n2) {
    Axis a;
    double c = g < 0.0 ? 0.0 : g;
    c = nm1 < c ? nm1 : c;
    a.d = g - c;
    a.i = min(__double2int_rd(c), n2);  // floor (c >= 0)
    a.f = c - __int2double_rn(a.i);
    (void)nm2;
    return a;
}

template <class T>
__device__ __forceinline__ double ld(const T *p) { return (double)__ldg(p); }

// tld4 (Gather4) of a 2D layered float texture: the 2 x 2 texels whose bilinear
// footprint contains (u, v) in layer l, as (x0 y1, x1 y1, x1 y0, x0 y0). With
// u = i + 1, v = j + 1 (exact in float) the footprint is texels i..i+1, j..j+1.
__device__ __forceinline__ float4 gather_a2d(unsigned long long tex, int l, float u, float v) {
    float4 r;
    asm("tld4.r.a2d.v4.f32.f32 {%0, %1, %2, %3}, [%4, {%5, %6, %7, %8}];"
        : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
        : "l"(tex), "r"(l), "f"(u), "f"(v), "f"(0.0f));
    return r;
}

// sample_point with the per-axis work precomputed (sdf/_kernels.py:253-309)
template <class T>
__device__ __forceinline__ double sample_axes(const GridT<T> &g, const Axis &ax, const Axis &ay, const Axis &az) {
    double c000, c100, c010, c110, c001, c101, c011, c111;
#ifndef CS_NO_TEX
    if (g.tex) {
        const float u = (float)(ax.i + 1), v = (float)(ay.i + 1);
        const float4 q0 = gather_a2d(g.tex, az.i, u, v), q1 = gather_a2d(g.tex, az.i + 1, u, v);
        c000 = q0.w; c100 = q0.z; c010 = q0.x; c110 = q0.y;
        c001 = q1.w; c101 = q1.z; c011 = q1.x; c111 = q1.y;
    } else
#endif
    {
        const T *p = g.v + (ax.i + g.nx * (ay.i + g.ny * az.i));
        const int sy = g.sy, sz = g.sz;
        c000 = ld(p); c100 = ld(p + 1); c010 = ld(p + sy); c110 = ld(p + 1 + sy);
        c001 = ld(p + sz); c101 = ld(p + 1 + sz); c011 = ld(p + sy + sz); c111 = ld(p + 1 + sy + sz);
    }
    double ox = 1.0 - ax.f, oy = 1.0 - ay.f, oz = 1.0 - az.f;
    double c00 = c000 * ox + c100 * ax.f;
    double c10 = c010 * ox + c110 * ax.f;
    double c01 = c001 * ox + c101 * ax.f;
    double c11 = c011 * ox + c111 * ax.f;
    double c0 = c00 * oy + c10 * ay.f;
    double c1 = c01 * oy + c11 * ay.f;
    double t = c0 * oz + c1 * az.f;
    // inside the grid the reference adds sqrt(0) * voxel == +0.0
    if ((__double_as_longlong(ax.d) | __double_as_longlong(ay.d) | __double_as_longlong(az.d)) == 0) return t + 0.0;
    return t + sqrt(ax.d * ax.d + ay.d * ay.d + az.d * az.d) * g.voxel;
}

template <class T>
__device__ __forceinline__ Axis axis_at(const GridT<T> &g, int k, double p) {
    return make_axis(div_rn(p - g.o[k], g.voxel, g.rv), g.nm1[k], g.nm2[k], g.n2[k]);
}

// A point with its three axes (so the gradient can reuse them).
struct GPoint {
    double x, y, z;
    Axis ax, ay, az;
};

template <class T>
__device__ __forceinline__ GPoint gpoint(const GridT<T> &g, double x, double y, double z) {
    GPoint q;
    q.x = x; q.y = y; q.z = z;
    q.ax = axis_at(g, 0, x);
    q.ay = axis_at(g, 1, y);
    q.az = axis_at(g, 2, z);
    return q;
}

template <class T>
__device__ __forceinline__ double sample(const GridT<T> &g, double px, double py, double pz) {
    return sample_axes(g, axis_at(g, 0, px), axis_at(g, 1, py), axis_at(g, 2, pz));
}

template <class T>
__device__ __forceinline__ double sample(const GridT<T> &g, const GPoint &q) {
    return sample_axes(g, q.ax, q.ay, q.az);
}

// gradient_point (sdf/_kernels.py:312-327): offsets added in metres before the
// grid conversion, so only the shifted axis is recomputed per sample.
template <class T>
__device__ __forceinline__ void gradient(const GridT<T> &g, const GPoint &p, double &gx, double &gy, double &gz) {
    const double h = g.voxel;
    gx = div_rn(sample_axes(g, axis_at(g, 0, p.x + h), p.ay, p.az) - sample_axes(g, axis_at(g, 0, p.x - h), p.ay, p.az),
                g.h2, g.rh2);
    gy = div_rn(sample_axes(g, p.ax, axis_at(g, 1, p.y + h), p.az) - sample_axes(g, p.ax, axis_at(g, 1, p.y - h), p.az),
                g.h2, g.rh2);
    gz = div_rn(sample_axes(g, p.ax, p.ay, axis_at(g, 2, p.z + h)) - sample_axes(g, p.ax, p.ay, axis_at(g, 2, p.z - h)),
                g.h2, g.rh2);
}

template <class T>
__device__ __forceinline__ void gradient(const GridT<T> &g, double px, double py, double pz, double &gx, double &gy,
                                         double &gz) {
    gradient(g, gpoint(g, px, py, pz), gx, gy, gz);
}

// A lower bound of every trilinear sample (sdf/_kernels.py:253-309) at points of
// the box [lo, hi] (grid frame, metres); -inf (no bound) when it would take more
// than CWIN_MAX_LOOKUPS window lookups. A sample is a convex combination of its
// cell's 8 corners (weights f and 1 - f, evaluated in float64) plus a non-negative
// outside term, and points outside the grid sample a clamped boundary cell, so no
// sample in the box's cells is below the minimum corner value over those cells,
// less the lerps' rounding. That rounding is relative to the LARGEST corner
// magnitude M, not to the minimum: each lerp c0 RN(1 - f) + c1 f rounds the weight,
// both products and the sum (<= 4 u M, u = 2^-53) and the three lerp levels compound
// to < 16 u M = 2^-49 M. The margin is |min| 2^-40 plus lbm = (max |value| over the
// grid) 2^-40, at least 2^9 times that, so the bound holds for any cd, including
// cd -> 0 where the minimum corner is near zero and others are not (grids holding
// NaN / inf get no bound at all: cs_sdf_register). The box is widened by 1e-6 voxel so roundings of the points themselves stay inside. cd_hint: a
// looser bound above it is returned early. The minimum over
// the box's cells is read from the window tables: with w = the largest power of two
// (<= 8) not above any axis' cell count, each axis is covered by windows of w cells
// (overlapping at the end; min is idempotent), so the bound is exactly the minimum
// over the box's cells.
template <class T>
__device__ __forceinline__ double sample_lower_bound(const GridT<T> &g, const double lo[3], const double hi[3],
                                                    double cd_hint) {
    int c0[3], c1[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const double a = (lo[k] - g.o[k]) * g.rv - 1e-6, b = (hi[k] - g.o[k]) * g.rv + 1e-6;
        c0[k] = a < 0.0 ? 0 : (a > g.nm2[k] ? g.n2[k] : (int)a);
        c1[k] = b < 0.0 ? 0 : (b > g.nm2[k] ? g.n2[k] : (int)b);
    }
    const int cnx = g.nx - 1, cny = g.ny - 1;
    const size_t ntab = (size_t)cnx * cny * (g.nz - 1);
    // First a cheap pass over the box's bricks (a superset of its cells: a lower bound
    // too), from the brick windows: per axis one width-1 window or width-2 windows
    // (overlapping at the end; min is idempotent). Faces it cannot settle take the exact
    // pass over the cells.
#ifndef NO_BWIN
    if (g.bwin) {
        int b0[3], w[3], last[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            b0[k] = c0[k] / BRICK;
            const int b1 = c1[k] / BRICK;
            w[k] = b1 > b0[k] ? 2 : 1;
            last[k] = b1 - w[k] + 1;
        }
        const float *tab = g.bwin + (size_t)((w[0] - 1) + 2 * (w[1] - 1) + 4 * (w[2] - 1)) * g.bnx * g.bny * g.bnz;
        float m = INFINITY;
        if (last[0] - b0[0] <= 2 && last[1] - b0[1] <= 2 && last[2] - b0[2] <= 2) {
            // at most two windows per axis (the usual case): eight independent loads in
            // flight together (repeats when one window suffices)
            const int x1 = last[0], y0 = g.bnx * b0[1], y1 = g.bnx * last[1];
            const int z0 = g.bnx * g.bny * b0[2], z1 = g.bnx * g.bny * last[2];
            const float *r00 = tab + y0 + z0, *r01 = tab + y0 + z1, *r10 = tab + y1 + z0, *r11 = tab + y1 + z1;
            m = fminf(fminf(fminf(__ldg(r00 + b0[0]), __ldg(r00 + x1)), fminf(__ldg(r10 + b0[0]), __ldg(r10 + x1))),
                      fminf(fminf(__ldg(r01 + b0[0]), __ldg(r01 + x1)), fminf(__ldg(r11 + b0[0]), __ldg(r11 + x1))));
        } else {
            for (int z = b0[2];; z = min(z + 2, last[2])) {
                for (int y = b0[1];; y = min(y + 2, last[1])) {
                    const float *row = tab + g.bnx * (y + g.bny * z);
                    for (int x = b0[0];; x = min(x + 2, last[0])) {
                        m = fminf(m, __ldg(row + x));
                        if (x >= last[0]) break;
                    }
                    if (y >= last[1]) break;
                }
                if (z >= last[2]) break;
            }
        }
        const double md = (double)m;
        const double lb = md - fabs(md) * 0x1p-40 - g.lbm - 1e-300;
        BOUND_STAT(0);
        if (lb > cd_hint) { BOUND_STAT(1); return lb; }
        // the cell pass lifts the bound by about a brick at most: it is skipped when the
        // brick bound is far below cd (a missed cull at worst, never a wrong one; measured
        // best at 1.5 voxels: faster prep, no extra descents)
        if (lb < cd_hint - CELL_SKIP * g.voxel) return lb;
    }
#endif
    const int rmin = min(c1[0] - c0[0], min(c1[1] - c0[1], c1[2] - c0[2])) + 1;
    const int lvl = rmin >= 8 ? 3 : rmin >= 4 ? 2 : rmin >= 2 ? 1 : 0, w = 1 << lvl;
    int n = 1, last[3], nw[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        last[k] = c1[k] - w + 1;                     // start of the last window (>= c0[k])
        nw[k] = ((last[k] - c0[k] + w - 1) >> lvl) + 1;  // windows along the axis
        n *= nw[k];
    }
    if (n > CWIN_MAX_LOOKUPS) { BOUND_STAT(3); return -INFINITY; }
    BOUND_STAT(2);
    const float *tab = g.cwin + (size_t)lvl * ntab;  // < 2^31 entries per table: 32-bit offsets
    float m = INFINITY;
    if (nw[0] <= 2 && nw[1] <= 2 && nw[2] <= 2) {
        // the usual case: per axis the windows start at c0 and at last (one window: the
        // same start twice; min is idempotent), eight independent loads
        const int x0 = c0[0], x1 = last[0], sy = cnx, sz = cnx * cny;
        const int y0 = sy * c0[1], y1 = sy * last[1], z0 = sz * c0[2], z1 = sz * last[2];
        m = fminf(fminf(fminf(__ldg(tab + (x0 + y0 + z0)), __ldg(tab + (x1 + y0 + z0))),
                        fminf(__ldg(tab + (x0 + y1 + z0)), __ldg(tab + (x1 + y1 + z0)))),
                  fminf(fminf(__ldg(tab + (x0 + y0 + z1)), __ldg(tab + (x1 + y0 + z1))),
                        fminf(__ldg(tab + (x0 + y1 + z1)), __ldg(tab + (x1 + y1 + z1)))));
    } else {
        // up to CWIN_MAX_LOOKUPS windows: (ix, iy, iz) walks them, loads predicated
        int ix = 0, iy = 0, iz = 0;
        float r[CWIN_MAX_LOOKUPS];
#pragma unroll
        for (int i = 0; i < CWIN_MAX_LOOKUPS; ++i) {
            const int x = min(c0[0] + ix * w, last[0]), y = min(c0[1] + iy * w, last[1]), z = min(c0[2] + iz * w, last[2]);
            r[i] = i < n ? __ldg(tab + (x + cnx * (y + cny * z))) : INFINITY;
            if (++ix == nw[0]) { ix = 0; if (++iy == nw[1]) { iy = 0; ++iz; } }
        }
#pragma unroll
        for (int i = 0; i < CWIN_MAX_LOOKUPS; ++i) m = fminf(m, r[i]);
    }
    const double md = (double)m;
    return md - fabs(md) * 0x1p-40 - g.lbm - 1e-300;
}

// sdf/_kernels.py:20-61
__device__ __forceinline__ void closest_point(double ax, double ay, double az, double bx, double by, double bz,
                                              double cx, double cy, double cz, double px, double py, double pz,
                                              double &qx, double &qy, double &qz) {
    double abx = bx - ax, aby = by - ay, abz = bz - az;
    double acx = cx - ax, acy = cy - ay, acz = cz - az;
    double apx = px - ax, apy = py - ay, apz = pz - az;
    double d1 = abx * apx + aby * apy + abz * apz;
    double d2 = acx * apx + acy * apy + acz * apz;
    if (d1 <= 0.0 && d2 <= 0.0) { qx = ax; qy = ay; qz = az; return; }
    double bpx = px - bx, bpy = py - by, bpz = pz - bz;
    double d3 = abx * bpx + aby * bpy + abz * bpz;
    double d4 = acx * bpx + acy * bpy + acz * bpz;
    if (d3 >= 0.0 && d4 <= d3) { qx = bx; qy = by; qz = bz; return; }
    double vc = d1 * d4 - d3 * d2;
    if (vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0) {
        double v = d1 / (d1 - d3);
        qx = ax + v * abx; qy = ay + v * aby; qz = az + v * abz; return;
    }
    double cpx = px - cx, cpy = py - cy, cpz = pz - cz;
    double d5 = abx * cpx + aby * cpy + abz * cpz;
    double d6 = acx * cpx + acy * cpy + acz * cpz;
    if (d6 >= 0.0 && d5 <= d6) { qx = cx; qy = cy; qz = cz; return; }
    double vb = d5 * d2 - d1 * d6;
    if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) {
        double w = d2 / (d2 - d6);
        qx = ax + w * acx; qy = ay + w * acy; qz = az + w * acz; return;
    }
    double va = d3 * d6 - d5 * d4;
    if (va <= 0.0 && (d4 - d3) >= 0.0 && (d5 - d6) >= 0.0) {
        double w = (d4 - d3) / ((d4 - d3) + (d5 - d6));
        qx = bx + w * (cx - bx); qy = by + w * (cy - by); qz = bz + w * (cz - bz); return;
    }
    double denom = 1.0 / (va + vb + vc);
    double v = vb * denom, w = vc * denom;
    qx = ax + abx * v + acx * w;
    qy = ay + aby * v + acy * w;
    qz = az + abz * v + acz * w;
}

__device__ __forceinline__ bool same3(double x, double y, double z, double a, double b, double c) {
    return __double_as_longlong(x) == __double_as_longlong(a) && __double_as_longlong(y) == __double_as_longlong(b) &&
           __double_as_longlong(z) == __double_as_longlong(c);
}

struct FaceResult {
    double px, py, pz, phi, gx, gy, gz;
    int nsamp;
};

// contacts/_kernels.py:20-87 for one face. Returns false if pruned by the
// Lipschitz bound (the reference then writes only found = 0).
// The final gradient equals the last in-loop gradient whenever the point did not
// move after it (same input -> same value), so it is reused in that case.
// COUNT: tally trilinear samples in r.nsamp (roofline accounting).
template <bool COUNT = false, class T>
__device__ __forceinline__ bool face_body(const GridT<T> &g, double ax, double ay, double az, double bx, double by,
                                          double bz, double cx, double cy, double cz, double cd, int max_iters,
                                          double tol, FaceResult &r) {
    if (COUNT) r.nsamp = 3;
    double phi_a = sample(g, ax, ay, az), phi_b = sample(g, bx, by, bz), phi_c = sample(g, cx, cy, cz);
    // max of the three edge lengths (contacts/_kernels.py:30-33): sqrt is correctly rounded and
    // monotone, so the max of the roots is the root of the max (one sqrt instead of three)
    const double s0 = (bx - ax) * (bx - ax) + (by - ay) * (by - ay) + (bz - az) * (bz - az);
    const double s1 = (cx - bx) * (cx - bx) + (cy - by) * (cy - by) + (cz - bz) * (cz - bz);
    const double s2 = (ax - cx) * (ax - cx) + (ay - cy) * (ay - cy) + (az - cz) * (az - cz);
    double diam = sqrt(dmax(s0, dmax(s1, s2)));
    double phi_min = dmin(phi_a, dmin(phi_b, phi_c));
    if (phi_min - diam > cd) return false;
    double sx = div3(ax + bx + cx), sy = div3(ay + by + cy), sz = div3(az + bz + cz);
    double phi = sample(g, sx, sy, sz);
    if (COUNT) r.nsamp += 1;
    if (phi_a < phi) { sx = ax; sy = ay; sz = az; phi = phi_a; }
    if (phi_b < phi) { sx = bx; sy = by; sz = bz; phi = phi_b; }
    if (phi_c < phi) { sx = cx; sy = cy; sz = cz; phi = phi_c; }
    GPoint p = gpoint(g, sx, sy, sz);  // axes recomputed (same inputs, same bits)
    double alpha = g.voxel, amax = 4.0 * g.voxel;
    double grx = 0.0, gry = 0.0, grz = 0.0;
    bool have_grad = false;  // gradient at the current p is in gr*
    for (int it = 0; it < max_iters; ++it) {
        gradient(g, p, grx, gry, grz);
        if (COUNT) r.nsamp += 6;
        have_grad = true;
        double gnorm = sqrt(grx * grx + gry * gry + grz * grz);
        if (gnorm < 1e-12) break;
        double ux = grx / gnorm, uy = gry / gnorm, uz = grz / gnorm;
        double moved = 0.0;
        for (int bt = 0; bt < 4; ++bt) {
            double qx, qy, qz;
            closest_point(ax, ay, az, bx, by, bz, cx, cy, cz, p.x - alpha * ux, p.y - alpha * uy, p.z - alpha * uz,
                          qx, qy, qz);
            // The projection often lands exactly on the current point or on a vertex
            // (Ericson's vertex regions return the corner itself): identical inputs,
            // so the sample's value is already known.
            double phi_new;
            int known = same3(qx, qy, qz, p.x, p.y, p.z) ? 0
                        : same3(qx, qy, qz, ax, ay, az)  ? 1
                        : same3(qx, qy, qz, bx, by, bz)  ? 2
                        : same3(qx, qy, qz, cx, cy, cz)  ? 3
                                                         : -1;
            if (known >= 0) {
                phi_new = known == 0 ? phi : known == 1 ? phi_a : known == 2 ? phi_b : phi_c;
            } else {
                phi_new = sample(g, qx, qy, qz);
                if (COUNT) r.nsamp += 1;
            }
            if (phi_new < phi) {
                moved = sqrt((qx - p.x) * (qx - p.x) + (qy - p.y) * (qy - p.y) + (qz - p.z) * (qz - p.z));
                p = gpoint(g, qx, qy, qz);
                phi = phi_new;
                have_grad = false;
                alpha = dmin(alpha * 1.5, amax);
                break;
            }
            alpha *= 0.5;
        }
        if (moved < tol) break;
    }
    if (!have_grad) {
        gradient(g, p, grx, gry, grz);
        if (COUNT) r.nsamp += 6;
    }
    r.px = p.x; r.py = p.y; r.pz = p.z; r.phi = phi;
    r.gx = grx; r.gy = gry; r.gz = grz;
    return true;
}

// ------------------------------------------------------------------ block helpers

__device__ __forceinline__ int warp_incl_scan(int v) {
    int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int n = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += n;
    }
    return v;
}

// Exclusive scan over the block; returns this thread's exclusive prefix and
// writes the block total to *total. `ws` needs WS_INTS ints of shared memory
// (one per warp plus the total, so 1024-thread blocks are safe).
constexpr int WS_INTS = 33;
__device__ __forceinline__ int block_excl_scan(int v, int *ws, int *total) {
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    int inc = warp_incl_scan(v);
    if (lane == 31) ws[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        int x = lane < nw ? ws[lane] : 0;
        int xi = warp_incl_scan(x);
        if (lane < nw) ws[lane] = xi - x;
        if (lane == nw - 1) ws[32] = xi;
    }
    __syncthreads();
    int r = ws[wid] + inc - v;
    *total = ws[32];
    __syncthreads();
    return r;
}

}  // namespace cs
