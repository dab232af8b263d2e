// Shared device code for the contact path. Compiled with -fmad=false: plain
// double arithmetic is never contracted, so every expression rounds exactly like
// the reference's numba kernels; the reference's BLAS dot products are
// reproduced with explicit fma (G3 / V3 below).
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

struct SdfDesc {
    const float *values;
    int32_t nx, ny, nz, pad;
    double ox, oy, oz, voxel;
    double lo[3], hi[3];  // mesh AABB (grid.mesh_aabb)
};

struct MeshDesc {
    const double4 *verts;  // (x, y, z, 0)
    const int4 *tris;      // (a, b, c, 0)
    int64_t nv, nt;
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

struct GridView {
    const float *__restrict__ v;
    int nx, ny, nz;
    double ox, oy, oz, voxel;
};

__device__ __forceinline__ GridView make_view(const SdfDesc &d) {
    GridView g;
    g.v = d.values;
    g.nx = d.nx; g.ny = d.ny; g.nz = d.nz;
    g.ox = d.ox; g.oy = d.oy; g.oz = d.oz; g.voxel = d.voxel;
    return g;
}

__device__ __forceinline__ double dmin(double a, double b) { return b < a ? b : a; }
__device__ __forceinline__ double dmax(double a, double b) { return b > a ? b : a; }

// sdf/_kernels.py:253-292
__device__ __forceinline__ double trilinear(const GridView &g, double gx, double gy, double gz) {
    int x0 = (int)floor(gx), y0 = (int)floor(gy), z0 = (int)floor(gz);
    x0 = x0 < 0 ? 0 : x0; x0 = x0 > g.nx - 2 ? g.nx - 2 : x0;
    y0 = y0 < 0 ? 0 : y0; y0 = y0 > g.ny - 2 ? g.ny - 2 : y0;
    z0 = z0 < 0 ? 0 : z0; z0 = z0 > g.nz - 2 ? g.nz - 2 : z0;
    double fx = gx - (double)x0, fy = gy - (double)y0, fz = gz - (double)z0;
    int sy = g.nx, sz = g.nx * g.ny;
    const float *p = g.v + (x0 + g.nx * (y0 + g.ny * z0));
    double c000 = __ldg(p), c100 = __ldg(p + 1), c010 = __ldg(p + sy), c110 = __ldg(p + 1 + sy);
    double c001 = __ldg(p + sz), c101 = __ldg(p + 1 + sz), c011 = __ldg(p + sy + sz), c111 = __ldg(p + 1 + sy + sz);
    double ox = 1.0 - fx, oy = 1.0 - fy, oz = 1.0 - fz;
    double c00 = c000 * ox + c100 * fx;
    double c10 = c010 * ox + c110 * fx;
    double c01 = c001 * ox + c101 * fx;
    double c11 = c011 * ox + c111 * fx;
    double c0 = c00 * oy + c10 * fy;
    double c1 = c01 * oy + c11 * fy;
    return c0 * oz + c1 * fz;
}

// sdf/_kernels.py:295-309
__device__ __forceinline__ double sample(const GridView &g, double px, double py, double pz) {
    double gx = (px - g.ox) / g.voxel;
    double gy = (py - g.oy) / g.voxel;
    double gz = (pz - g.oz) / g.voxel;
    double cx = dmin(dmax(gx, 0.0), (double)g.nx - 1.0);
    double cy = dmin(dmax(gy, 0.0), (double)g.ny - 1.0);
    double cz = dmin(dmax(gz, 0.0), (double)g.nz - 1.0);
    double dx = gx - cx, dy = gy - cy, dz = gz - cz;
    double out = dx * dx + dy * dy + dz * dz;
    double t = trilinear(g, cx, cy, cz);
    // sqrt(0) * voxel == 0 exactly: skip the sqrt for the (98.6%) inside samples.
    return out == 0.0 ? t + 0.0 * g.voxel : t + sqrt(out) * g.voxel;
}

// sdf/_kernels.py:312-327
__device__ __forceinline__ void gradient(const GridView &g, double px, double py, double pz, double &gx, double &gy,
                                         double &gz) {
    double h = g.voxel, h2 = 2.0 * g.voxel;
    gx = (sample(g, px + h, py, pz) - sample(g, px - h, py, pz)) / h2;
    gy = (sample(g, px, py + h, pz) - sample(g, px, py - h, pz)) / h2;
    gz = (sample(g, px, py, pz + h) - sample(g, px, py, pz - h)) / h2;
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

struct FaceResult {
    double px, py, pz, phi, gx, gy, gz;
    int nsamp;
};

// contacts/_kernels.py:20-87 for one face. Returns false if pruned by the
// Lipschitz bound (the reference then writes only found = 0).
// The final gradient equals the last in-loop gradient whenever the point did not
// move after it (same input -> same value), so it is reused in that case.
// COUNT: tally trilinear samples in r.nsamp (roofline accounting).
template <bool COUNT = false>
__device__ __forceinline__ bool face_body(const GridView &g, double ax, double ay, double az, double bx, double by,
                                          double bz, double cx, double cy, double cz, double cd, int max_iters,
                                          double tol, FaceResult &r) {
    if (COUNT) r.nsamp = 3;
    double phi_a = sample(g, ax, ay, az);
    double phi_b = sample(g, bx, by, bz);
    double phi_c = sample(g, cx, cy, cz);
    double e0 = sqrt((bx - ax) * (bx - ax) + (by - ay) * (by - ay) + (bz - az) * (bz - az));
    double e1 = sqrt((cx - bx) * (cx - bx) + (cy - by) * (cy - by) + (cz - bz) * (cz - bz));
    double e2 = sqrt((ax - cx) * (ax - cx) + (ay - cy) * (ay - cy) + (az - cz) * (az - cz));
    double diam = dmax(e0, dmax(e1, e2));
    double phi_min = dmin(phi_a, dmin(phi_b, phi_c));
    if (phi_min - diam > cd) return false;
    double gxc = (ax + bx + cx) / 3.0, gyc = (ay + by + cy) / 3.0, gzc = (az + bz + cz) / 3.0;
    double phi = sample(g, gxc, gyc, gzc);
    if (COUNT) r.nsamp += 1;
    double px = gxc, py = gyc, pz = gzc;
    if (phi_a < phi) { px = ax; py = ay; pz = az; phi = phi_a; }
    if (phi_b < phi) { px = bx; py = by; pz = bz; phi = phi_b; }
    if (phi_c < phi) { px = cx; py = cy; pz = cz; phi = phi_c; }
    double alpha = g.voxel, amax = 4.0 * g.voxel;
    double grx = 0.0, gry = 0.0, grz = 0.0;
    bool have_grad = false;  // gradient at the current (px,py,pz) is in gr*
    for (int it = 0; it < max_iters; ++it) {
        gradient(g, px, py, pz, grx, gry, grz);
        if (COUNT) r.nsamp += 6;
        have_grad = true;
        double gnorm = sqrt(grx * grx + gry * gry + grz * grz);
        if (gnorm < 1e-12) break;
        double ux = grx / gnorm, uy = gry / gnorm, uz = grz / gnorm;
        double moved = 0.0;
        for (int bt = 0; bt < 4; ++bt) {
            double qx, qy, qz;
            closest_point(ax, ay, az, bx, by, bz, cx, cy, cz, px - alpha * ux, py - alpha * uy, pz - alpha * uz, qx,
                          qy, qz);
            double phi_new = sample(g, qx, qy, qz);
            if (COUNT) r.nsamp += 1;
            if (phi_new < phi) {
                moved = sqrt((qx - px) * (qx - px) + (qy - py) * (qy - py) + (qz - pz) * (qz - pz));
                px = qx; py = qy; pz = qz; phi = phi_new;
                have_grad = false;
                alpha = dmin(alpha * 1.5, amax);
                break;
            }
            alpha *= 0.5;
        }
        if (moved < tol) break;
    }
    if (!have_grad) {
        gradient(g, px, py, pz, grx, gry, grz);
        if (COUNT) r.nsamp += 6;
    }
    r.px = px; r.py = py; r.pz = pz; r.phi = phi;
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
