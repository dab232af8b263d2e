// GPU SDF generation, bit-identical to the reference's CPU generate_sdf.
//
//   k_unsigned   one thread per node: min over all triangles of the squared
//                Ericson distance (triangles staged through shared memory in
//                tiles; a conservative AABB bound skips far triangles without
//                changing the exact minimum), then sqrt.
//   k_cross      per ray axis, one thread per triangle: count / fill the
//                ray-column crossings (sdf/_kernels.py:169-218).
//   k_vote       one thread per column: sort crossings, parity vote per node
//                (sdf/_kernels.py:221-245).
//   k_sign       values = float32(unsigned * (votes > 0 ? 1 : -1)) (grid.py:204-205).
#include <vector>

#include "cs_sdfgen.cuh"

namespace cs {

namespace {

constexpr int UD_BLOCK = 256;
constexpr int UD_TILE = 256;
constexpr double NUDGE_U = 2.0954e-4;  // grid.py:32-33
constexpr double NUDGE_V = 3.1416e-4;

// point_triangle_sqdist (sdf/_kernels.py:64-73)
__device__ __forceinline__ double tri_sqdist(const double *t, double px, double py, double pz) {
    double qx, qy, qz;
    closest_point(t[0], t[1], t[2], t[3], t[4], t[5], t[6], t[7], t[8], px, py, pz, qx, qy, qz);
    double dx = px - qx, dy = py - qy, dz = pz - qz;
    return dx * dx + dy * dy + dz * dz;
}

__global__ void __launch_bounds__(UD_BLOCK) k_unsigned(const double *__restrict__ tv, const double *__restrict__ tbox,
                                                       int64_t nt, int nx, int ny, int nz, double ox, double oy,
                                                       double oz, double voxel, double *__restrict__ out) {
    __shared__ double st[UD_TILE * 9];
    __shared__ double sb[UD_TILE * 6];
    const int64_t total = (int64_t)nx * ny * nz;
    const int64_t idx = blockIdx.x * (int64_t)UD_BLOCK + threadIdx.x;
    const bool active = idx < total;
    double px = 0, py = 0, pz = 0;
    if (active) {
        int64_t iz = idx / ((int64_t)nx * ny);
        int64_t rem = idx - iz * ((int64_t)nx * ny);
        int64_t iy = rem / nx;
        int64_t ix = rem - iy * nx;
        px = ox + (double)ix * voxel;  // sdf/_kernels.py:153-155
        py = oy + (double)iy * voxel;
        pz = oz + (double)iz * voxel;
    }
    double best = 1e30;  // BIG (sdf/_kernels.py:12)
    for (int64_t t0 = 0; t0 < nt; t0 += UD_TILE) {
        int cnt = (int)((nt - t0) < UD_TILE ? (nt - t0) : UD_TILE);
        __syncthreads();
        for (int k = threadIdx.x; k < cnt * 9; k += UD_BLOCK) st[k] = tv[t0 * 9 + k];
        for (int k = threadIdx.x; k < cnt * 6; k += UD_BLOCK) sb[k] = tbox[t0 * 6 + k];
        __syncthreads();
        if (!active) continue;
        for (int k = 0; k < cnt; ++k) {
            const double *b = sb + 6 * k;
            double d = 0.0, v;
            v = b[0] - px; if (v > 0.0) d += v * v;
            v = px - b[3]; if (v > 0.0) d += v * v;
            v = b[1] - py; if (v > 0.0) d += v * v;
            v = py - b[4]; if (v > 0.0) d += v * v;
            v = b[2] - pz; if (v > 0.0) d += v * v;
            v = pz - b[5]; if (v > 0.0) d += v * v;
            // conservative: the box bound is only used to skip triangles that
            // cannot be within 1e-9 relative of the current minimum
            if (d > best * (1.0 + 1e-9) + 1e-24) continue;
            double dsq = tri_sqdist(st + 9 * k, px, py, pz);
            if (dsq < best) best = dsq;
        }
    }
    if (active) out[idx] = sqrt(best);
}

struct AxisSetup {
    int pu, pv, pw;       // coordinate permutation
    int nu, nv, nw;
    int64_t su, sv, sw;   // node strides
    double ou, ov, ow;
};

// _count_or_fill_crossings (sdf/_kernels.py:169-218); fill == 0 counts, 1 writes.
__global__ void k_cross(const double *__restrict__ tv, int64_t nt, AxisSetup a, double voxel, double nudge_u,
                        double nudge_v, int fill, int *__restrict__ counts, int *__restrict__ cursor,
                        double *__restrict__ cross_w) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= nt) return;
    const double *p = tv + 9 * t;
    double au = p[a.pu], bu = p[3 + a.pu], cu = p[6 + a.pu];
    double av = p[a.pv], bv = p[3 + a.pv], cv = p[6 + a.pv];
    double aw = p[a.pw], bw = p[3 + a.pw], cw = p[6 + a.pw];
    double area = (bu - au) * (cv - av) - (bv - av) * (cu - au);
    if (area == 0.0) return;
    double min_u = dmin(au, dmin(bu, cu)), max_u = dmax(au, dmax(bu, cu));
    double min_v = dmin(av, dmin(bv, cv)), max_v = dmax(av, dmax(bv, cv));
    int64_t iu0 = (int64_t)ceil((min_u - a.ou - nudge_u) / voxel); if (iu0 < 0) iu0 = 0;
    int64_t iu1 = (int64_t)floor((max_u - a.ou - nudge_u) / voxel); if (iu1 > a.nu - 1) iu1 = a.nu - 1;
    int64_t iv0 = (int64_t)ceil((min_v - a.ov - nudge_v) / voxel); if (iv0 < 0) iv0 = 0;
    int64_t iv1 = (int64_t)floor((max_v - a.ov - nudge_v) / voxel); if (iv1 > a.nv - 1) iv1 = a.nv - 1;
    for (int64_t iu = iu0; iu <= iu1; ++iu) {
        double pu = a.ou + (double)iu * voxel + nudge_u;
        for (int64_t iv = iv0; iv <= iv1; ++iv) {
            double pv = a.ov + (double)iv * voxel + nudge_v;
            double e0 = (bu - au) * (pv - av) - (bv - av) * (pu - au);
            double e1 = (cu - bu) * (pv - bv) - (cv - bv) * (pu - bu);
            double e2 = (au - cu) * (pv - cv) - (av - cv) * (pu - cu);
            bool inside = (e0 > 0.0 && e1 > 0.0 && e2 > 0.0) || (e0 < 0.0 && e1 < 0.0 && e2 < 0.0);
            if (!inside) continue;
            int64_t col = iu * a.nv + iv;
            if (fill == 0) {
                atomicAdd(counts + col, 1);
            } else {
                double wa = e1 / area, wb = e2 / area;
                double wc = 1.0 - wa - wb;
                double w = wa * aw + wb * bw + wc * cw;
                int pos = atomicAdd(cursor + col, 1);
                cross_w[pos] = w;
            }
        }
    }
}

__global__ void k_scan_serial(const int *__restrict__ counts, int64_t n, int *__restrict__ starts) {
    // single block: chunked block scan
    __shared__ int ws[WS_INTS];
    int running = 0;
    for (int64_t i0 = 0; i0 < n; i0 += blockDim.x) {
        int64_t i = i0 + threadIdx.x;
        int v = i < n ? counts[i] : 0;
        int tot;
        int x = block_excl_scan(v, ws, &tot);
        if (i < n) starts[i] = running + x;
        running += tot;
    }
}

// _vote_columns (sdf/_kernels.py:221-245); the crossing multiset is sorted, so
// the fill order (atomics) does not matter.
__global__ void k_vote(AxisSetup a, double voxel, const int *__restrict__ starts, const int *__restrict__ counts,
                       double *__restrict__ cross_w, int *__restrict__ votes) {
    int64_t col = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (col >= (int64_t)a.nu * a.nv) return;
    int64_t iu = col / a.nv, iv = col - iu * a.nv;
    int start = starts[col], cnt = counts[col];
    double *cw = cross_w + start;
    for (int i = 1; i < cnt; ++i) {
        double key = cw[i];
        int j = i - 1;
        while (j >= 0 && cw[j] > key) { cw[j + 1] = cw[j]; --j; }
        cw[j + 1] = key;
    }
    int k = 0;
    for (int64_t iw = 0; iw < a.nw; ++iw) {
        double w = a.ow + (double)iw * voxel;
        while (k < cnt && cw[k] < w) ++k;
        int64_t node = iu * a.su + iv * a.sv + iw * a.sw;
        votes[node] += (k & 1) ? -1 : 1;
    }
}

__global__ void k_sign(const double *__restrict__ ud, const int *__restrict__ votes, int64_t n, float *__restrict__ out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) out[i] = __double2float_rn(ud[i] * (votes[i] > 0 ? 1.0 : -1.0));
}

template <class T>
struct DevBuf {
    T *p = nullptr;
    ~DevBuf() { if (p) cudaFree(p); }
    cudaError_t alloc(size_t n) { return cudaMalloc(&p, (n ? n : 1) * sizeof(T)); }
};

}  // namespace

int sdf_generate(const double *vertices, int64_t nv, const int32_t *triangles, int64_t nt, int nx, int ny, int nz,
                 const double origin[3], double voxel, float *values_out, std::string *err) {
    (void)nv;
    const int64_t n = (int64_t)nx * ny * nz;
    // triangle corners in mesh order (mesh.triangle_corners(), bvh.py:24) and boxes
    std::vector<double> tv((size_t)nt * 9), tb((size_t)nt * 6);
    for (int64_t t = 0; t < nt; ++t) {
        for (int c = 0; c < 3; ++c)
            for (int k = 0; k < 3; ++k) tv[(size_t)(9 * t + 3 * c + k)] = vertices[3 * (int64_t)triangles[3 * t + c] + k];
        for (int k = 0; k < 3; ++k) {
            double a = tv[(size_t)(9 * t + k)], b = tv[(size_t)(9 * t + 3 + k)], c = tv[(size_t)(9 * t + 6 + k)];
            tb[(size_t)(6 * t + k)] = std::min(a, std::min(b, c));
            tb[(size_t)(6 * t + 3 + k)] = std::max(a, std::max(b, c));
        }
    }
    DevBuf<double> d_tv, d_tb, d_ud, d_cw;
    DevBuf<int> d_votes, d_cnt, d_start, d_cur;
    DevBuf<float> d_out;
    auto chk = [&](cudaError_t e, const char *what) {
        if (e != cudaSuccess) { *err = std::string(what) + ": " + cudaGetErrorString(e); return false; }
        return true;
    };
    if (!chk(d_tv.alloc(tv.size()), "alloc") || !chk(d_tb.alloc(tb.size()), "alloc") ||
        !chk(d_ud.alloc((size_t)n), "alloc") || !chk(d_votes.alloc((size_t)n), "alloc") ||
        !chk(d_out.alloc((size_t)n), "alloc"))
        return CS_ERR_OOM;
    if (!chk(cudaMemcpy(d_tv.p, tv.data(), tv.size() * 8, cudaMemcpyHostToDevice), "upload") ||
        !chk(cudaMemcpy(d_tb.p, tb.data(), tb.size() * 8, cudaMemcpyHostToDevice), "upload") ||
        !chk(cudaMemset(d_votes.p, 0, (size_t)n * sizeof(int)), "memset"))
        return CS_ERR_CUDA;
    k_unsigned<<<(unsigned)((n + UD_BLOCK - 1) / UD_BLOCK), UD_BLOCK>>>(d_tv.p, d_tb.p, nt, nx, ny, nz, origin[0],
                                                                       origin[1], origin[2], voxel, d_ud.p);
    if (!chk(cudaGetLastError(), "k_unsigned")) return CS_ERR_CUDA;

    const int dims[3] = {nx, ny, nz};
    const int64_t strides[3] = {1, nx, (int64_t)nx * ny};
    const int perms[3][3] = {{1, 2, 0}, {2, 0, 1}, {0, 1, 2}};  // rays along x, y, z (grid.py:214-218)
    for (int s = 0; s < 3; ++s) {
        AxisSetup a;
        a.pu = perms[s][0]; a.pv = perms[s][1]; a.pw = perms[s][2];
        a.nu = dims[a.pu]; a.nv = dims[a.pv]; a.nw = dims[a.pw];
        a.su = strides[a.pu]; a.sv = strides[a.pv]; a.sw = strides[a.pw];
        a.ou = origin[a.pu]; a.ov = origin[a.pv]; a.ow = origin[a.pw];
        const int64_t ncol = (int64_t)a.nu * a.nv;
        DevBuf<int> cnt, start, cur;
        if (!chk(cnt.alloc((size_t)ncol), "alloc") || !chk(start.alloc((size_t)ncol), "alloc") ||
            !chk(cur.alloc((size_t)ncol), "alloc"))
            return CS_ERR_OOM;
        if (!chk(cudaMemset(cnt.p, 0, (size_t)ncol * sizeof(int)), "memset")) return CS_ERR_CUDA;
        const double nu_ = NUDGE_U * voxel, nv_ = NUDGE_V * voxel;
        unsigned gb = (unsigned)((nt + 127) / 128);
        k_cross<<<gb, 128>>>(d_tv.p, nt, a, voxel, nu_, nv_, 0, cnt.p, nullptr, nullptr);
        k_scan_serial<<<1, 1024>>>(cnt.p, ncol, start.p);
        int last_start = 0, last_cnt = 0;
        if (!chk(cudaMemcpy(&last_start, start.p + ncol - 1, sizeof(int), cudaMemcpyDeviceToHost), "scan") ||
            !chk(cudaMemcpy(&last_cnt, cnt.p + ncol - 1, sizeof(int), cudaMemcpyDeviceToHost), "scan"))
            return CS_ERR_CUDA;
        int64_t total = (int64_t)last_start + last_cnt;
        DevBuf<double> cw;
        if (!chk(cw.alloc((size_t)total), "alloc")) return CS_ERR_OOM;
        if (!chk(cudaMemcpy(cur.p, start.p, (size_t)ncol * sizeof(int), cudaMemcpyDeviceToDevice), "copy")) return CS_ERR_CUDA;
        k_cross<<<gb, 128>>>(d_tv.p, nt, a, voxel, nu_, nv_, 1, cnt.p, cur.p, cw.p);
        k_vote<<<(unsigned)((ncol + 127) / 128), 128>>>(a, voxel, start.p, cnt.p, cw.p, d_votes.p);
        if (!chk(cudaGetLastError(), "k_vote")) return CS_ERR_CUDA;
        if (!chk(cudaDeviceSynchronize(), "parity votes")) return CS_ERR_CUDA;
    }
    k_sign<<<(unsigned)((n + 255) / 256), 256>>>(d_ud.p, d_votes.p, n, d_out.p);
    if (!chk(cudaGetLastError(), "k_sign")) return CS_ERR_CUDA;
    if (!chk(cudaMemcpy(values_out, d_out.p, (size_t)n * sizeof(float), cudaMemcpyDeviceToHost), "download"))
        return CS_ERR_CUDA;
    return CS_OK;
}

}  // namespace cs
