// Contact generation on sm_100a.
//
//   k_env_xf       per env: poses -> to_grid transform, cull box, status
//                  (generation.py:64-83, math3d.py:45-53,168-179)
//   k_faces        per (env, face): grid-frame corners, AABB cull, face_contacts
//                  (generation.py:70-96, contacts/_kernels.py:11-87)
//   k_compact      per env: ordered compaction of found faces + world-frame
//                  epilogue (generation.py:98-114)
//   k_face_contacts / k_sdf_sample / k_sdf_gradient: per-pair drop-ins for the
//                  reference's numba kernels.
#include "cs_generate.cuh"

namespace cs {

__device__ __forceinline__ void quat_to_matrix(const double *q, double *R) {
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

__global__ void k_env_xf(int64_t E, const int32_t *__restrict__ env_sdf, const int32_t *__restrict__ env_mesh,
                         const SdfDesc *__restrict__ sdfs, const double *__restrict__ sdf_pose,
                         const double *__restrict__ mesh_pose, int pose_format, const double *__restrict__ cdv,
                         EnvXf *__restrict__ xf, int32_t *__restrict__ env_status,
                         double *__restrict__ env_min_depth) {
    int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= E) return;
    double Rs[9], Rm[9], ts[3], tm[3];
    int ok = 1;
    if (pose_format == CS_POSE7) {
        const double *s = sdf_pose + 7 * e, *m = mesh_pose + 7 * e;
        quat_to_matrix(s + 3, Rs);
        quat_to_matrix(m + 3, Rm);
        for (int k = 0; k < 3; ++k) { ts[k] = s[k]; tm[k] = m[k]; }
    } else {
        const double *s = sdf_pose + 12 * e, *m = mesh_pose + 12 * e;
        for (int k = 0; k < 9; ++k) { Rs[k] = s[k]; Rm[k] = m[k]; }
        for (int k = 0; k < 3; ++k) { ts[k] = s[9 + k]; tm[k] = m[9 + k]; }
    }
    for (int k = 0; k < 9; ++k) ok &= isfinite(Rs[k]) && isfinite(Rm[k]);
    for (int k = 0; k < 3; ++k) ok &= isfinite(ts[k]) && isfinite(tm[k]);
    EnvXf X;
    // inverse (math3d.py:174-176): rt = Rs^T (F-contiguous view), ti = (-rt) @ ts
    double ti[3];
    for (int i = 0; i < 3; ++i) ti[i] = G3(-Rs[0 + i], -Rs[3 + i], -Rs[6 + i], ts[0], ts[1], ts[2]);
    // compose (math3d.py:178-179): R = rt @ Rm, t = rt @ tm + ti
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) X.R[3 * i + j] = G3(Rs[i], Rs[3 + i], Rs[6 + i], Rm[j], Rm[3 + j], Rm[6 + j]);
    for (int i = 0; i < 3; ++i) X.t[i] = G3(Rs[i], Rs[3 + i], Rs[6 + i], tm[0], tm[1], tm[2]) + ti[i];
    for (int k = 0; k < 9; ++k) X.Rs[k] = Rs[k];
    for (int k = 0; k < 3; ++k) X.ts[k] = ts[k];
    double cd = cdv[e];
    const SdfDesc &S = sdfs[env_sdf[e]];
    X.cd = cd;
    X.tol = 0.1 * S.voxel;  // CONVERGENCE_TOL_VOXELS * voxel (generation.py:20,91)
    double margin = cd + 2.0 * S.voxel;
    for (int k = 0; k < 3; ++k) { X.cull_lo[k] = S.lo[k] - margin; X.cull_hi[k] = S.hi[k] + margin; }
    X.status = ok ? (cd < 0.0 ? 2 : 0) : 1;
    X.sdf = env_sdf[e];
    X.mesh = env_mesh[e];
    X.pad = 0;
    xf[e] = X;
    env_status[e] = X.status;
    if (env_min_depth) env_min_depth[e] = -cd;
}

__device__ __forceinline__ double4 ld_vert(const double4 *p) {
    const double2 *q = reinterpret_cast<const double2 *>(p);
    double2 a = __ldg(q), b = __ldg(q + 1);
    return make_double4(a.x, a.y, b.x, b.y);
}

// verts_grid = to_grid.apply(vertices) (math3d.py:168-169): (V,3) @ R.T + t, V >= 2 -> G3
__device__ __forceinline__ double3 to_grid(const EnvXf &X, double4 v) {
    double3 r;
    r.x = G3(v.x, v.y, v.z, X.R[0], X.R[1], X.R[2]) + X.t[0];
    r.y = G3(v.x, v.y, v.z, X.R[3], X.R[4], X.R[5]) + X.t[1];
    r.z = G3(v.x, v.y, v.z, X.R[6], X.R[7], X.R[8]) + X.t[2];
    return r;
}

// UNIFORM: every env of the plan samples the same SDF, passed by value so its
// scalars are constant-bank operands; otherwise the env's SDF view is staged in
// shared memory per block.
template <bool COUNT, bool UNIFORM>
__global__ void __launch_bounds__(FACE_BLOCK) k_faces(const int2 *__restrict__ block_map, const EnvXf *__restrict__ xf,
                                                      const SdfDesc *__restrict__ sdfs,
                                                      const MeshDesc *__restrict__ meshes,
                                                      const int64_t *__restrict__ cand_base, Staging st,
                                                      unsigned long long *__restrict__ counter,
                                                      const GridT<double> gu) {
    __shared__ EnvXf sx;
    __shared__ GridT<double> sg;
    int2 bm = block_map[blockIdx.x];
    int e = bm.x;
    if (threadIdx.x < sizeof(EnvXf) / 8)
        reinterpret_cast<double *>(&sx)[threadIdx.x] = reinterpret_cast<const double *>(xf + e)[threadIdx.x];
    __syncthreads();
    if (!UNIFORM) {
        static_assert(sizeof(GridT<double>) % 8 == 0 && sizeof(GridT<double>) / 8 <= FACE_BLOCK, "GridT copy");
        if (threadIdx.x < sizeof(GridT<double>) / 8)
            reinterpret_cast<double *>(&sg)[threadIdx.x] = reinterpret_cast<const double *>(&sdfs[sx.sdf].g64)[threadIdx.x];
        __syncthreads();
    }
    const GridT<double> &grid = UNIFORM ? gu : sg;
    const MeshDesc M = meshes[sx.mesh];
    const int64_t f = (int64_t)bm.y + threadIdx.x;
    bool found = false;
    FaceResult r;
    if (f < M.nt && sx.status == 0) {
        int4 tri = __ldg(M.tris + f);
        double3 a = to_grid(sx, ld_vert(M.verts + tri.x));
        double3 b = to_grid(sx, ld_vert(M.verts + tri.y));
        double3 c = to_grid(sx, ld_vert(M.verts + tri.z));
        // AABB cull (generation.py:74-83)
        bool near = dmin(dmin(a.x, b.x), c.x) <= sx.cull_hi[0] && dmax(dmax(a.x, b.x), c.x) >= sx.cull_lo[0] &&
                    dmin(dmin(a.y, b.y), c.y) <= sx.cull_hi[1] && dmax(dmax(a.y, b.y), c.y) >= sx.cull_lo[1] &&
                    dmin(dmin(a.z, b.z), c.z) <= sx.cull_hi[2] && dmax(dmax(a.z, b.z), c.z) >= sx.cull_lo[2];
        if (near) {
            bool computed = face_body<COUNT>(grid, a.x, a.y, a.z, b.x, b.y, b.z, c.x, c.y, c.z, sx.cd,
                                             MAX_MINIMIZE_ITERS, sx.tol, r);
            if (COUNT) atomicAdd(counter, (unsigned long long)r.nsamp);
            found = computed && r.phi <= sx.cd;
        }
    }
    // chunk-local ordered compaction: this block's found faces land at the start of
    // its staging rows in ascending face order; k_compact stitches the chunks.
    __shared__ int ws[WS_INTS];
    int total;
    const int pos = block_excl_scan(found ? 1 : 0, ws, &total);
    if (found) {
        const int64_t s = cand_base[e] + bm.y + pos;
        st.point[3 * s + 0] = r.px;
        st.point[3 * s + 1] = r.py;
        st.point[3 * s + 2] = r.pz;
        st.phi[s] = r.phi;
        st.grad[3 * s + 0] = r.gx;
        st.grad[3 * s + 1] = r.gy;
        st.grad[3 * s + 2] = r.gz;
        st.face[s] = (int32_t)f;
    }
    if (threadIdx.x == 0) st.chunk_count[blockIdx.x] = total;
}

// Stitch the per-chunk compacted rows into the env's candidate list (ascending
// face order) and apply the world-frame epilogue (generation.py:98-114).
// One CTA per env: chunk offsets by a block scan, then one warp per chunk.
__global__ void __launch_bounds__(COMPACT_BLOCK) k_compact(const EnvXf *__restrict__ xf,
                                                           const int64_t *__restrict__ cand_base,
                                                           const int2 *__restrict__ block_map,
                                                           const int32_t *__restrict__ chunk_first, Staging st,
                                                           Candidates cs, int32_t *__restrict__ n_cand) {
    __shared__ int ws[WS_INTS];
    __shared__ EnvXf sx;
    const int e = blockIdx.x;
    if (threadIdx.x < sizeof(EnvXf) / 8)
        reinterpret_cast<double *>(&sx)[threadIdx.x] = reinterpret_cast<const double *>(xf + e)[threadIdx.x];
    const int c0 = chunk_first[e], nch = chunk_first[e + 1] - c0;
    const int64_t base = cand_base[e];
    int running = 0;
    for (int j0 = 0; j0 < nch; j0 += blockDim.x) {
        const int j = j0 + threadIdx.x;
        const int v = j < nch ? st.chunk_count[c0 + j] : 0;
        int tot;
        const int x = block_excl_scan(v, ws, &tot);
        if (j < nch) st.chunk_off[c0 + j] = running + x;
        running += tot;
    }
    __syncthreads();
    const int C = running;
    const bool gemm = C >= 2;  // the world transform's BLAS path (C >= 2 -> G3)
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int j = wid; j < nch; j += nw) {
        const int cnt = st.chunk_count[c0 + j];
        const int64_t src0 = base + block_map[c0 + j].y;
        const int64_t dst0 = base + st.chunk_off[c0 + j];
        for (int i = lane; i < cnt; i += 32) {
            const int64_t s = src0 + i, d = dst0 + i;
            double px = st.point[3 * s], py = st.point[3 * s + 1], pz = st.point[3 * s + 2];
            double gx = st.grad[3 * s], gy = st.grad[3 * s + 1], gz = st.grad[3 * s + 2];
            double nrm = sqrt(gx * gx + gy * gy + gz * gz);  // np.linalg.norm(axis=1): ((x2+y2)+z2)
            if (nrm < 1e-12) { gx = 0.0; gy = 0.0; gz = 1.0; nrm = 1.0; }
            const double nx = gx / nrm, ny = gy / nrm, nz = gz / nrm;
            for (int k = 0; k < 3; ++k) {
                const double *rr = sx.Rs + 3 * k;
                cs.normal[3 * d + k] = gemm ? G3(nx, ny, nz, rr[0], rr[1], rr[2]) : V3(nx, ny, nz, rr[0], rr[1], rr[2]);
                cs.point[3 * d + k] =
                    (gemm ? G3(px, py, pz, rr[0], rr[1], rr[2]) : V3(px, py, pz, rr[0], rr[1], rr[2])) + sx.ts[k];
            }
            cs.depth[d] = -st.phi[s];
            cs.face[d] = st.face[s];
        }
    }
    if (threadIdx.x == 0) n_cand[e] = C;
}

// ---------------------------------------------------------------- per-pair drop-ins

__global__ void k_face_contacts(GridView g, const double *__restrict__ tv, int64_t m, double cd, int max_iters,
                                double tol, double *__restrict__ op, double *__restrict__ ophi,
                                double *__restrict__ og, uint8_t *__restrict__ ofd) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= m) return;
    const double *p = tv + 9 * t;
    FaceResult r;
    if (!face_body(g, p[0], p[1], p[2], p[3], p[4], p[5], p[6], p[7], p[8], cd, max_iters, tol, r)) {
        ofd[t] = 0;
        return;
    }
    op[3 * t] = r.px; op[3 * t + 1] = r.py; op[3 * t + 2] = r.pz;
    ophi[t] = r.phi;
    og[3 * t] = r.gx; og[3 * t + 1] = r.gy; og[3 * t + 2] = r.gz;
    ofd[t] = (r.phi <= cd) ? 1 : 0;
}

__global__ void k_sdf_sample(GridView g, const double *__restrict__ p, int64_t n, double *__restrict__ out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) out[i] = sample(g, p[3 * i], p[3 * i + 1], p[3 * i + 2]);
}

__global__ void k_sdf_gradient(GridView g, const double *__restrict__ p, int64_t n, double *__restrict__ out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) gradient(g, p[3 * i], p[3 * i + 1], p[3 * i + 2], out[3 * i], out[3 * i + 1], out[3 * i + 2]);
}

// ---------------------------------------------------------------- launchers

void launch_env_xf(int64_t E, const int32_t *env_sdf, const int32_t *env_mesh, const SdfDesc *sdfs,
                   const double *sdf_pose, const double *mesh_pose, int pose_format, const double *cd, EnvXf *xf,
                   int32_t *env_status, double *env_min_depth, cudaStream_t s) {
    int bs = 128;
    k_env_xf<<<(unsigned)((E + bs - 1) / bs), bs, 0, s>>>(E, env_sdf, env_mesh, sdfs, sdf_pose, mesh_pose,
                                                          pose_format, cd, xf, env_status, env_min_depth);
}

void launch_faces(int64_t nblocks, const int2 *block_map, const EnvXf *xf, const SdfDesc *sdfs,
                  const MeshDesc *meshes, const int64_t *cand_base, const Staging &st, unsigned long long *counter,
                  const GridT<double> *uniform, cudaStream_t s) {
    if (nblocks <= 0) return;
    const GridT<double> gu = uniform ? *uniform : GridT<double>{};
    const unsigned nb = (unsigned)nblocks;
    if (uniform) {
        if (counter) k_faces<true, true><<<nb, FACE_BLOCK, 0, s>>>(block_map, xf, sdfs, meshes, cand_base, st, counter, gu);
        else k_faces<false, true><<<nb, FACE_BLOCK, 0, s>>>(block_map, xf, sdfs, meshes, cand_base, st, nullptr, gu);
    } else {
        if (counter) k_faces<true, false><<<nb, FACE_BLOCK, 0, s>>>(block_map, xf, sdfs, meshes, cand_base, st, counter, gu);
        else k_faces<false, false><<<nb, FACE_BLOCK, 0, s>>>(block_map, xf, sdfs, meshes, cand_base, st, nullptr, gu);
    }
}

void launch_compact(int64_t E, const EnvXf *xf, const int64_t *cand_base, const int2 *block_map,
                    const int32_t *chunk_first, const Staging &st, const Candidates &cs, int32_t *n_cand,
                    cudaStream_t s) {
    if (E > 0)
        k_compact<<<(unsigned)E, COMPACT_BLOCK, 0, s>>>(xf, cand_base, block_map, chunk_first, st, cs, n_cand);
}

void launch_face_contacts(const GridView &g, const double *tv, int64_t m, double cd, int max_iters, double tol,
                          double *op, double *ophi, double *og, uint8_t *ofd, cudaStream_t s) {
    int bs = 128;
    if (m > 0)
        k_face_contacts<<<(unsigned)((m + bs - 1) / bs), bs, 0, s>>>(g, tv, m, cd, max_iters, tol, op, ophi, og, ofd);
}

void launch_sdf_sample(const GridView &g, const double *p, int64_t n, double *out, cudaStream_t s) {
    int bs = 256;
    if (n > 0) k_sdf_sample<<<(unsigned)((n + bs - 1) / bs), bs, 0, s>>>(g, p, n, out);
}

void launch_sdf_gradient(const GridView &g, const double *p, int64_t n, double *out, cudaStream_t s) {
    int bs = 256;
    if (n > 0) k_sdf_gradient<<<(unsigned)((n + bs - 1) / bs), bs, 0, s>>>(g, p, n, out);
}

}  // namespace cs
