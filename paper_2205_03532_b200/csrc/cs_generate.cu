// Contact generation on sm_100a.
//
//   k_env_xf       per env: poses -> to_grid transform, cull box, status
//                  (generation.py:64-83, math3d.py:45-53,168-179)
//   k_face_prep    per (env, chunk): grid-frame vertices, AABB cull, Lipschitz
//                  prune, descent start (generation.py:70-96, contacts/_kernels.py:20-43)
//   k_pgd_grad / k_pgd_first / k_pgd_rest: the projected-gradient descent
//                  (contacts/_kernels.py:44-87) as a wavefront over the survivors
//   k_compact      per env: ordered compaction of found faces + world-frame
//                  epilogue (generation.py:98-114)
//   k_face_contacts / k_sdf_sample / k_sdf_gradient: per-pair drop-ins for the
//                  reference's numba kernels.
#include <algorithm>

#include "cs_generate.cuh"

namespace cs {

__global__ void k_env_xf(int64_t E, const int32_t *__restrict__ env_sdf, const int32_t *__restrict__ env_mesh,
                         const SdfDesc *__restrict__ sdfs, const double *__restrict__ sdf_pose,
                         const double *__restrict__ mesh_pose, int pose_format, const double *__restrict__ cdv,
                         EnvXf *__restrict__ xf, int32_t *__restrict__ env_status,
                         double *__restrict__ env_min_depth, unsigned *__restrict__ work_count,
                         const int32_t *__restrict__ active) {
    int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e == 0 && work_count) { work_count[0] = 0; work_count[1] = 0; work_count[2] = 0; work_count[3] = 0; }
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
    // an inactive pair slot (active[e] == 0: no broadphase overlap this step) generates
    // nothing and its pose is not validated
    X.status = (active && !active[e]) ? 3 : (ok ? (cd < 0.0 ? 2 : 0) : 1);
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

#ifdef PREP_STATS
#define PREP_PROF
#define PREP_CONST
#else
#define PREP_CONST const
#endif
#ifdef PREP_PROF
__device__ unsigned long long g_prep_prof[16];
#define PREP_MARK(i) do { if (threadIdx.x == 0) { const long long t_ = clock64(); atomicAdd(&g_prep_prof[i], (unsigned long long)(t_ - t_last)); t_last = t_; } } while (0)
extern "C" int cs_debug_prep_prof(unsigned long long *out) { return (int)cudaMemcpyFromSymbol(out, g_prep_prof, sizeof(g_prep_prof)); }
#ifdef PREP_STATS
extern "C" int cs_debug_bound_stat(unsigned long long *out) { return (int)cudaMemcpyFromSymbol(out, g_bound_stat, sizeof(g_bound_stat)); }
#endif
#else
#define PREP_MARK(i) do {} while (0)
#endif
#ifdef BOX_STATS
__device__ unsigned long long g_box_stat[8];  // chunks, sum of box cells, boxes <= 4k / 8k / 16k cells, samples
extern "C" int cs_debug_box_stat(unsigned long long *out) { return (int)cudaMemcpyFromSymbol(out, g_box_stat, sizeof(g_box_stat)); }
#endif
constexpr int FACE_ITEM = 1 << 30;  // sample-list code of a face centre (else a vertex slot)

// k_face_prep: one CTA per (env, chunk of FACE_CHUNK faces). The chunk's distinct
// vertices are transformed and (where a face needs them) sampled once into shared
// memory; each thread then culls one face (generation.py:74-83), applies the
// Lipschitz prune and picks the descent start (contacts/_kernels.py:28-43). The
// survivors are appended, in face order within the chunk, to a dense work list.
// UNIFORM: every env of the plan samples the same SDF, passed by value so its
// scalars are constant-bank operands; otherwise the env's grid view is staged in
// shared memory.
template <bool COUNT, bool UNIFORM>
__global__ void __launch_bounds__(FACE_CHUNK, PREP_MINB) k_face_prep(const int4 *__restrict__ prep_map,
                                                          const EnvXf *__restrict__ xf,
                                                          const SdfDesc *__restrict__ sdfs,
                                                          const MeshDesc *__restrict__ meshes,
                                                          const int64_t *__restrict__ cand_base, Staging st, int maxcv,
                                                          unsigned long long *__restrict__ counter,
                                                          const PlanGrid gu,
                                                          const MeshDesc mu, int um) {
    extern __shared__ double dsm[];
    __shared__ EnvXf sx;
    __shared__ PlanGrid sg;
    __shared__ int ws[WS_INTS];
    __shared__ unsigned sbase;
#ifdef PREP_PROF
    long long t_last = clock64();
#endif
    // (env, first face, chunk vertex offset, vertex count | mesh << 16): the mesh and
    // chunk loads below need not wait for the env's transform
    const int4 bm = prep_map[blockIdx.x];
    const int e = bm.x, f0 = bm.y, v0 = bm.z, ncv = bm.w & 0xffff, mesh = bm.w >> 16;
    const MeshDesc &M = um ? mu : meshes[mesh];  // uniform-mesh plans: a kernel parameter
    const double4 *verts = M.verts;
    const int32_t *cverts = M.chunk_verts;
    const int64_t nt = M.nt;
    const uint2 *face_loc = M.face_loc;
    if (threadIdx.x < sizeof(EnvXf) / 8)
        reinterpret_cast<double *>(&sx)[threadIdx.x] = reinterpret_cast<const double *>(xf + e)[threadIdx.x];
    __syncthreads();
    PREP_MARK(0);
    if (sx.status != 0) {  // non-finite pose or cd < 0: nothing is generated
        if (threadIdx.x == 0) { st.chunk_count[blockIdx.x] = 0; st.chunk_found[blockIdx.x] = 0; }
        return;
    }
    if (!UNIFORM) {
        static_assert(sizeof(PlanGrid) % 8 == 0 && sizeof(PlanGrid) / 8 <= FACE_CHUNK, "grid view copy");
        if (threadIdx.x < sizeof(PlanGrid) / 8)
            reinterpret_cast<double *>(&sg)[threadIdx.x] = reinterpret_cast<const double *>(&sdfs[sx.sdf].gp)[threadIdx.x];
    }
    const PlanGrid &grid = UNIFORM ? gu : sg;
    // shared: vertex x/y/z/phi [maxcv], centre phi [FACE_CHUNK], face corner slots
    // [FACE_CHUNK], the sample list [maxcv + FACE_CHUNK], vertex flags [maxcv]
    double *vx = dsm, *vy = dsm + maxcv, *vz = dsm + 2 * maxcv, *vphi = dsm + 3 * maxcv, *cphi = dsm + 4 * maxcv;
    uint2 *sloc = reinterpret_cast<uint2 *>(cphi + FACE_CHUNK);
    int *list = reinterpret_cast<int *>(sloc + FACE_CHUNK);
    unsigned char *need = reinterpret_cast<unsigned char *>(list + maxcv + FACE_CHUNK);
    __shared__ int s_nl;
    const int64_t f = (int64_t)f0 + threadIdx.x;
    const uint2 loc = f < nt ? __ldg(face_loc + f) : make_uint2(0, 0);  // in flight during the transform
    // verts_grid = to_grid.apply(vertices) (generation.py:70), per distinct vertex
    for (int j = threadIdx.x; j < ncv; j += FACE_CHUNK) {
        const double3 p = to_grid(sx, ld_vert(verts + __ldg(cverts + v0 + j)));
        vx[j] = p.x; vy[j] = p.y; vz[j] = p.z;
        need[j] = 0;
    }
    if (threadIdx.x == 0) s_nl = 0;
    __syncthreads();
    PREP_MARK(1);
    const int lane = threadIdx.x & 31;
    int la = 0, lb = 0, lc = 0;
    bool near = false;
#ifdef PREP_STATS
    bool bcull = false;
#endif
    if (f < nt) {
        sloc[threadIdx.x] = loc;
        la = (int)(loc.x & 0xffffu); lb = (int)(loc.x >> 16); lc = (int)loc.y;
        const double ax = vx[la], bx = vx[lb], cx = vx[lc];
        const double ay = vy[la], by = vy[lb], cy = vy[lc];
        const double az = vz[la], bz = vz[lb], cz = vz[lc];
        const double lo[3] = {dmin(dmin(ax, bx), cx), dmin(dmin(ay, by), cy), dmin(dmin(az, bz), cz)};
        const double hi[3] = {dmax(dmax(ax, bx), cx), dmax(dmax(ay, by), cy), dmax(dmax(az, bz), cz)};
        near = lo[0] <= sx.cull_hi[0] && hi[0] >= sx.cull_lo[0] && lo[1] <= sx.cull_hi[1] && hi[1] >= sx.cull_lo[1] &&
               lo[2] <= sx.cull_hi[2] && hi[2] >= sx.cull_lo[2];
        // Every sample that can become the face's phi lies on the triangle, inside its
        // box; when the grid is provably above cd there, the reference ends with
        // found = 0 (prune or descent), so the face is not descended at all (exact:
        // only a proof skips).
#ifdef PREP_STATS
        bcull = near && grid.cwin && sample_lower_bound(grid, lo, hi, sx.cd) > sx.cd;
        atomicAdd(&g_prep_prof[8], 1ull);
        if (near) atomicAdd(&g_prep_prof[9], 1ull);
        if (bcull) atomicAdd(&g_prep_prof[10], 1ull);
#else
        if (near && grid.cwin && sample_lower_bound(grid, lo, hi, sx.cd) > sx.cd) near = false;
#endif
        if (near) { need[la] = 1; need[lb] = 1; need[lc] = 1; }
    }
    {   // near faces queue their centre sample
        const unsigned b = __ballot_sync(0xffffffffu, near);
        int base = 0;
        if (lane == 0 && b) base = atomicAdd(&s_nl, __popc(b));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (near) list[base + __popc(b & ((1u << lane) - 1))] = FACE_ITEM | threadIdx.x;
    }
    __syncthreads();
    PREP_MARK(2);
    for (int j0 = threadIdx.x & ~31; j0 < ncv; j0 += FACE_CHUNK) {  // needed vertices queue theirs
        const int j = j0 + lane;
        const bool q = j < ncv && need[j];
        const unsigned b = __ballot_sync(0xffffffffu, q);
        int base = 0;
        if (lane == 0 && b) base = atomicAdd(&s_nl, __popc(b));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (q) list[base + __popc(b & ((1u << lane) - 1))] = j;
    }
    __syncthreads();
    PREP_MARK(3);
    // One dense pass over the queued samples: every needed vertex (phi at the vertices,
    // generation.py:92) and the centre of every near face (the centroid start point;
    // only used when the face survives the Lipschitz prune below).
    const int nl = s_nl;
#ifdef BOX_STATS
    {   // the chunk's sample box (cells of every queued sample): could it be staged in shared memory?
        __shared__ int bb[6];
        if (threadIdx.x < 3) { bb[threadIdx.x] = INT_MAX; bb[3 + threadIdx.x] = INT_MIN; }
        __syncthreads();
        for (int i = threadIdx.x; i < nl; i += FACE_CHUNK) {
            const int code = list[i];
            double px, py, pz;
            if (code & FACE_ITEM) {
                const uint2 loc = sloc[code & 0xffff];
                const int a = (int)(loc.x & 0xffffu), b = (int)(loc.x >> 16), c = (int)loc.y;
                px = div3(vx[a] + vx[b] + vx[c]); py = div3(vy[a] + vy[b] + vy[c]); pz = div3(vz[a] + vz[b] + vz[c]);
            } else {
                px = vx[code]; py = vy[code]; pz = vz[code];
            }
            const GPoint q = gpoint(grid, px, py, pz);
            atomicMin(bb + 0, q.ax.i); atomicMin(bb + 1, q.ay.i); atomicMin(bb + 2, q.az.i);
            atomicMax(bb + 3, q.ax.i); atomicMax(bb + 4, q.ay.i); atomicMax(bb + 5, q.az.i);
        }
        __syncthreads();
        if (threadIdx.x == 0 && nl > 0) {
            const long long V = (long long)(bb[3] - bb[0] + 2) * (bb[4] - bb[1] + 2) * (bb[5] - bb[2] + 2);
            atomicAdd(&g_box_stat[0], 1ull);
            atomicAdd(&g_box_stat[1], (unsigned long long)V);
            if (V <= 4096) atomicAdd(&g_box_stat[2], 1ull);
            if (V <= 8192) atomicAdd(&g_box_stat[3], 1ull);
            if (V <= 16384) atomicAdd(&g_box_stat[4], 1ull);
            atomicAdd(&g_box_stat[5], (unsigned long long)nl);
        }
    }
#endif
    for (int i = threadIdx.x; i < nl; i += FACE_CHUNK) {
        const int code = list[i];
        double px, py, pz;
        if (code & FACE_ITEM) {
            const uint2 loc = sloc[code & 0xffff];
            const int a = (int)(loc.x & 0xffffu), b = (int)(loc.x >> 16), c = (int)loc.y;
            px = div3(vx[a] + vx[b] + vx[c]);
            py = div3(vy[a] + vy[b] + vy[c]);
            pz = div3(vz[a] + vz[b] + vz[c]);
        } else {
            px = vx[code]; py = vy[code]; pz = vz[code];
        }
        const double r = sample(grid, px, py, pz);
        if (code & FACE_ITEM) cphi[code & 0xffff] = r;
        else vphi[code] = r;
    }
    __syncthreads();
    PREP_MARK(4);
    int ns = 0;
    if (COUNT)
        for (int j = threadIdx.x; j < ncv; j += FACE_CHUNK) ns += need[j];
    bool survive = false;
    int which = 0;
    double pa = 0.0, pb = 0.0, pc = 0.0, ps = 0.0;
    if (near) {
        const double ax = vx[la], ay = vy[la], az = vz[la];
        const double bx = vx[lb], by = vy[lb], bz = vz[lb];
        const double cx = vx[lc], cy = vy[lc], cz = vz[lc];
        pa = vphi[la]; pb = vphi[lb]; pc = vphi[lc];
        // max of the three edge lengths (contacts/_kernels.py:30-33): sqrt is correctly rounded and
        // monotone, so the max of the roots is the root of the max (one sqrt instead of three)
        const double s0 = (bx - ax) * (bx - ax) + (by - ay) * (by - ay) + (bz - az) * (bz - az);
        const double s1 = (cx - bx) * (cx - bx) + (cy - by) * (cy - by) + (cz - bz) * (cz - bz);
        const double s2 = (ax - cx) * (ax - cx) + (ay - cy) * (ay - cy) + (az - cz) * (az - cz);
        const double diam = sqrt(dmax(s0, dmax(s1, s2)));
        PREP_CONST double phi_min = dmin(pa, dmin(pb, pc));
#ifdef PREP_STATS
        const bool pcull = phi_min - diam > sx.cd;
        if (pcull) atomicAdd(&g_prep_prof[11], 1ull);
        if (pcull && bcull) atomicAdd(&g_prep_prof[12], 1ull);
        if (!pcull && !bcull) atomicAdd(&g_prep_prof[13], 1ull);
        if (bcull) phi_min = sx.cd + diam + 1.0;
#endif
        if (!(phi_min - diam > sx.cd)) {
            ps = cphi[threadIdx.x];
            ++ns;
            if (pa < ps) { ps = pa; which = 1; }
            if (pb < ps) { ps = pb; which = 2; }
            if (pc < ps) { ps = pc; which = 3; }
            survive = true;
        }
    }
    if (COUNT) {
        for (int o = 16; o; o >>= 1) ns += __shfl_xor_sync(0xffffffffu, ns, o);
        if ((threadIdx.x & 31) == 0 && ns) atomicAdd(counter, (unsigned long long)ns);
    }
#if GROUP_STARTS
    // Survivors' staging rows follow face order (rank among the chunk's survivors: the
    // compaction reads them in order); their work-list slots are grouped by start
    // (centroid, corner a, b, c) so the descent's warps mostly see one kind of start.
    int total, pos, slot;
    {
        __shared__ int wc[FACE_CHUNK / 32][4];
        const unsigned lt = (1u << lane) - 1u;
        const unsigned m0 = __ballot_sync(0xffffffffu, survive && which == 0);
        const unsigned m1 = __ballot_sync(0xffffffffu, survive && which == 1);
        const unsigned m2 = __ballot_sync(0xffffffffu, survive && which == 2);
        const unsigned m3 = __ballot_sync(0xffffffffu, survive && which == 3);
        const int wid = threadIdx.x >> 5;
        if (lane < 4) wc[wid][lane] = __popc(lane == 0 ? m0 : (lane == 1 ? m1 : (lane == 2 ? m2 : m3)));
        __syncthreads();
        int before = 0, before_w = 0, tot_w = 0, cat_off = 0;
        total = 0;
#pragma unroll
        for (int w = 0; w < FACE_CHUNK / 32; ++w) {
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const int v = wc[w][c];
                total += v;
                if (w < wid) before += v;
                if (c == which) { tot_w += v; if (w < wid) before_w += v; }
                else if (c < which) cat_off += v;
            }
        }
        const unsigned mw = which == 0 ? m0 : (which == 1 ? m1 : (which == 2 ? m2 : m3));
        pos = before + __popc((m0 | m1 | m2 | m3) & lt);
        slot = cat_off + before_w + __popc(mw & lt);
        (void)tot_w;
    }
#else
    int total;
    const int pos = block_excl_scan(survive ? 1 : 0, ws, &total);
    const int slot = pos;
#endif
    if (threadIdx.x == 0) {
        sbase = total ? atomicAdd(st.work_count, (unsigned)total) : 0u;
        st.chunk_count[blockIdx.x] = total;
        st.chunk_found[blockIdx.x] = 0;
    }
    __syncthreads();
    if (survive) {
        FaceWork *w = st.work + sbase + slot;
        // the record as three 16-byte stores
        reinterpret_cast<int4 *>(w)[0] =
            make_int4((int32_t)(cand_base[e] + f0 + pos), (int32_t)blockIdx.x, (int32_t)f | (which << 30), e);
        reinterpret_cast<double2 *>(w)[1] = make_double2(pa, pb);
        reinterpret_cast<double2 *>(w)[2] = make_double2(pc, ps);
    }
    PREP_MARK(5);
}

// ---------------------------------------------------------------- the descent as a wavefront
//
// contacts/_kernels.py:44-87 for every surviving face, as a sequence of uniform
// kernels over lists (the state -- point, phi, gradient, step -- lives in the face's
// staging row):
//   k_pgd_grad(stage 0)  gradient at the start point, every face
//   k_pgd_first          iteration 0 after its gradient: normalise, up to four
//                        backtracking projections; faces that do not move (or
//                        have a vanishing gradient) are done; moved faces go to
//                        the accepted list, flagged final when they moved less than
//                        the tolerance
//   k_pgd_grad(stage 1)  gradient at the moved point, accepted faces: the final
//                        gradient of the final ones, iteration 1's of the others
//   k_pgd_rest           the rest of the descent for the faces still moving (about
//                        1%), one thread each
// Same operations in the same order as the sequential loop; only the schedule
// differs (uniform work per kernel instead of one divergent state machine).

#ifndef GROUP_STARTS
#define GROUP_STARTS 1  // k_face_prep groups each chunk's work-list slots by start kind
#endif
#ifndef STUCK0
#define STUCK0 1  // stage 0 finishes the faces whose iteration 0 provably does not move (see k_pgd_grad)
#endif
#ifndef GRAD_ONE_VERT
#define GRAD_ONE_VERT 1  // stage 0: a corner start transforms only its own vertex
#endif
#ifndef PGD_FUSE_REST
#define PGD_FUSE_REST 0  // stage 1 and the rest of the descent in one kernel (k_pgd_grad1_rest)
#endif
#ifndef PGD_FUSE0
#define PGD_FUSE0 0  // iteration 0's gradient inside k_pgd_first (no stage-0 k_pgd_grad launch)
#endif

constexpr unsigned ACC_FINAL = 0x80000000u;  // accepted-list flag: the move ended the descent

__device__ __forceinline__ void finish_face(const Staging &st, int64_t row, int blk, int face, double phi, double cd) {
    const bool found = phi <= cd;  // contacts/_kernels.py:87
    if (found) atomicAdd(st.chunk_found + blk, 1);
    st.face[row] = found ? face : -1;
}

template <bool UNIFORM>
__device__ __forceinline__ const PlanGrid &grid_of(const PlanGrid &gu, const SdfDesc *sdfs, const EnvXf *xf, int e) {
    return UNIFORM ? gu : sdfs[xf[e].sdf].gp;
}

// The face's corners in the grid frame (generation.py:70-72), its vertex phis and start.
struct FaceGeom {
    double ax, ay, az, bx, by, bz, cx, cy, cz;
};

// um: every env of the plan uses mesh mu (a kernel parameter): the triangle and
// vertex loads then do not wait for the env's descriptor
__device__ __forceinline__ FaceGeom face_geom(const EnvXf &X, const MeshDesc *meshes, const MeshDesc &mu, int um,
                                              int face) {
    const int4 *tris;
    const double4 *verts;
    if (um) { tris = mu.tris; verts = mu.verts; }
    else { tris = meshes[X.mesh].tris; verts = meshes[X.mesh].verts; }
    const int4 tri = __ldg(tris + face);
    const double3 a = to_grid(X, ld_vert(verts + tri.x));
    const double3 b = to_grid(X, ld_vert(verts + tri.y));
    const double3 c = to_grid(X, ld_vert(verts + tri.z));
    return FaceGeom{a.x, a.y, a.z, b.x, b.y, b.z, c.x, c.y, c.z};
}

// The descent's start (contacts/_kernels.py:40-52): the centroid, or the corner k_face_prep chose.
__device__ __forceinline__ void face_start(const FaceGeom &f, int which, double &px, double &py, double &pz) {
    if (which == 0) {
        px = div3(f.ax + f.bx + f.cx); py = div3(f.ay + f.by + f.cy); pz = div3(f.az + f.bz + f.cz);
    } else if (which == 1) {
        px = f.ax; py = f.ay; pz = f.az;
    } else if (which == 2) {
        px = f.bx; py = f.by; pz = f.bz;
    } else {
        px = f.cx; py = f.cy; pz = f.cz;
    }
}

// True when all four backtracking projections of iteration 0 (alpha = voxel, /2, /4, /8)
// return the corner p itself. closest_point's first three region tests (corner a,
// corner b, edge ab, then corner c) with every dot product evaluated for every lane,
// each with closest_point's own expression (so the same bits), and the outcome
// selected without branches: the four tries cost the same on every lane of a warp.
//
// With the starts grouped (GROUP_STARTS) a warp mostly holds one start corner, and
// only the tests that decide it are evaluated: corner a stays iff closest_point takes
// its first branch (it returns a == p); corner b iff the first fails and the second
// holds; corner c needs all four. (A later branch returning a corner bitwise equal
// to p -- a degenerate triangle -- is left to k_pgd_first: conservative.)
__device__ __forceinline__ bool corner_stays_which(const FaceGeom &f, int which, double px, double py, double pz,
                                                   double ux, double uy, double uz, double alpha) {
    const double abx = f.bx - f.ax, aby = f.by - f.ay, abz = f.bz - f.az;
    const double acx = f.cx - f.ax, acy = f.cy - f.ay, acz = f.cz - f.az;
    bool stays = true;
    for (int bt = 0; bt < 4 && stays; ++bt) {
        const double qx = px - alpha * ux, qy = py - alpha * uy, qz = pz - alpha * uz;
        const double apx = qx - f.ax, apy = qy - f.ay, apz = qz - f.az;
        const double d1 = abx * apx + aby * apy + abz * apz;
        const double d2 = acx * apx + acy * apy + acz * apz;
        const bool ra = d1 <= 0.0 && d2 <= 0.0;
        if (which == 1) {
            stays = ra;
        } else {
            const double bpx = qx - f.bx, bpy = qy - f.by, bpz = qz - f.bz;
            const double d3 = abx * bpx + aby * bpy + abz * bpz;
            const double d4 = acx * bpx + acy * bpy + acz * bpz;
            const bool rb = d3 >= 0.0 && d4 <= d3;
            if (which == 2) {
                stays = !ra && rb;
            } else {
                const double vc = d1 * d4 - d3 * d2;
                const double cpx = qx - f.cx, cpy = qy - f.cy, cpz = qz - f.cz;
                const double d5 = abx * cpx + aby * cpy + abz * cpz;
                const double d6 = acx * cpx + acy * cpy + acz * cpz;
                const bool eab = vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0;
                const bool rc = d6 >= 0.0 && d5 <= d6;
                stays = !ra && !rb && !eab && rc;
            }
        }
        alpha *= 0.5;
    }
    return stays;
}

__device__ __forceinline__ bool corner_stays(const FaceGeom &f, double px, double py, double pz, double ux,
                                             double uy, double uz, double alpha) {
    const double abx = f.bx - f.ax, aby = f.by - f.ay, abz = f.bz - f.az;
    const double acx = f.cx - f.ax, acy = f.cy - f.ay, acz = f.cz - f.az;
    bool stays = true;
    for (int bt = 0; bt < 4 && stays; ++bt) {
        const double qx = px - alpha * ux, qy = py - alpha * uy, qz = pz - alpha * uz;
        const double apx = qx - f.ax, apy = qy - f.ay, apz = qz - f.az;
        const double d1 = abx * apx + aby * apy + abz * apz;
        const double d2 = acx * apx + acy * apy + acz * apz;
        const double bpx = qx - f.bx, bpy = qy - f.by, bpz = qz - f.bz;
        const double d3 = abx * bpx + aby * bpy + abz * bpz;
        const double d4 = acx * bpx + acy * bpy + acz * bpz;
        const double vc = d1 * d4 - d3 * d2;
        const double cpx = qx - f.cx, cpy = qy - f.cy, cpz = qz - f.cz;
        const double d5 = abx * cpx + aby * cpy + abz * cpz;
        const double d6 = acx * cpx + acy * cpy + acz * cpz;
        const bool ra = d1 <= 0.0 && d2 <= 0.0;
        const bool rb = d3 >= 0.0 && d4 <= d3;
        const bool eab = vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0;
        const bool rc = d6 >= 0.0 && d5 <= d6;
        // the corner closest_point returns (a, b, c in test order), if any
        const int r = ra ? 1 : (rb ? 2 : (eab ? 0 : (rc ? 3 : 0)));
        const double vx = r == 1 ? f.ax : (r == 2 ? f.bx : f.cx);
        const double vy = r == 1 ? f.ay : (r == 2 ? f.by : f.cy);
        const double vz = r == 1 ? f.az : (r == 2 ? f.bz : f.cz);
        stays = r != 0 && same3(vx, vy, vz, px, py, pz);
        alpha *= 0.5;
    }
    return stays;
}

template <bool COUNT, bool UNIFORM>
__global__ void __launch_bounds__(256, UNIFORM ? GRAD_MINB : GRAD_MINB_NU) k_pgd_grad(const int2 *__restrict__ block_map, const EnvXf *__restrict__ xf,
                                                  const SdfDesc *__restrict__ sdfs, const MeshDesc *__restrict__ meshes,
                                                  Staging st, int stage,
                                                  unsigned long long *__restrict__ counter, const PlanGrid gu,
                                                  const MeshDesc mu, int um) {
    const unsigned n = stage == 0 ? st.work_count[0] : st.work_count[2];
    unsigned long long ns = 0;
    for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        unsigned idx = i, flag = 0;
        int4 hd;  // row, blk, face, env: from the record, or (moved faces) beside the index
        if (stage == 1) {
            const unsigned a = st.acc[i];
            hd = st.acc_hd[i];
            idx = a & ~ACC_FINAL;
            flag = a & ACC_FINAL;
        } else {
            hd = __ldg(reinterpret_cast<const int4 *>(st.work + idx));
        }
        const int64_t row = hd.x;
        const int blk = hd.y;
        const int e = hd.w;
        const PlanGrid &g = grid_of<UNIFORM>(gu, sdfs, xf, e);
        double px, py, pz;
        if (stage == 0) {  // the start point, from the corners (not staged: recomputing is cheaper than the traffic)
            const int which = (int)((unsigned)hd.z >> 30), face = hd.z & 0x3fffffff;
#if GRAD_ONE_VERT
            if (which != 0) {  // a corner start (91% of the faces): only that vertex, same to_grid rounding
                const EnvXf &X = xf[e];
                const int4 tri = __ldg((um ? mu.tris : meshes[X.mesh].tris) + face);
                const int vi = which == 1 ? tri.x : (which == 2 ? tri.y : tri.z);
                const double3 q = to_grid(X, ld_vert((um ? mu.verts : meshes[X.mesh].verts) + vi));
                px = q.x; py = q.y; pz = q.z;
            } else
#endif
                face_start(face_geom(xf[e], meshes, mu, um, face), which, px, py, pz);
        } else {
            px = st.point[3 * row]; py = st.point[3 * row + 1]; pz = st.point[3 * row + 2];
        }
        double gx, gy, gz;
        gradient(g, px, py, pz, gx, gy, gz);
        if (COUNT) ns += 6;
        st.grad[3 * row] = gx; st.grad[3 * row + 1] = gy; st.grad[3 * row + 2] = gz;
#if STUCK0 && !PGD_FUSE0
        if (stage == 0) {
            // Iteration 0 without k_pgd_first when it provably leaves the face where it is:
            // a vanishing gradient, or a corner start whose four backtracking projections
            // (contacts/_kernels.py:64-75, the same operations as backtrack()) all return the
            // corner itself -- then every try's phi equals the current phi (no sample) and
            // none is accepted. 78% of the descended faces; the rest go to k_pgd_first's list.
            const int which = (int)((unsigned)hd.z >> 30);
            const double gnorm = sqrt(gx * gx + gy * gy + gz * gz);
            bool stuck = gnorm < 1e-12;
            if (!stuck && which != 0) {
                const double rg = 1.0 / gnorm;
                const double ux = div_rn(gx, gnorm, rg), uy = div_rn(gy, gnorm, rg), uz = div_rn(gz, gnorm, rg);
                const FaceGeom f = face_geom(xf[e], meshes, mu, um, hd.z & 0x3fffffff);
                stuck = GROUP_STARTS ? corner_stays_which(f, which, px, py, pz, ux, uy, uz, g.voxel)
                                     : corner_stays(f, px, py, pz, ux, uy, uz, g.voxel);
            }
            const unsigned bal = __ballot_sync(__activemask(), !stuck);
            if (stuck) {  // k_pgd_first's no-move branch
                const double phi = __ldg(st.work[idx].phi + 3);
                const double cd = xf[e].cd;
                if (phi <= cd) {
                    st.point[3 * row] = px; st.point[3 * row + 1] = py; st.point[3 * row + 2] = pz; st.phi[row] = phi;
                }
                finish_face(st, row, blk, hd.z & 0x3fffffff, phi, cd);
            } else {  // k_pgd_first's list (warp-aggregated append)
                const unsigned lane = threadIdx.x & 31, lead = __ffs(bal) - 1;
                unsigned b0 = 0;
                if (lane == lead) b0 = atomicAdd(st.work_count + 1, (unsigned)__popc(bal));
                b0 = __shfl_sync(bal, b0, lead);
                st.slow[b0 + __popc(bal & ((1u << lane) - 1u))] = idx;
            }
        }
#endif
        if (stage == 1) {
            if (flag) finish_face(st, row, blk, hd.z & 0x3fffffff, st.phi[row], xf[e].cd);
            else st.slow[atomicAdd(st.work_count + 3, 1u)] = idx;
        }
    }
    if (COUNT) {
        for (int o = 16; o; o >>= 1) ns += __shfl_xor_sync(0xffffffffu, ns, o);
        if ((threadIdx.x & 31) == 0 && ns) atomicAdd(counter, ns);
    }
}

// One backtracking search (contacts/_kernels.py:64-75) from (p, phi) along -g/|g|.
// Returns true on an accepted move (p, phi, alpha updated, moved set).
#ifdef BT_STATS
__device__ unsigned long long g_bt_stat[16];  // accepted at try 0..3, no move, known projections, sampled; [8..]: k_pgd_first by start
extern "C" int cs_debug_bt_stat(unsigned long long *out) { return (int)cudaMemcpyFromSymbol(out, g_bt_stat, sizeof(g_bt_stat)); }
#define BT_STAT(i) atomicAdd(&g_bt_stat[i], 1ull)
#else
#define BT_STAT(i) ((void)0)
#endif

template <bool COUNT, class G>
__device__ __forceinline__ bool backtrack(const G &g, const FaceGeom &f, const double *vphi, double gx, double gy,
                                          double gz, double gnorm, double &px, double &py, double &pz, double &phi,
                                          double &alpha, double &moved, unsigned long long &ns) {
    // gnorm = sqrt(gx gx + gy gy + gz gz): the caller's (it tested it against 1e-12)
    // g / gnorm, correctly rounded: one reciprocal for the three (div_rn proves each
    // quotient or falls back to the IEEE division)
    const double rg = 1.0 / gnorm;
    const double ux = div_rn(gx, gnorm, rg), uy = div_rn(gy, gnorm, rg), uz = div_rn(gz, gnorm, rg);
    for (int bt = 0; bt < 4; ++bt) {
        double qx, qy, qz;
        closest_point(f.ax, f.ay, f.az, f.bx, f.by, f.bz, f.cx, f.cy, f.cz, px - alpha * ux, py - alpha * uy,
                      pz - alpha * uz, qx, qy, qz);
        // the projection often is the current point or a corner itself: identical
        // inputs, so the sample's value is already known
        double phi_new;
        if (same3(qx, qy, qz, px, py, pz)) { phi_new = phi; BT_STAT(5); BT_STAT(12); }
        else if (same3(qx, qy, qz, f.ax, f.ay, f.az)) { phi_new = __ldg(vphi); BT_STAT(5); }
        else if (same3(qx, qy, qz, f.bx, f.by, f.bz)) { phi_new = __ldg(vphi + 1); BT_STAT(5); }
        else if (same3(qx, qy, qz, f.cx, f.cy, f.cz)) { phi_new = __ldg(vphi + 2); BT_STAT(5); }
        else {
            phi_new = sample(g, qx, qy, qz);
            BT_STAT(6);
            if (COUNT) ns += 1;
        }
        if (phi_new < phi) {
            BT_STAT(bt);
            moved = sqrt((qx - px) * (qx - px) + (qy - py) * (qy - py) + (qz - pz) * (qz - pz));
            px = qx; py = qy; pz = qz;
            phi = phi_new;
            alpha = dmin(alpha * 1.5, 4.0 * g.voxel);
            return true;
        }
        alpha *= 0.5;
    }
    BT_STAT(4);
    moved = 0.0;
    return false;
}

template <bool COUNT, bool UNIFORM>
__global__ void __launch_bounds__(256, UNIFORM ? FIRST_MINB : FIRST_MINB - 1) k_pgd_first(const int2 *__restrict__ block_map, const EnvXf *__restrict__ xf,
                                                   const SdfDesc *__restrict__ sdfs, const MeshDesc *__restrict__ meshes,
                                                   Staging st, unsigned long long *__restrict__ counter, const PlanGrid gu,
                                                  const MeshDesc mu, int um) {
#if STUCK0 && !PGD_FUSE0
    const unsigned n = st.work_count[1];  // the faces stage 0 could not finish, listed in st.slow
#else
    const unsigned n = st.work_count[0];
#endif
    unsigned long long ns = 0;
    for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
#if STUCK0 && !PGD_FUSE0
        const unsigned idx = st.slow[i];
#else
        const unsigned idx = i;
#endif
        const FaceWork *w = st.work + idx;
        double px, py, pz, gx, gy, gz, phi = w->phi[3];
        FaceGeom f;
        const PlanGrid *gp;
        {   // the header's fields die here: the tail reads them again (registers are this kernel's limit)
            const int4 hd = __ldg(reinterpret_cast<const int4 *>(w));  // row, blk, face, env in one load
            const int64_t row = hd.x;
            f = face_geom(xf[hd.w], meshes, mu, um, hd.z & 0x3fffffff);
            face_start(f, (int)((unsigned)hd.z >> 30), px, py, pz);
            gp = &grid_of<UNIFORM>(gu, sdfs, xf, hd.w);
#if PGD_FUSE0
            // iteration 0's gradient at the start point, here (no k_pgd_grad stage 0)
            gradient(*gp, px, py, pz, gx, gy, gz);
            if (COUNT) ns += 6;
#else
            gx = st.grad[3 * row]; gy = st.grad[3 * row + 1]; gz = st.grad[3 * row + 2];
#endif
        }
        const double gnorm = sqrt(gx * gx + gy * gy + gz * gz);
        double alpha = gp->voxel, moved = 0.0;
        // contacts/_kernels.py:61-62: a vanishing gradient ends the descent here
        const bool mv = !(gnorm < 1e-12) &&
                        backtrack<COUNT>(*gp, f, w->phi, gx, gy, gz, gnorm, px, py, pz, phi, alpha, moved, ns);
        const int4 hd = __ldg(reinterpret_cast<const int4 *>(w));
        const int64_t row = hd.x;
        const int blk = hd.y, face = hd.z & 0x3fffffff;
        const EnvXf &X = xf[hd.w];
        BT_STAT(mv ? (((unsigned)hd.z >> 30) == 0 ? 10 : 11) : (((unsigned)hd.z >> 30) == 0 ? 8 : 9));
        if (!mv && ((unsigned)hd.z >> 30) != 0) BT_STAT(12 + ((unsigned)hd.z >> 30));  // [13..15]: stuck at a / b / c
        if (!mv) {
            // no move: this gradient is the final one; the point and phi go to the staging row
            // only when the face is found (the only rows k_compact reads)
            if (phi <= X.cd) {
                st.point[3 * row] = px; st.point[3 * row + 1] = py; st.point[3 * row + 2] = pz; st.phi[row] = phi;
#if PGD_FUSE0
                st.grad[3 * row] = gx; st.grad[3 * row + 1] = gy; st.grad[3 * row + 2] = gz;
#endif
            }
            finish_face(st, row, blk, face, phi, X.cd);
            continue;
        }
        st.point[3 * row] = px; st.point[3 * row + 1] = py; st.point[3 * row + 2] = pz;
        st.phi[row] = phi;
        st.alpha[row] = alpha;
        // moved < tol ends the descent (its final gradient is at the new point); 1 < max_iters
        const unsigned slot = atomicAdd(st.work_count + 2, 1u);
        st.acc[slot] = idx | (moved < X.tol ? ACC_FINAL : 0u);
        st.acc_hd[slot] = hd;
    }
    if (COUNT) {
        for (int o = 16; o; o >>= 1) ns += __shfl_xor_sync(0xffffffffu, ns, o);
        if ((threadIdx.x & 31) == 0 && ns) atomicAdd(counter, ns);
    }
}

// Iterations 1.. of a face still moving: (gx, gy, gz) is the gradient at p; on return
// (p, phi, g) are the descent's final point, value and gradient.
template <bool COUNT, class G>
__device__ __forceinline__ void descend_rest(const G &g, const EnvXf &X, const FaceGeom &f, const double *vphi,
                                             double &px, double &py, double &pz, double &phi, double alpha,
                                             double &gx, double &gy, double &gz, unsigned long long &ns) {
    for (int it = 1; it < MAX_MINIMIZE_ITERS; ++it) {
        const double gnorm = sqrt(gx * gx + gy * gy + gz * gz);
        if (gnorm < 1e-12) break;
        double moved;
        const bool acc = backtrack<COUNT>(g, f, vphi, gx, gy, gz, gnorm, px, py, pz, phi, alpha, moved, ns);
        if (acc) {  // the gradient at the new point: the next iteration's, or the final one
            gradient(g, px, py, pz, gx, gy, gz);
            if (COUNT) ns += 6;
        }
        if (moved < X.tol) break;
    }
}

// Stage 1 fused with the rest of the descent: the gradient at the moved point of every
// accepted face; faces not yet done continue their descent in the same thread (no
// k_pgd_rest launch, and the long descents start as soon as their gradient is known).
template <bool COUNT, bool UNIFORM>
__global__ void __launch_bounds__(256, UNIFORM ? FIRST_MINB : FIRST_MINB - 1) k_pgd_grad1_rest(const EnvXf *__restrict__ xf,
                                                  const SdfDesc *__restrict__ sdfs, const MeshDesc *__restrict__ meshes,
                                                  Staging st, unsigned long long *__restrict__ counter, const PlanGrid gu,
                                                  const MeshDesc mu, int um) {
    const unsigned n = st.work_count[2];
    unsigned long long ns = 0;
    for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const unsigned a = st.acc[i];
        const int4 hd = st.acc_hd[i];
        const unsigned idx = a & ~ACC_FINAL;
        const int64_t row = hd.x;
        const int blk = hd.y, face = hd.z & 0x3fffffff, e = hd.w;
        const PlanGrid &g = grid_of<UNIFORM>(gu, sdfs, xf, e);
        double px = st.point[3 * row], py = st.point[3 * row + 1], pz = st.point[3 * row + 2];
        double gx, gy, gz;
        gradient(g, px, py, pz, gx, gy, gz);
        if (COUNT) ns += 6;
        double phi = st.phi[row];
        if (!(a & ACC_FINAL)) {
            const EnvXf &X = xf[e];
            const FaceWork *w = st.work + idx;
            const FaceGeom f = face_geom(X, meshes, mu, um, face);
            descend_rest<COUNT>(g, X, f, w->phi, px, py, pz, phi, st.alpha[row], gx, gy, gz, ns);
            st.point[3 * row] = px; st.point[3 * row + 1] = py; st.point[3 * row + 2] = pz;
            st.phi[row] = phi;
        }
        st.grad[3 * row] = gx; st.grad[3 * row + 1] = gy; st.grad[3 * row + 2] = gz;
        finish_face(st, row, blk, face, phi, xf[e].cd);
    }
    if (COUNT) {
        for (int o = 16; o; o >>= 1) ns += __shfl_xor_sync(0xffffffffu, ns, o);
        if ((threadIdx.x & 31) == 0 && ns) atomicAdd(counter, ns);
    }
}

// Iterations 1.. of the faces still moving (the gradient at their point is in the row).
template <bool COUNT, bool UNIFORM>
__global__ void __launch_bounds__(128, UNIFORM ? REST_MINB : REST_MINB - 1) k_pgd_rest(const int2 *__restrict__ block_map, const EnvXf *__restrict__ xf,
                                                  const SdfDesc *__restrict__ sdfs, const MeshDesc *__restrict__ meshes,
                                                  Staging st, unsigned long long *__restrict__ counter, const PlanGrid gu,
                                                  const MeshDesc mu, int um) {
    const unsigned n = st.work_count[3];
    unsigned long long ns = 0;
    for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const unsigned idx = st.slow[i];
        const FaceWork *w = st.work + idx;
        const int4 hd = __ldg(reinterpret_cast<const int4 *>(w));  // row, blk, face, env in one load
        const int64_t row = hd.x;
        const int blk = hd.y;
        const int face = hd.z & 0x3fffffff;
        const int e = hd.w;
        const EnvXf &X = xf[e];
        const PlanGrid &g = grid_of<UNIFORM>(gu, sdfs, xf, e);
        const FaceGeom f = face_geom(X, meshes, mu, um, face);
        const double *vphi = w->phi;
        double px = st.point[3 * row], py = st.point[3 * row + 1], pz = st.point[3 * row + 2];
        double phi = st.phi[row];
        double gx = st.grad[3 * row], gy = st.grad[3 * row + 1], gz = st.grad[3 * row + 2];
        descend_rest<COUNT>(g, X, f, vphi, px, py, pz, phi, st.alpha[row], gx, gy, gz, ns);
        st.point[3 * row] = px; st.point[3 * row + 1] = py; st.point[3 * row + 2] = pz;
        st.phi[row] = phi;
        st.grad[3 * row] = gx; st.grad[3 * row + 1] = gy; st.grad[3 * row + 2] = gz;
        finish_face(st, row, blk, face, phi, X.cd);
    }
    if (COUNT) {
        for (int o = 16; o; o >>= 1) ns += __shfl_xor_sync(0xffffffffu, ns, o);
        if ((threadIdx.x & 31) == 0 && ns) atomicAdd(counter, ns);
    }
}

// Stitch the per-chunk survivor rows into the env's candidate list (found faces
// in ascending face order) and apply the world-frame epilogue (generation.py:98-114).
// One CTA per env: chunk offsets by a block scan of the found counts, then one
// warp per chunk compacts its rows with a ballot.
__global__ void __launch_bounds__(COMPACT_BLOCK, COMPACT_MINB) k_compact(const EnvXf *__restrict__ xf,
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
        const int v = j < nch ? st.chunk_found[c0 + j] : 0;
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
        if (st.chunk_found[c0 + j] == 0) continue;
        const int cnt = st.chunk_count[c0 + j];
        const int64_t src0 = base + block_map[c0 + j].y;
        int64_t dst = base + st.chunk_off[c0 + j];
        // two groups of 32 rows per round, every load of both in flight at once (rows
        // not found carry stale values that are never used)
        for (int i0 = 0; i0 < cnt; i0 += 64) {
            int fidx[2];
            double px[2], py[2], pz[2], gx[2], gy[2], gz[2], phi[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int i = i0 + 32 * h + lane;
                const int64_t s = src0 + i;
                fidx[h] = -1;
                px[h] = py[h] = pz[h] = gx[h] = gy[h] = gz[h] = phi[h] = 0.0;
                if (i < cnt) {
                    fidx[h] = st.face[s];
                    px[h] = st.point[3 * s]; py[h] = st.point[3 * s + 1]; pz[h] = st.point[3 * s + 2];
                    gx[h] = st.grad[3 * s]; gy[h] = st.grad[3 * s + 1]; gz[h] = st.grad[3 * s + 2];
                    phi[h] = st.phi[s];
                }
            }
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const unsigned bal = __ballot_sync(0xffffffffu, fidx[h] >= 0);
                if (fidx[h] >= 0) {
                    const int64_t d = dst + __popc(bal & ((1u << lane) - 1u));
                    double ux = gx[h], uy = gy[h], uz = gz[h];
                    double nrm = sqrt(ux * ux + uy * uy + uz * uz);  // np.linalg.norm(axis=1): ((x2+y2)+z2)
                    if (nrm < 1e-12) { ux = 0.0; uy = 0.0; uz = 1.0; nrm = 1.0; }
                    const double nx = ux / nrm, ny = uy / nrm, nz = uz / nrm;
                    for (int k = 0; k < 3; ++k) {
                        const double *rr = sx.Rs + 3 * k;
                        cs.normal[3 * d + k] =
                            gemm ? G3(nx, ny, nz, rr[0], rr[1], rr[2]) : V3(nx, ny, nz, rr[0], rr[1], rr[2]);
                        cs.point[3 * d + k] = (gemm ? G3(px[h], py[h], pz[h], rr[0], rr[1], rr[2])
                                                    : V3(px[h], py[h], pz[h], rr[0], rr[1], rr[2])) + sx.ts[k];
                    }
                    cs.depth[d] = -phi[h];
                    cs.face[d] = fidx[h];
                }
                dst += __popc(bal);
            }
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
                   int32_t *env_status, double *env_min_depth, unsigned *work_count, cudaStream_t s,
                   const int32_t *active) {
    int bs = 128;
    k_env_xf<<<(unsigned)((E + bs - 1) / bs), bs, 0, s>>>(E, env_sdf, env_mesh, sdfs, sdf_pose, mesh_pose,
                                                          pose_format, cd, xf, env_status, env_min_depth, work_count,
                                                          active);
}

size_t face_prep_smem(int maxcv) {
    return (size_t)maxcv * (4 * sizeof(double) + sizeof(int) + 1) + (size_t)FACE_CHUNK * (sizeof(double) + sizeof(uint2) + sizeof(int));
}

void launch_face_prep(int64_t nblocks, const int4 *block_map, const EnvXf *xf, const SdfDesc *sdfs,
                      const MeshDesc *meshes, const int64_t *cand_base, const Staging &st, int maxcv,
                      unsigned long long *counter, const PlanGrid *uniform, cudaStream_t s,
                      const MeshDesc *umesh) {
    const MeshDesc mu = umesh ? *umesh : MeshDesc{};
    const int um = umesh ? 1 : 0;
    if (nblocks <= 0) return;
    const PlanGrid gu = uniform ? *uniform : PlanGrid{};
    const unsigned nb = (unsigned)nblocks;
    const size_t sm = face_prep_smem(maxcv);
    if (uniform) {
        if (counter) k_face_prep<true, true><<<nb, FACE_CHUNK, sm, s>>>(block_map, xf, sdfs, meshes, cand_base, st, maxcv, counter, gu, mu, um);
        else k_face_prep<false, true><<<nb, FACE_CHUNK, sm, s>>>(block_map, xf, sdfs, meshes, cand_base, st, maxcv, nullptr, gu, mu, um);
    } else {
        if (counter) k_face_prep<true, false><<<nb, FACE_CHUNK, sm, s>>>(block_map, xf, sdfs, meshes, cand_base, st, maxcv, counter, gu, mu, um);
        else k_face_prep<false, false><<<nb, FACE_CHUNK, sm, s>>>(block_map, xf, sdfs, meshes, cand_base, st, maxcv, nullptr, gu, mu, um);
    }
}

void launch_pgd_wave(int sm_count, const int2 *block_map, const EnvXf *xf, const SdfDesc *sdfs, const MeshDesc *meshes,
                     const Staging &st, unsigned long long *counter, const PlanGrid *uniform, cudaStream_t s,
                     const MeshDesc *umesh) {
    const PlanGrid gu = uniform ? *uniform : PlanGrid{};
    const MeshDesc mu = umesh ? *umesh : MeshDesc{};
    const int um = umesh ? 1 : 0;
    const unsigned g = (unsigned)sm_count * WAVE_GRID, gr = (unsigned)sm_count * REST_GRID;
#define CS_WAVE(C, U)                                                                                 \
    do {                                                                                              \
        if (!PGD_FUSE0) k_pgd_grad<C, U><<<g, 256, 0, s>>>(block_map, xf, sdfs, meshes, st, 0, counter, gu, mu, um); \
        k_pgd_first<C, U><<<g, 256, 0, s>>>(block_map, xf, sdfs, meshes, st, counter, gu, mu, um);   \
        if (PGD_FUSE_REST) {                                                                          \
            k_pgd_grad1_rest<C, U><<<g, 256, 0, s>>>(xf, sdfs, meshes, st, counter, gu, mu, um);         \
        } else {                                                                                      \
            k_pgd_grad<C, U><<<g, 256, 0, s>>>(block_map, xf, sdfs, meshes, st, 1, counter, gu, mu, um); \
            k_pgd_rest<C, U><<<gr, 128, 0, s>>>(block_map, xf, sdfs, meshes, st, counter, gu, mu, um);   \
        }                                                                                             \
    } while (0)
    if (uniform) {
        if (counter) CS_WAVE(true, true); else CS_WAVE(false, true);
    } else {
        if (counter) CS_WAVE(true, false); else CS_WAVE(false, false);
    }
#undef CS_WAVE
}

// ---------------------------------------------------------------- cell-window minima
// (GridT::cwin; built once at SDF registration)

__global__ void k_cell_min(const float *__restrict__ v, int nx, int ny, int nz, float *__restrict__ out) {
    const int cnx = nx - 1, cny = ny - 1, cnz = nz - 1;
    const int64_t nc = (int64_t)cnx * cny * cnz;
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < nc; c += (int64_t)gridDim.x * blockDim.x) {
        const int x = (int)(c % cnx), y = (int)((c / cnx) % cny), z = (int)(c / ((int64_t)cnx * cny));
        const float *p = v + x + (int64_t)nx * (y + (int64_t)ny * z);
        const int64_t sy = nx, sz = (int64_t)nx * ny;
        out[c] = fminf(fminf(fminf(p[0], p[1]), fminf(p[sy], p[sy + 1])),
                       fminf(fminf(p[sz], p[sz + 1]), fminf(p[sy + sz], p[sy + sz + 1])));
    }
}

// out[c] = min(in[c], in[c + h along axis]) (the second term dropped past the last cell)
__global__ void k_min_shift(const float *__restrict__ in, float *__restrict__ out, int cnx, int cny, int cnz, int axis,
                            int h) {
    const int64_t nc = (int64_t)cnx * cny * cnz;
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < nc; c += (int64_t)gridDim.x * blockDim.x) {
        const int x = (int)(c % cnx), y = (int)((c / cnx) % cny), z = (int)(c / ((int64_t)cnx * cny));
        const int pos = axis == 0 ? x : axis == 1 ? y : z, n = axis == 0 ? cnx : axis == 1 ? cny : cnz;
        const int64_t stride = axis == 0 ? 1 : axis == 1 ? (int64_t)cnx : (int64_t)cnx * cny;
        float m = in[c];
        if (pos + h < n) m = fminf(m, in[c + h * stride]);
        out[c] = m;
    }
}

// tables: CWIN_LEVELS x (nx-1)(ny-1)(nz-1) floats; tmp: one table
void build_cell_windows(const float *values, int nx, int ny, int nz, float *tables, float *tmp, cudaStream_t s) {
    const int cnx = nx - 1, cny = ny - 1, cnz = nz - 1;
    const int64_t nc = (int64_t)cnx * cny * cnz;
    const unsigned grid = (unsigned)std::min<int64_t>((nc + 255) / 256, 148 * 32);
    k_cell_min<<<grid, 256, 0, s>>>(values, nx, ny, nz, tables);
    for (int l = 1; l < CWIN_LEVELS; ++l) {  // width 2^l from width 2^(l-1): shift by half per axis
        const int h = 1 << (l - 1);
        const float *prev = tables + (int64_t)(l - 1) * nc;
        float *cur = tables + (int64_t)l * nc;
        k_min_shift<<<grid, 256, 0, s>>>(prev, cur, cnx, cny, cnz, 0, h);
        k_min_shift<<<grid, 256, 0, s>>>(cur, tmp, cnx, cny, cnz, 1, h);
        k_min_shift<<<grid, 256, 0, s>>>(tmp, cur, cnx, cny, cnz, 2, h);
    }
}

// ---------------------------------------------------------------- brick-window minima
// (GridT::bwin; built once at SDF registration, on the device)

// bm[b] = min over the nodes of brick b: nodes k B .. k B + B per axis (closed, clamped
// to the last node); bricks per axis (n - 2) / B + 1
__global__ void k_brick_min(const float *__restrict__ v, int nx, int ny, int nz, int bx, int by, int bz,
                            float *__restrict__ bm) {
    const int64_t nb = (int64_t)bx * by * bz;
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x) {
        const int kx = (int)(b % bx), ky = (int)((b / bx) % by), kz = (int)(b / ((int64_t)bx * by));
        const int x1 = min(kx * BRICK + BRICK, nx - 1), y1 = min(ky * BRICK + BRICK, ny - 1),
                  z1 = min(kz * BRICK + BRICK, nz - 1);
        float m = INFINITY;
        for (int z = kz * BRICK; z <= z1; ++z)
            for (int y = ky * BRICK; y <= y1; ++y) {
                const float *row = v + (int64_t)nx * (y + (int64_t)ny * z);
                for (int x = kx * BRICK; x <= x1; ++x) m = fminf(m, row[x]);
            }
        bm[b] = m;
    }
}

// the 8 window tables: widths {1, 2} per axis, window [b, b + w - 1] clamped to the last brick
__global__ void k_brick_windows(const float *__restrict__ bm, int bx, int by, int bz, float *__restrict__ bw) {
    const int64_t nb = (int64_t)bx * by * bz;
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x) {
        const int x = (int)(b % bx), y = (int)((b / bx) % by), z = (int)(b / ((int64_t)bx * by));
        const int x2 = min(x + 1, bx - 1), y2 = min(y + 1, by - 1), z2 = min(z + 1, bz - 1);
        auto at = [&](int xx, int yy, int zz) { return bm[xx + (int64_t)bx * (yy + (int64_t)by * zz)]; };
        const float m000 = at(x, y, z), m100 = at(x2, y, z), m010 = at(x, y2, z), m110 = at(x2, y2, z);
        const float m001 = at(x, y, z2), m101 = at(x2, y, z2), m011 = at(x, y2, z2), m111 = at(x2, y2, z2);
        const float w1 = m000, w2 = fminf(m000, m100);                       // (wx, 1, 1)
        const float w3 = fminf(m000, m010), w4 = fminf(w2, fminf(m010, m110));  // (1, 2, 1), (2, 2, 1)
        const float z0[4] = {w1, w2, w3, w4};
        const float z1[4] = {m001, fminf(m001, m101), fminf(m001, m011), fminf(fminf(m001, m101), fminf(m011, m111))};
        for (int t = 0; t < 8; ++t) bw[(int64_t)t * nb + b] = t < 4 ? z0[t] : fminf(z0[t - 4], z1[t - 4]);
    }
}

// scan[0] |= 1 if a value is not finite; scan[1] = max |value| (float bits, finite values)
__global__ void k_grid_scan(const float *__restrict__ v, int64_t n, unsigned *__restrict__ scan) {
    unsigned bad = 0, mx = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float a = fabsf(v[i]);
        if (!(a <= 3.402823466e38f)) bad = 1;
        else mx = max(mx, __float_as_uint(a));
    }
    bad = __reduce_or_sync(0xffffffffu, bad);
    mx = __reduce_max_sync(0xffffffffu, mx);
    if ((threadIdx.x & 31) == 0) {
        if (bad) atomicOr(scan, 1u);
        atomicMax(scan + 1, mx);
    }
}

void build_brick_windows(const float *values, int nx, int ny, int nz, int bx, int by, int bz, float *bm, float *bw,
                         unsigned *scan, cudaStream_t s) {
    const int64_t nb = (int64_t)bx * by * bz, n = (int64_t)nx * ny * nz;
    const unsigned gb = (unsigned)std::min<int64_t>((nb + 255) / 256, 148 * 32);
    const unsigned gn = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 32);
    k_brick_min<<<gb, 256, 0, s>>>(values, nx, ny, nz, bx, by, bz, bm);
    k_brick_windows<<<gb, 256, 0, s>>>(bm, bx, by, bz, bw);
    cudaMemsetAsync(scan, 0, 2 * sizeof(unsigned), s);
    k_grid_scan<<<gn, 256, 0, s>>>(values, n, scan);
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
