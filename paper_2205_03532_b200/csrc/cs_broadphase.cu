// Broadphase kernels (cs_broadphase.cuh), bit-identical to the reference: the
// world AABB corners go through the reference's dgemm rounding (G3 per element,
// then + t, math3d.py:168-169), the margin is applied as numpy does (lo - m,
// hi + m), and the overlap tests are the reference's comparisons — all three axes
// both ways up to SWEEP_THRESHOLD bodies (broadphase.py:47-52), the sweep's tests
// above it (:55-68: for k before idx in the stable lo.x order, hi_k.x >= lo_idx.x
// and y/z both ways). The two agree on valid boxes and differ on inverted ones;
// both are reproduced. Pairs come out sorted by (id_a, id_b) (:43).
#include "cs_broadphase.cuh"

namespace cs {

namespace {

// numpy min/max reduction step: NaN propagates
__device__ __forceinline__ double np_min(double acc, double x) { return (isnan(acc) || acc < x) ? acc : x; }
__device__ __forceinline__ double np_max(double acc, double x) { return (isnan(acc) || acc > x) ? acc : x; }

// RigidBody.world_aabb: the mesh AABB's 8 corners in the reference's order
// (x outer, z inner) through Transform.from_pose(p, q).apply, then min/max
__global__ void k_world_aabb(int64_t n, const double *__restrict__ mesh_lo, const double *__restrict__ mesh_hi,
                             const double *__restrict__ pose7, double *__restrict__ lo, double *__restrict__ hi) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    double R[9];
    quat_to_matrix(pose7 + 7 * i + 3, R);
    const double *t = pose7 + 7 * i, *ml = mesh_lo + 3 * i, *mh = mesh_hi + 3 * i;
    double l[3], h[3];
    for (int c = 0; c < 8; ++c) {
        const double p0 = (c & 4) ? mh[0] : ml[0], p1 = (c & 2) ? mh[1] : ml[1], p2 = (c & 1) ? mh[2] : ml[2];
        for (int j = 0; j < 3; ++j) {
            const double w = G3(p0, p1, p2, R[3 * j], R[3 * j + 1], R[3 * j + 2]) + t[j];
            l[j] = c ? np_min(l[j], w) : w;
            h[j] = c ? np_max(h[j], w) : w;
        }
    }
    for (int j = 0; j < 3; ++j) { lo[3 * i + j] = l[j]; hi[3 * i + j] = h[j]; }
}

constexpr int BP_T = 256;

__global__ void __launch_bounds__(BP_T) k_broadphase(int64_t S, BroadIO io) {
    __shared__ int ord[BROAD_MAX_BODIES];  // id rank -> local body
    __shared__ int xr[BROAD_MAX_BODIES];   // local body -> rank in the sweep order (n > threshold)
    __shared__ int ws[WS_INTS];
    __shared__ int s_flags;
    const int64_t s = blockIdx.x;
    if (s >= S) return;
    const int64_t b0 = io.body_off[s];
    const int n = (int)(io.body_off[s + 1] - b0);
    const double m = io.margin[s];
    const int64_t cap = io.pair_off[s + 1] - io.pair_off[s];
    int64_t *out = io.pairs + 2 * io.pair_off[s];
    if (threadIdx.x == 0) s_flags = 0;
    __syncthreads();
    if (n > BROAD_MAX_BODIES) {
        if (threadIdx.x == 0) { io.n_pairs[s] = 0; io.status[s] = 3; }
        return;
    }
    const double *lo = io.lo + 3 * b0, *hi = io.hi + 3 * b0;
    const int64_t *ids = io.ids + b0;
    for (int i = threadIdx.x; i < n; i += BP_T) {
        bool ok = true;
        for (int k = 0; k < 3; ++k) ok &= isfinite(lo[3 * i + k] - m) && isfinite(hi[3 * i + k] + m);
        if (!ok) atomicOr(&s_flags, 1);
        const int64_t id = ids[i];
        const double xi = lo[3 * i] - m;
        int r = 0, rx = 0, dup = 0;
        for (int j = 0; j < n; ++j) {
            const int64_t o = ids[j];
            r += o < id;
            dup += (o == id) & (j != i);
            const double xj = lo[3 * j] - m;
            rx += (xj < xi) | ((xj == xi) & (j < i));  // stable argsort (broadphase.py:56)
        }
        if (dup) atomicOr(&s_flags, 4);
        ord[r] = i;
        xr[i] = rx;
    }
    __syncthreads();
    if (s_flags) {
        if (threadIdx.x == 0) { io.n_pairs[s] = 0; io.status[s] = (s_flags & 1) ? 1 : 4; }
        return;
    }
    const bool sweep = n > BROAD_SWEEP_THRESHOLD;
    const int64_t T = (int64_t)n * (n - 1) / 2;
    int64_t cnt = 0;
    for (int64_t k0 = 0; k0 < T; k0 += BP_T) {
        const int64_t k = k0 + threadIdx.x;
        bool hit = false;
        int i = 0, j = 0;
        if (k < T) {
            // pair k of the (p, q), p < q, lexicographic enumeration of the id ranks
            const double nn = n - 0.5;
            int p = (int)(nn - sqrt(nn * nn - 2.0 * (double)k));
            p = max(0, min(p, n - 2));
            auto start = [&](int pp) { return (int64_t)pp * (2 * (int64_t)n - pp - 1) / 2; };
            while (p > 0 && start(p) > k) --p;
            while (p < n - 2 && start(p + 1) <= k) ++p;
            const int q = p + 1 + (int)(k - start(p));
            i = ord[p];
            j = ord[q];
            if (sweep) {
                const int a = xr[i] < xr[j] ? i : j, b = xr[i] < xr[j] ? j : i;  // a swept first
                hit = hi[3 * a] + m >= lo[3 * b] - m;
                for (int c = 1; c < 3; ++c)
                    hit &= (lo[3 * b + c] - m <= hi[3 * a + c] + m) && (lo[3 * a + c] - m <= hi[3 * b + c] + m);
            } else {
                hit = true;
                for (int c = 0; c < 3; ++c)
                    hit &= (lo[3 * i + c] - m <= hi[3 * j + c] + m) && (lo[3 * j + c] - m <= hi[3 * i + c] + m);
            }
        }
        int tot;
        const int pos = block_excl_scan(hit ? 1 : 0, ws, &tot);
        if (hit && cnt + pos < cap) {
            out[2 * (cnt + pos)] = ids[i];
            out[2 * (cnt + pos) + 1] = ids[j];
        }
        cnt += tot;
    }
    if (threadIdx.x == 0) {
        io.n_pairs[s] = (int32_t)(cnt < cap ? cnt : cap);
        io.status[s] = cnt > cap ? 2 : 0;
    }
}

// active[t] = slot t's (id_a, id_b) is among its scene's broadphase pairs (binary search)
__global__ void k_pair_slots(int64_t n, const int64_t *__restrict__ slot_scene, const int64_t *__restrict__ slot_pair,
                             const int64_t *__restrict__ pair_off, const int64_t *__restrict__ pairs,
                             const int32_t *__restrict__ n_pairs, int32_t *__restrict__ active) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= n) return;
    const int64_t s = slot_scene[t], a = slot_pair[2 * t], b = slot_pair[2 * t + 1];
    const int64_t *P = pairs + 2 * pair_off[s];
    int lo = 0, hi = n_pairs[s];
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        const int64_t pa = P[2 * mid], pb = P[2 * mid + 1];
        if (pa < a || (pa == a && pb < b)) lo = mid + 1;
        else hi = mid;
    }
    active[t] = lo < n_pairs[s] && P[2 * lo] == a && P[2 * lo + 1] == b;
}

}  // namespace

void launch_world_aabb(int64_t n, const double *mesh_lo, const double *mesh_hi, const double *pose7, double *lo,
                       double *hi, cudaStream_t s) {
    if (n <= 0) return;
    k_world_aabb<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(n, mesh_lo, mesh_hi, pose7, lo, hi);
}

void launch_broadphase(int64_t n_scenes, const BroadIO &io, cudaStream_t s) {
    if (n_scenes <= 0) return;
    k_broadphase<<<(unsigned)n_scenes, BP_T, 0, s>>>(n_scenes, io);
}

void launch_pair_slots(int64_t n_slots, const int64_t *slot_scene, const int64_t *slot_pair, const int64_t *pair_off,
                       const int64_t *pairs, const int32_t *n_pairs, int32_t *active, cudaStream_t s) {
    if (n_slots <= 0) return;
    k_pair_slots<<<(unsigned)((n_slots + 255) / 256), 256, 0, s>>>(n_slots, slot_scene, slot_pair, pair_off, pairs,
                                                                   n_pairs, active);
}

}  // namespace cs
