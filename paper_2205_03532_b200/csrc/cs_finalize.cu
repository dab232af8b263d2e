// Per-patch finalisation on sm_100a (reduction.py:146-236), split by the kind of
// parallelism each part has:
//
//   k_patch_off       exclusive scan of patch counts -> work list [E+1].
//   k_fin_sort_warp   ONE WARP PER PATCH (<= FW_SMEM members), in shared memory:
//                     deepest member (first argmax), max depth, touching count, the
//                     weighted sums (reduction.py:162-165), the (u, v) projections
//                     (reduction.py:202-204) and a merge-path sort by (u, v, member)
//                     -- lexsort's order (reduction.py:211) -- written to the
//                     patch's scratch rows; queues the patch's chain jobs.
//   k_fin_sort_block  the same, ONE CTA per larger patch.
//   k_fin_chain       ONE WARP PER PATCH, an 8-lane group per half chain of Andrew's
//                     monotone chain (reduction.py:214-223), lower and upper, over all
//                     members (the area hull) and, when the kept selection uses them,
//                     over the touching members (reduction.py:183-185); the pops of a
//                     key are tested in parallel. Longest patches first.
//   k_fin_kept        one warp per patch: hull assembly, kept selection
//                     (reduction.py:172-199), hull area (reduction.py:227-236), rows.
//   k_stats           per env stats (the multi-GPU all-gather payload).
//
// The chains are sequential by definition (each step depends on the stack the
// previous steps left), so their parallelism is across patches, not within one.
// One sort serves both hulls: lexsort of the touching subset breaks (u, v) ties by
// position in that subset, which is monotone in the member position, so its order
// is the all-members order (u, v, member) filtered to the touching members; the
// projections are the same V3 gemv dot products either way.
#include <cstdint>
#include <stdint.h>

#include "cs_reduce_util.cuh"

namespace cs {

#ifndef FW_WARPS
#define FW_WARPS 4      // warp teams per k_fin_sort_warp CTA
#endif
#ifndef FW_SMEM
#define FW_SMEM 128     // members per warp-path patch (all in shared memory)
#endif
#ifndef FIN_GRID
#define FIN_GRID 16  // scale of the finalize grids (patches assigned by grid stride): patch sizes vary
                     // widely, so many CTAs balance the tail (x1: +0.10 ms; x8..x64 alike)
#endif
#ifndef FIN_GRID_CHAIN
#define FIN_GRID_CHAIN 1  // k_fin_chain claims jobs dynamically: x4 is no faster
#endif
#ifndef FB_THREADS
#define FB_THREADS 128  // k_fin_sort_block
#endif
constexpr int CH_BUCKETS = 64;   // chain jobs bucketed by length (16 keys per bucket)

__device__ __forceinline__ int job_bucket(int len) { return max(0, CH_BUCKETS - 1 - len / 16); }  // longest first

__global__ void k_patch_off(int64_t E, const int32_t *__restrict__ n_patch, int32_t *__restrict__ off,
                            int32_t *__restrict__ large_count, int32_t *__restrict__ njob) {
    __shared__ int ws[WS_INTS];
    if (threadIdx.x == 0) *large_count = 0;
    if (threadIdx.x <= CH_BUCKETS) njob[threadIdx.x] = 0;
    int running = 0;
    for (int64_t e0 = 0; e0 < E; e0 += blockDim.x) {
        int64_t e = e0 + threadIdx.x;
        int v = e < E ? n_patch[e] : 0;
        int tot;
        int x = block_excl_scan(v, ws, &tot);
        if (e < E) off[e] = running + x;
        running += tot;
    }
    if (threadIdx.x == 0) off[E] = running;
}

// patch (work index) -> env, so stage 1 finds a patch's env with one load; patches
// above FW_SMEM members go to the list of the CTA-per-patch kernels
__global__ void k_patch_env(int64_t E, int N, const int32_t *__restrict__ n_patch, const int32_t *__restrict__ off,
                            const int32_t *__restrict__ member_offsets, int32_t *__restrict__ wenv,
                            int32_t *__restrict__ large_list, int32_t *__restrict__ large_count) {
    const int64_t e = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (e >= E) return;
    const int o = off[e], n = n_patch[e];
    const int32_t *mo = member_offsets + e * (N + 1);
    for (int q = lane; q < n; q += 32) {
        wenv[o + q] = (int32_t)e;
        if (mo[q + 1] - mo[q] > FW_SMEM) large_list[atomicAdd(large_count, 1)] = o + q;
    }
}

// numpy stable argsort(-depths) order: depth descending, ties by index, NaN last.
__device__ __forceinline__ bool depth_before(double da, int a, double db, int b) {
    bool an = isnan(da), bnn = isnan(db);
    if (an != bnn) return !an;
    if (!an && da != db) return da > db;
    return a < b;
}

__device__ __forceinline__ double weight_of(double d) {
    return (d > 0.0) ? d : (isnan(d) ? d : 0.0);  // np.maximum(deps, 0.0)
}

// ------------------------------------------------------------------ teams

struct WarpTeam {
    int *misc;  // >= 4 ints of shared memory owned by this warp
    __device__ int rank() const { return threadIdx.x & 31; }
    __device__ int size() const { return 32; }
    __device__ void sync() const { __syncwarp(); }
    __device__ ArgMax argmax(ArgMax a) const { return warp_argmax(a); }
    __device__ double max(double x) const {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, o));
        return x;
    }
    __device__ int isum(int x) const {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        return x;
    }
    __device__ bool any(bool b) const { return __any_sync(0xffffffffu, b); }
    // first argmax, max (NaN ignored here, flagged by nan), any NaN, count: one pass
    __device__ void stats(ArgMax &am, double &mx, int &nan, int &cnt) const {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            ArgMax b;
            b.v = __shfl_xor_sync(0xffffffffu, am.v, o);
            b.i = __shfl_xor_sync(0xffffffffu, am.i, o);
            b.cnt = 0;
            am = argmax_combine(am, b);
            mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            nan |= __shfl_xor_sync(0xffffffffu, nan, o);
            cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        }
    }
    __device__ int excl_scan(int f, int *total) const {  // f in {0, 1}
        const unsigned b = __ballot_sync(0xffffffffu, f != 0);
        *total = __popc(b);
        return __popc(b & ((1u << rank()) - 1u));
    }
    // best (bk, bd) under depth_before over the team
    __device__ void best_depth(int &bk, double &bd) const {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            int ok = __shfl_xor_sync(0xffffffffu, bk, o);
            double od = __shfl_xor_sync(0xffffffffu, bd, o);
            if (ok >= 0 && (bk < 0 || depth_before(od, ok, bd, bk))) { bk = ok; bd = od; }
        }
    }
};

struct BlockTeam {
    ArgMax *am;    // 32 entries
    double *dred;  // 32 doubles
    int *ired;     // 32 ints
    int *ws;       // WS_INTS ints
    __device__ int rank() const { return threadIdx.x; }
    __device__ int size() const { return blockDim.x; }
    __device__ void sync() const { __syncthreads(); }
    __device__ ArgMax argmax(ArgMax a) const { return block_argmax(a, am); }
    __device__ double max(double x) const {
        int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, o));
        if (lane == 0) dred[wid] = x;
        __syncthreads();
        double r = -INFINITY;
        for (int i = 0; i < nw; ++i) r = fmax(r, dred[i]);
        __syncthreads();
        return r;
    }
    __device__ int isum(int x) const {
        int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if (lane == 0) ired[wid] = x;
        __syncthreads();
        int r = 0;
        for (int i = 0; i < nw; ++i) r += ired[i];
        __syncthreads();
        return r;
    }
    __device__ bool any(bool b) const { return __syncthreads_or(b) != 0; }
    __device__ int excl_scan(int f, int *total) const { return block_excl_scan(f, ws, total); }
    __device__ void stats(ArgMax &am, double &mx, int &nan, int &cnt) const {
        const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
        WarpTeam{nullptr}.stats(am, mx, nan, cnt);
        if (lane == 0) { this->am[wid] = am; dred[wid] = mx; ired[wid] = cnt | (nan << 29); }  // nan: 2 flag bits
        __syncthreads();
        am = this->am[0]; mx = dred[0]; cnt = ired[0] & ((1 << 29) - 1); nan = ired[0] >> 29;
        for (int i = 1; i < nw; ++i) {
            am = argmax_combine(am, this->am[i]);
            mx = fmax(mx, dred[i]);
            cnt += ired[i] & ((1 << 29) - 1);
            nan |= ired[i] >> 29;
        }
        __syncthreads();
    }
    __device__ void best_depth(int &bk, double &bd) const {
        int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            int ok = __shfl_xor_sync(0xffffffffu, bk, o);
            double od = __shfl_xor_sync(0xffffffffu, bd, o);
            if (ok >= 0 && (bk < 0 || depth_before(od, ok, bd, bk))) { bk = ok; bd = od; }
        }
        if (lane == 0) { ired[wid] = bk; dred[wid] = bd; }
        __syncthreads();
        bk = -1;
        for (int i = 0; i < nw; ++i)
            if (ired[i] >= 0 && (bk < 0 || depth_before(dred[i], ired[i], bd, bk))) { bk = ired[i]; bd = dred[i]; }
        __syncthreads();
    }
};

// ------------------------------------------------------------------ sort

struct Keys {
    double *u, *v;
    int32_t *k;
};

// Merge-path merge sort of m (u, v, k) keys (k distinct, so the order is total).
// Each rank owns c = ceil(m / T) consecutive output slots: it insertion-sorts its
// segment, then in every round binary-searches its split of the merge path of the
// two runs it falls in and merges c outputs into the other buffer. log2(T) rounds.
// Returns the buffer holding the result (0: a, 1: b).
template <bool NANS, class Team>
__device__ int team_merge_sort(const Team &t, Keys a, Keys b, int m) {
    const int T = t.size(), r = t.rank();
    const int c = (m + T - 1) / T;
    const int s0 = r * c, s1 = min(s0 + c, m);
    for (int i = s0 + 1; i < s1; ++i) {
        const double u = a.u[i], v = a.v[i];
        const int k = a.k[i];
        int j = i - 1;
        while (j >= s0) {
            const double uj = a.u[j], vj = a.v[j];
            const int kj = a.k[j];
            if (!key_less<NANS>(u, v, k, uj, vj, kj)) break;
            a.u[j + 1] = uj; a.v[j + 1] = vj; a.k[j + 1] = kj;
            --j;
        }
        a.u[j + 1] = u; a.v[j + 1] = v; a.k[j + 1] = k;
    }
    t.sync();
    int src = 0;
    for (int run = c, pm = 1; run < m; run <<= 1, pm = 2 * pm + 1) {
        const Keys S = src ? b : a, D = src ? a : b;
        if (s0 < m) {
            const int ps = (r & ~pm) * c;  // (s0 / (2 run)) (2 run): run = c 2^k, s0 = r c, pm = 2^(k+1) - 1
            const int a0 = ps, a1 = min(ps + run, m), b1 = min(ps + 2 * run, m);
            const int d = s0 - ps;
            int lo = max(0, d - (b1 - a1)), hi = min(d, a1 - a0);
            while (lo < hi) {  // first A element that is not among the first d outputs
                const int mid = (lo + hi) >> 1, bj = a1 + d - 1 - mid;
                if (key_less<NANS>(S.u[a0 + mid], S.v[a0 + mid], S.k[a0 + mid], S.u[bj], S.v[bj], S.k[bj])) lo = mid + 1;
                else hi = mid;
            }
            int i = a0 + lo, j = a1 + (d - lo);
            double ua = 0.0, va = 0.0, ub = 0.0, vb = 0.0;
            int ka = 0, kb = 0;
            if (i < a1) { ua = S.u[i]; va = S.v[i]; ka = S.k[i]; }
            if (j < b1) { ub = S.u[j]; vb = S.v[j]; kb = S.k[j]; }
            // branch-free: the lanes of a warp take A or B in any mix, so both sides are
            // written as selects (one store set, one load set per output)
            for (int o = s0; o < s1; ++o) {
                const bool ta = j >= b1 || (i < a1 && key_less<NANS>(ua, va, ka, ub, vb, kb));
                D.u[o] = ta ? ua : ub; D.v[o] = ta ? va : vb; D.k[o] = ta ? ka : kb;
                i += ta ? 1 : 0;
                j += ta ? 0 : 1;
                const int x = ta ? i : j;  // the consumed side's next key
                if (x < (ta ? a1 : b1)) {
                    const double nu = S.u[x], nv = S.v[x];
                    const int nk = S.k[x];
                    if (ta) { ua = nu; va = nv; ka = nk; } else { ub = nu; vb = nv; kb = nk; }
                }
            }
        }
        t.sync();
        src ^= 1;
    }
    return src;
}

// Which hulls a patch needs (reduction.py:152,174-185,227-231).
__device__ __forceinline__ bool needs_all_hull(int m, int K) { return m >= 3 || m > K; }
__device__ __forceinline__ bool needs_touch_hull(int m, int nt, int K) { return m > K && nt >= 3 && nt < m; }

// ------------------------------------------------------------------ stage 1: per patch

// Patch w = (e, q), by a team (warp or CTA). A/B: the team's sort buffers (shared
// memory, or the patch's global rows when it is very large); B holds the member
// weights until the sort. tile: 9 x (T + 1) doubles of shared memory (padded rows).
//   * one pass over the members: deepest (first argmax), max depth, touching count,
//     weights, the nine weighted products (np.cross(pts, norms) * w etc.) through
//     the tile, folded by ranks 0..8 in member order (numpy's axis-0 sums add row
//     after row, reduction.py:163-165), and the (u, v) projections
//     (reduction.py:202-204);
//   * the pairwise weight sum (reduction.py:162);
//   * a merge-path sort by (u, v, member) (lexsort, reduction.py:211), written to
//     the patch's rows of suv/sp (non-touching members as ~k), and the patch's
//     chain jobs queued (long patches and short patches in separate lists).
template <bool FOLD, class Team>
__device__ void sort_patch(const Team &t, const ReduceIO &io, const ReduceParams &p, int w, int64_t e, int q, Keys A,
                           Keys B, double *tile) {
    const int N = p.N, K = p.K;
    const int64_t base = io.cand_base[e];
    const int32_t *mo = io.member_offsets + e * (N + 1);
    const int moff = mo[q], m = mo[q + 1] - moff;
    const int32_t *mem = io.members + base + moff;
    const int64_t pq = e * N + q, row0 = base + moff;
    const double *P = io.point + 3 * base, *Nn = io.normal + 3 * base, *D = io.depth + base;
    const bool hull = needs_all_hull(m, K);
    double t1[3] = {0.0, 0.0, 0.0}, t2[3] = {0.0, 0.0, 0.0};
    if (hull) tangent_basis(io.patch_normal + 3 * pq, t1, t2);
    double *wb = B.u;
    const int r = t.rank(), T = t.size();
    ArgMax am = {0.0, -1, 0};
    double mx = -INFINITY, s = 0.0;
    bool anynan = false, uvnan = false;
    int nt = 0;
    // member data of this rank's next member, loaded one chunk ahead (the loads are
    // DRAM latency: the candidate rows outgrow L2)
    double fd = 0.0, fpx = 0.0, fpy = 0.0, fpz = 0.0, fnx = 0.0, fny = 0.0, fnz = 0.0;
    auto fetch = [&](int k) {
        if (k < m) {
            const int64_t i = __ldg(mem + k);
            fd = __ldg(D + i);
            fpx = __ldg(P + 3 * i); fpy = __ldg(P + 3 * i + 1); fpz = __ldg(P + 3 * i + 2);
            fnx = __ldg(Nn + 3 * i); fny = __ldg(Nn + 3 * i + 1); fnz = __ldg(Nn + 3 * i + 2);
        }
    };
    fetch(r);
    for (int c0 = 0; c0 < m; c0 += T) {
        const int k = c0 + r;
        if (k < m) {
            const double d = fd, px = fpx, py = fpy, pz = fpz, nx = fnx, ny = fny, nz = fnz;
            fetch(k + T);
            am = argmax_combine(am, ArgMax{d, k, 1});
            anynan |= isnan(d);
            if (d > mx) mx = d;
            nt += d >= 0.0 ? 1 : 0;
            if (FOLD) {
                const double wk = weight_of(d);
                wb[k] = wk;
                const int TP = T + 1;  // padded tile rows: the folding ranks read distinct banks
                tile[0 * TP + r] = px * wk; tile[1 * TP + r] = py * wk; tile[2 * TP + r] = pz * wk;
                tile[3 * TP + r] = nx * wk; tile[4 * TP + r] = ny * wk; tile[5 * TP + r] = nz * wk;
                tile[6 * TP + r] = (py * nz - pz * ny) * wk;
                tile[7 * TP + r] = (pz * nx - px * nz) * wk;
                tile[8 * TP + r] = (px * ny - py * nx) * wk;
            }
            if (hull) {
                A.u[k] = V3(px, py, pz, t1[0], t1[1], t1[2]);  // _project_2d: (n,3) @ (3,), n >= 2
                A.v[k] = V3(px, py, pz, t2[0], t2[1], t2[2]);
                // tie key 2k + touching: orders like k (k distinct) and carries the flag
                // through the sort, so the rows below need no second gather of the depth
                A.k[k] = 2 * k + (d >= 0.0 ? 1 : 0);
                uvnan |= isnan(A.u[k]) || isnan(A.v[k]);
            }
        }
        if (FOLD) {
            t.sync();
            if (r < 9) {
                const int cnt = min(T, m - c0);
                const double *row = tile + r * (T + 1);
                int j = 0;
                if (c0 == 0) { s = row[0]; j = 1; }
#pragma unroll 8
                for (; j < cnt; ++j) s = s + row[j];
            }
            t.sync();
        }
    }
    {
        int nan = (anynan ? 1 : 0) | (uvnan ? 2 : 0);
        t.stats(am, mx, nan, nt);
        anynan = (nan & 1) != 0;
        uvnan = (nan & 2) != 0;
    }
    if (FOLD && r < 9) {
        const int kind = r / 3, c = r % 3;
        double *o = (kind == 0 ? io.wp_sum : kind == 1 ? io.wn_sum : io.wt_sum) + 3 * pq;
        o[c] = s;
    } else if (FOLD && r == 9) {
        io.w_sum[pq] = 0.0 + pairwise([&](int k) { return wb[k]; }, 0, m);
    } else if (r == 10) {
        io.max_depth[pq] = anynan ? (double)NAN : mx;  // deps.max() propagates NaN
        io.pdeep[w] = am.i;
        io.pnt[w] = nt;
        if (hull) {  // chain jobs (4w + kind), bucketed by chain length (k_fin_chain: longest first)
            const int64_t cap = 4 * io.E * N;
            int k = job_bucket(m);
            int32_t *J = io.jobs + (int64_t)k * cap + atomicAdd(io.njob + k, 2);
            J[0] = 4 * w; J[1] = 4 * w + 1;
            if (needs_touch_hull(m, nt, K)) {
                k = job_bucket(nt);
                J = io.jobs + (int64_t)k * cap + atomicAdd(io.njob + k, 2);
                J[0] = 4 * w + 2; J[1] = 4 * w + 3;
            }
        }
    }
    t.sync();
    if (!hull) return;
    // numpy's NaN order only where a projection is NaN (the comparisons stay plain otherwise)
    const Keys R = (uvnan ? team_merge_sort<true>(t, A, B, m) : team_merge_sort<false>(t, A, B, m)) ? B : A;
    // sorted keys -> rows (non-touching members as ~k), and the touching keys alone,
    // in the same order, with their sorted positions (the touching chains' input)
    int run = 0;
    for (int j0 = 0; j0 < m; j0 += T) {
        const int j = j0 + r;
        bool touch = false;
        double2 uv = make_double2(0.0, 0.0);
        if (j < m) {
            const int kk = R.k[j], k = kk >> 1;
            uv = make_double2(R.u[j], R.v[j]);
            touch = kk & 1;
            io.suv[row0 + j] = uv;
            io.sp[row0 + j] = touch ? k : ~k;
        }
        int tot;
        const int pos = run + t.excl_scan(touch ? 1 : 0, &tot);
        if (touch) { io.tuv[row0 + pos] = uv; io.tpos[row0 + pos] = j; }
        run += tot;
    }
    t.sync();
}

// shared-memory sort buffers of `cap` keys, A then B, from `p`
__device__ __forceinline__ void carve(unsigned char *p, int cap, Keys &A, Keys &B) {
    double *d = reinterpret_cast<double *>(p);
    int32_t *k = reinterpret_cast<int32_t *>(d + 4 * cap);
    A = Keys{d, d + cap, k};
    B = Keys{d + 2 * cap, d + 3 * cap, k + cap};
}

constexpr size_t FW_BYTES_PER_WARP = (size_t)FW_SMEM * 2 * (8 + 8 + 4) + 9 * 33 * 8;
#ifndef FB_SMEM_DEF
#define FB_SMEM_DEF 768  // measured: 1024 -> 5 CTAs/SM by shared memory, 768 -> 7: step -0.05 ms (640: -0.04, 512: +0.01)
#endif
constexpr int FB_SMEM = FB_SMEM_DEF;  // members a k_fin_sort_block CTA sorts in shared memory
constexpr size_t FB_BYTES = (size_t)FB_SMEM * 2 * (8 + 8 + 4);

// Patches of <= FW_SMEM members: one warp each.
#ifndef FW_MINB
#define FW_MINB 6  // 4 x 6 warps per SM at <= 85 registers (measured: 8 warps x 3 CTAs at 80: +0.03 ms; 4 x 8: +0.007; 4 x 10: +0.04)
#endif
__global__ void __launch_bounds__(FW_WARPS * 32, FW_MINB) k_fin_sort_warp(ReduceIO io, ReduceParams p) {
    extern __shared__ __align__(16) unsigned char dyn[];
    const int wib = threadIdx.x >> 5;
    unsigned char *mine = dyn + wib * FW_BYTES_PER_WARP;
    Keys A, B;
    carve(mine, FW_SMEM, A, B);
    double *tile = reinterpret_cast<double *>(mine + (size_t)FW_SMEM * 40);
    WarpTeam t{nullptr};
    const int64_t E = io.E;
    const int total = io.patch_off[E];
    for (int w = blockIdx.x * FW_WARPS + wib; w < total; w += gridDim.x * FW_WARPS) {
        const int64_t e = io.wenv[w];
        const int q = w - io.patch_off[e];
        const int32_t *mo = io.member_offsets + e * (p.N + 1);
        if (mo[q + 1] - mo[q] > FW_SMEM) continue;  // the CTA path's (k_patch_env listed it)
        sort_patch<true>(t, io, p, w, e, q, A, B, tile);
    }
}

// Larger patches: one CTA each; shared memory up to FB_SMEM members, global scratch rows beyond.
__global__ void __launch_bounds__(FB_THREADS) k_fin_sort_block(ReduceIO io, ReduceParams p) {
    extern __shared__ __align__(16) unsigned char dyn[];
    __shared__ ArgMax s_am[32];
    __shared__ double s_dred[32];
    __shared__ int s_ired[32];
    __shared__ int s_ws[WS_INTS];
    BlockTeam t{s_am, s_dred, s_ired, s_ws};
    const int64_t E = io.E;
    const int total = *io.large_count;
    for (int li = blockIdx.x; li < total; li += gridDim.x) {
        const int w = io.large_list[li];
        const int64_t e = io.wenv[w];
        const int q = w - io.patch_off[e];
        const int32_t *mo = io.member_offsets + e * (p.N + 1);
        Keys A, B;
        if (mo[q + 1] - mo[q] <= FB_SMEM) {
            carve(dyn, FB_SMEM, A, B);
        } else {
            const int64_t row0 = io.cand_base[e] + mo[q];
            A = Keys{io.su + row0, io.sv + row0, io.sp + row0};
            B = Keys{io.tu + row0, io.tv + row0, io.tk + row0};
        }
        sort_patch<false>(t, io, p, w, e, q, A, B, nullptr);
    }
}

// The sequential sums of the larger patches (reduction.py:162-165), one warp per patch
// (k_fin_sort_block leaves them out: 9 lanes folding while the CTA waits at a barrier
// was a third of its time). Per chunk of 32 members the warp loads the rows (one
// member per lane, the next chunk's loads in flight), writes the nine weighted
// products (np.cross(pts, norms) * w etc.) to a shared tile, and lanes 0..8 fold
// the tile in member order (numpy's axis-0 sums add row after row); the weights
// are kept for lane 9's pairwise sum.
constexpr int FL_WARPS = 4;
#ifndef FOLD_TILE_STRIDE
#define FOLD_TILE_STRIDE 33
#endif
constexpr int FT = FOLD_TILE_STRIDE;  // tile row stride (doubles)
constexpr int FL_W = 1024;  // weights per warp in shared memory (larger patches: global scratch)

__global__ void __launch_bounds__(FL_WARPS * 32) k_fin_fold_large(ReduceIO io, ReduceParams p) {
    __shared__ double s_tile[FL_WARPS][9 * FT];
    __shared__ double s_w[FL_WARPS][FL_W];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    double *tile = s_tile[wib];
    const int64_t E = io.E;
    const int total = *io.large_count;
    for (int li = blockIdx.x * FL_WARPS + wib; li < total; li += gridDim.x * FL_WARPS) {
        const int w = io.large_list[li];
        const int64_t e = io.wenv[w];
        const int q = w - io.patch_off[e];
        const int64_t base = io.cand_base[e];
        const int32_t *mo = io.member_offsets + e * (p.N + 1);
        const int moff = mo[q], m = mo[q + 1] - moff;
        const int32_t *mem = io.members + base + moff;
        const double *P = io.point + 3 * base, *Nn = io.normal + 3 * base, *D = io.depth + base;
        const int64_t pq = e * p.N + q;
        double *wb = m <= FL_W ? s_w[wib] : io.fw + base + moff;
        double fd = 0.0, fpx = 0.0, fpy = 0.0, fpz = 0.0, fnx = 0.0, fny = 0.0, fnz = 0.0;
        auto fetch = [&](int k) {
            if (k < m) {
                const int64_t i = __ldg(mem + k);
                fd = __ldg(D + i);
                fpx = __ldg(P + 3 * i); fpy = __ldg(P + 3 * i + 1); fpz = __ldg(P + 3 * i + 2);
                fnx = __ldg(Nn + 3 * i); fny = __ldg(Nn + 3 * i + 1); fnz = __ldg(Nn + 3 * i + 2);
            }
        };
        fetch(lane);
        double s = 0.0;
        for (int c0 = 0; c0 < m; c0 += 32) {
            const int k = c0 + lane;
            if (k < m) {
                const double px = fpx, py = fpy, pz = fpz, nx = fnx, ny = fny, nz = fnz;
                const double wk = weight_of(fd);
                fetch(k + 32);
                wb[k] = wk;
                tile[0 * FT + lane] = px * wk; tile[1 * FT + lane] = py * wk; tile[2 * FT + lane] = pz * wk;
                tile[3 * FT + lane] = nx * wk; tile[4 * FT + lane] = ny * wk; tile[5 * FT + lane] = nz * wk;
                tile[6 * FT + lane] = (py * nz - pz * ny) * wk;
                tile[7 * FT + lane] = (pz * nx - px * nz) * wk;
                tile[8 * FT + lane] = (px * ny - py * nx) * wk;
            }
            __syncwarp();
            if (lane < 9) {  // lane l folds tile row l (rows FT doubles apart: distinct banks)
                const int cnt = min(32, m - c0);
                const double *row = tile + lane * FT;
                int j = 0;
                if (c0 == 0) { s = row[0]; j = 1; }
#pragma unroll 8
                for (; j < cnt; ++j) s = s + row[j];
            }
            __syncwarp();
        }
        if (lane < 9) {
            const int kind = lane / 3, c = lane % 3;
            double *o = (kind == 0 ? io.wp_sum : kind == 1 ? io.wn_sum : io.wt_sum) + 3 * pq;
            o[c] = s;
        } else if (lane == 9) {
            io.w_sum[pq] = 0.0 + pairwise([&](int k) { return wb[k]; }, 0, m);
        }
        __syncwarp();
    }
}

// ------------------------------------------------------------------ stage 2: chains


constexpr int CH_WARPS = 4;   // warps per k_fin_chain CTA
#ifndef CH_CG
#define CH_CG 8  // measured best: 4 lanes (8 chains per warp) is 3% slower
#endif
constexpr int CG = CH_CG;     // lanes per half chain: pops tested per round
constexpr int NG = 32 / CG;   // half chains per warp
constexpr int CS = 64;        // stack entries per half chain in shared memory

// One half of _monotone_hull (reduction.py:214-223) by one thread with its stack in
// global memory: the fallback for the rare chains whose stack outgrows CS.
__device__ int half_chain_global(const double2 *kuv, const int32_t *kpos, int L, int dir, int32_t *hj, double *hu,
                                 double *hv) {
    int top = 0;
    for (int x = 0; x < L; ++x) {
        const int s = dir > 0 ? x : L - 1 - x;
        const double2 b = kuv[s];
        while (top >= 2) {
            const double ou = hu[top - 2], ov = hv[top - 2], au = hu[top - 1], av = hv[top - 1];
            if (!((au - ou) * (b.y - ov) - (av - ov) * (b.x - ou) <= 0.0)) break;  // NaN: no pop (Python)
            --top;
        }
        hu[top] = b.x; hv[top] = b.y; hj[top] = kpos ? kpos[s] : s;
        ++top;
    }
    return top;
}

// ONE 8-LANE GROUP PER HALF CHAIN of _monotone_hull (reduction.py:214-223), four
// chains per warp. Job 4w + kind: kind 0/1 the lower/upper chain over patch w's
// sorted members (the hull area), 2/3 over its touching members (the kept
// selection; k_fin_sort wrote them compacted, in sorted order, with their sorted
// positions). Jobs come bucketed by chain length, longest first; a warp takes four
// consecutive ones, so its groups step through chains of similar length.
//
// A chain is sequential in its keys but not in the pops of one key: the sequential
// loop tests cross(h[top-2-i], h[top-1-i], b) for i = 0, 1, ... on the unchanged
// stack below, stopping at the first positive one. Lane i of a group reads stack
// entries top-1-i and top-2-i and evaluates that same test, and a ballot gives the
// number of pops, so a key costs one round whatever it pops (measured: at most 8
// pops per key on the headline workload; more take further rounds). The stack
// ((u, v) and sorted position) lives in shared memory; pushing is one store.
// Measured stacks stay under 26 entries; a chain that would exceed CS is redone by
// one thread with a global stack (half_chain_global). Keys stream from the sorted
// rows, each lane prefetching every 8th key one octet ahead. The stack is the half
// hull.
__global__ void __launch_bounds__(CH_WARPS * 32) k_fin_chain(ReduceIO io, ReduceParams p) {
    __shared__ double2 s_st[CH_WARPS * NG][CS];
    __shared__ int32_t s_stp[CH_WARPS * NG][CS];
    __shared__ int bstart[CH_BUCKETS + 1];
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int g = lane / CG, li = lane & (CG - 1), gb = g * CG;
    double2 *st = s_st[wib * NG + g];
    int32_t *stp = s_stp[wib * NG + g];
    if (threadIdx.x == 0) {
        int r = 0;
        for (int k = 0; k < CH_BUCKETS; ++k) { bstart[k] = r; r += io.njob[k]; }
        bstart[CH_BUCKETS] = r;
    }
    __syncthreads();
    const int ntot = bstart[CH_BUCKETS];
    const int64_t bcap = 4 * io.E * (int64_t)p.N;
    while (true) {
        int base = 0;
        if (lane == 0) base = atomicAdd(io.njob + CH_BUCKETS, NG);
        base = __shfl_sync(FULL, base, 0);
        if (base >= ntot) break;
        // this group's chain: job base + g (4 consecutive jobs: similar lengths)
        const int idx = base + g;
        bool run = idx < ntot;
        int w = 0, kind = 0, L = 0, m = 0;
        int64_t row0 = 0;
        if (run) {
            int k = 0;
            for (int sz = CH_BUCKETS / 2; sz > 0; sz >>= 1)  // last k with bstart[k] <= idx
                if (bstart[k + sz] <= idx) k += sz;
            const int jw = io.jobs[k * bcap + idx - bstart[k]];
            w = jw >> 2;
            kind = jw & 3;
            const int64_t e = io.wenv[w];
            const int q = w - io.patch_off[e];
            const int32_t *mo = io.member_offsets + e * (p.N + 1);
            m = mo[q + 1] - mo[q];
            row0 = io.cand_base[e] + mo[q];
            L = kind < 2 ? m : io.pnt[w];
        }
        const int dir = (kind & 1) ? -1 : 1;
        const double2 *kuv = kind < 2 ? io.suv + row0 : io.tuv + row0;
        const int32_t *kpos = kind < 2 ? nullptr : io.tpos + row0;
        int Lmax = 0;
#pragma unroll
        for (int gg = 0; gg < NG; ++gg) Lmax = max(Lmax, __shfl_sync(FULL, L, gg * CG));
        // key x of the chain (index clamped into the list: no branch around the loads)
        auto key = [&](int x, double &u, double &v, int &ps) {
            const int c = min(x, L - 1);
            const int sidx = max(dir > 0 ? c : L - 1 - c, 0);  // L == 0: row 0, unused
            const double2 uv = __ldg(kuv + sidx);
            u = uv.x; v = uv.y;
            ps = kpos ? __ldg(kpos + sidx) : sidx;
        };
        double cu, cv, nu_ = 0.0, nv_ = 0.0;
        int cp, np_ = 0;
        key(li, cu, cv, cp);
        int top = 0;
        bool ovf = false;  // the stack outgrew CS: redone by half_chain_global
        // one octet of keys per outer iteration, the inner loop unrolled: the key of step
        // c comes from lane gb + c of the group (a constant shuffle source), and the next
        // octet's loads go out at the octet's start
        for (int t0 = 0; t0 < Lmax; t0 += CG) {
            if (t0 + CG < Lmax) key(t0 + CG + li, nu_, nv_, np_);
#pragma unroll
            for (int c = 0; c < CG; ++c) {
                const int t = t0 + c;
                if (t >= Lmax) break;
                const double ub = __shfl_sync(FULL, cu, gb + c), vb = __shfl_sync(FULL, cv, gb + c);
                const int pb = __shfl_sync(FULL, cp, gb + c);
                const bool act = t < L && !ovf;
                bool more = act;
                while (true) {
                    // lane li: o = h[top-2-li], a = h[top-1-li];
                    // cross(o, a, b) = (a.u - o.u)(b.v - o.v) - (a.v - o.v)(b.u - o.u)
                    bool popi = false;
                    if (more && top - li >= 2) {
                        const double2 a = st[top - 1 - li], o = st[top - 2 - li];
                        popi = (a.x - o.x) * (vb - o.y) - (a.y - o.y) * (ub - o.x) <= 0.0;  // NaN: no pop (Python)
                    }
                    // pops = the group's first non-popping lane (a sentinel above the group's
                    // bits: CG when all pop; 0 when the group is done, its lanes do not pop)
                    const int npop = __ffs((__ballot_sync(FULL, !popi) >> gb) | (1u << CG)) - 1;
                    top -= npop;
                    more = npop == CG;
                    if (!__any_sync(FULL, more)) break;
                }
                __syncwarp();  // the pop rounds' stack reads are ordered before the push (memory model)
                if (act) {  // push b
                    if (top < CS) {
                        if (li == 0) { st[top] = make_double2(ub, vb); stp[top] = pb; }
                        ++top;
                    } else {
                        ovf = true;
                    }
                }
                __syncwarp();
            }
            cu = nu_; cv = nv_; cp = np_;
        }
        if (run) {  // the stack is the half hull (sorted positions)
            const int64_t h0 = 4 * row0 + (int64_t)kind * m;
            int32_t *hj = io.hj + h0;
            if (!ovf) {
                for (int j = li; j < top; j += CG) hj[j] = stp[j];
            } else if (li == 0) {
                top = half_chain_global(kuv, kpos, L, dir, hj, io.hu + h0, io.hv + h0);
            }
            if (li == 0) io.hlen[4 * (int64_t)w + kind] = top;
        }
        __syncwarp();
    }
}

// ------------------------------------------------------------------ stage 4: kept selection

__device__ __forceinline__ int dec_k(int k) { return k < 0 ? ~k : k; }

// hull = lower[:-1] + upper[:-1] as sorted positions
struct HullView {
    const int32_t *lo, *up;
    int L, H;
    __device__ int at(int h) const { return h < L - 1 ? __ldg(lo + h) : __ldg(up + h - (L - 1)); }
};

// One patch per warp: hull assembly, kept selection (reduction.py:172-199), hull
// area (reduction.py:227-236), the kept rows.
constexpr int KH = 256;  // hull entries a k_fin_kept warp stages in shared memory (longer hulls: read in place)

__device__ void kept_patch(const WarpTeam &t, const ReduceIO &io, const ReduceParams &p, int w, int *chosen,
                           double2 *huv, int *hk) {
    const int N = p.N, K = p.K;
    const int64_t e = io.wenv[w];
    const int q = w - io.patch_off[e];
    const int64_t base = io.cand_base[e];
    const int32_t *mo = io.member_offsets + e * (N + 1);
    const int moff = mo[q], m = mo[q + 1] - moff;
    const int32_t *mem = io.members + base + moff;
    const int64_t pq = e * N + q, row0 = base + moff;
    const double *P = io.point + 3 * base, *Nn = io.normal + 3 * base, *D = io.depth + base;
    const double2 *suv = io.suv + row0;
    const int32_t *sk = io.sp + row0, *hj = io.hj + 4 * row0;
    const int nt = io.pnt[w], deepest = io.pdeep[w];
    const int4 len = *reinterpret_cast<const int4 *>(io.hlen + 4 * (int64_t)w);
    const int lane = t.rank();
    double area = 0.0;
    if (m >= 3) {
        const HullView h{hj, hj + m, len.x, (len.x - 1) + (len.y - 1)};
        const int H = h.H;
        if (H >= 3 && H <= KH) {  // the hull's (u, v) staged by the warp; lanes 0 and 1 run the two dots
            for (int k = lane; k < H; k += 32) huv[k] = suv[h.at(k)];
            __syncwarp();
            if (lane < 2) {  // lane 0: d1 = x . roll(y, -1), lane 1: d2 = y . roll(x, -1) (same code, own data)
                const double *hd = reinterpret_cast<const double *>(huv);
                const double d = ddot_x2(H, [&](int k) { return hd[2 * k + lane]; },
                                         [&](int k) { return hd[2 * (k + 1 == H ? 0 : k + 1) + 1 - lane]; });
                const double d2 = __shfl_sync(0x3u, d, 1);
                if (lane == 0) area = 0.5 * fabs(d - d2);
            }
            __syncwarp();
        } else if (H >= 3 && lane == 0) {
            const double d1 = ddot_x2(H, [&](int k) { return suv[h.at(k)].x; }, [&](int k) { return suv[h.at((k + 1) % H)].y; });
            const double d2 = ddot_x2(H, [&](int k) { return suv[h.at(k)].y; }, [&](int k) { return suv[h.at((k + 1) % H)].x; });
            area = 0.5 * fabs(d1 - d2);
        }
    }
    int nc;
    if (m <= K) {
        for (int k = lane; k < m; k += 32) chosen[k] = k;
        nc = m;
    } else {
        const HullView hb = needs_touch_hull(m, nt, K)  // base = touching members, else all
                                ? HullView{hj + 2 * m, hj + 3 * m, len.z, (len.z - 1) + (len.w - 1)}
                                : HullView{hj, hj + m, len.x, (len.x - 1) + (len.y - 1)};
        const bool staged = hb.H <= KH;  // the hull's members staged by the warp
        if (staged) {
            for (int k = lane; k < hb.H; k += 32) hk[k] = dec_k(sk[hb.at(k)]);
            __syncwarp();
        }
        if (lane == 0) {
            struct {
                const HullView &h;
                const int32_t *sk;
                const int *hk;
                bool staged;
                __device__ int at(int j) const { return staged ? hk[j] : dec_k(sk[h.at(j)]); }
                int H;
            } h{hb, sk, hk, staged, hb.H};
            int nh = 0;  // hull members other than the deepest
            for (int j = 0; j < h.H; ++j) nh += h.at(j) != deepest;
            chosen[0] = deepest;
            int c = 1;
            if (nh <= K - 1) {
                for (int j = 0; j < h.H; ++j) {
                    const int k = h.at(j);
                    if (k != deepest) chosen[c++] = k;
                }
            } else {  // picks = linspace(0, len(hull), K-1, endpoint=False).astype(int), strictly increasing
                const double step = (double)nh / (double)(K - 1);
                int f = -1, j = -1, k = -1;  // f: position among the non-deepest hull members
                for (int pk = 0; pk < K - 1; ++pk) {
                    const int target = (int)((double)pk * step + 0.0);
                    while (f < target) {
                        k = h.at(++j);
                        if (k != deepest) ++f;
                    }
                    chosen[c++] = k;
                }
            }
            t.misc[0] = c;
        }
        t.sync();
        nc = t.misc[0];
        t.sync();
        while (nc < K) {  // fill by np.argsort(-depths, kind="stable"), skipping chosen
            int bk = -1;
            double bd = 0.0;
            for (int k = lane; k < m; k += 32) {
                bool in = false;
                for (int j = 0; j < nc; ++j) in |= (chosen[j] == k);
                if (in) continue;
                const double d = __ldg(D + mem[k]);
                if (bk < 0 || depth_before(d, k, bd, bk)) { bk = k; bd = d; }
            }
            t.best_depth(bk, bd);
            if (bk < 0) break;
            if (lane == 0) chosen[nc] = bk;
            t.sync();
            ++nc;
        }
    }
    t.sync();
    const int nk = nc < K ? nc : K;
    if (lane == 0) {
        io.area[pq] = area;
        io.patch_nkept[pq] = nk;
    }
    for (int j = lane; j < K; j += 32) {
        const int64_t o = pq * K + j;
        if (j < nk) {
            const int k = chosen[j];
            const int i = mem[k];
            io.kept_cand[o] = i;
            io.kept_face[o] = io.face ? io.face[base + i] : -1;
            io.kept_depth[o] = __ldg(D + i);
            for (int c = 0; c < 3; ++c) {
                io.kept_point[3 * o + c] = __ldg(P + 3 * (int64_t)i + c);
                io.kept_normal[3 * o + c] = __ldg(Nn + 3 * (int64_t)i + c);
            }
        } else {
            io.kept_cand[o] = -1;
            io.kept_face[o] = -1;
            io.kept_depth[o] = 0.0;
            for (int c = 0; c < 3; ++c) { io.kept_point[3 * o + c] = 0.0; io.kept_normal[3 * o + c] = 0.0; }
        }
    }
    t.sync();
}

constexpr int FK_WARPS = 4;

__global__ void __launch_bounds__(FK_WARPS * 32) k_fin_kept(ReduceIO io, ReduceParams p) {
    __shared__ int s_chosen[FK_WARPS][MAX_KEPT];
    __shared__ int s_misc[FK_WARPS][4];
    __shared__ double2 s_huv[FK_WARPS][KH];
    __shared__ int s_hk[FK_WARPS][KH];
    const int wib = threadIdx.x >> 5;
    WarpTeam t{s_misc[wib]};
    const int total = io.patch_off[io.E];
    for (int w = blockIdx.x * FK_WARPS + wib; w < total; w += gridDim.x * FK_WARPS)
        kept_patch(t, io, p, w, s_chosen[wib], s_huv[wib], s_hk[wib]);
}

// Per env stats, one warp per env (lanes over the patches).
__global__ void k_stats(ReduceIO io, ReduceParams p) {
    const int64_t e = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (e >= io.E) return;
    const int N = p.N, K = p.K;
    const int P = io.n_patch[e];
    int nk = 0;
    double mx = 0.0;  // StepReport.max_penetration = max(max(depth, 0)) (scene.py:160-161)
    for (int q = lane; q < P; q += 32) {
        const int k = io.patch_nkept[e * N + q];
        nk += k;
        for (int j = 0; j < k; ++j) {
            const double d = io.kept_depth[(e * N + q) * K + j];
            if (d > mx) mx = d;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        nk += __shfl_xor_sync(0xffffffffu, nk, o);
        const double om = __shfl_xor_sync(0xffffffffu, mx, o);
        if (om > mx) mx = om;
    }
    if (lane == 0) {
        io.n_kept[e] = nk;
        io.stats[4 * e + 0] = (float)io.n_cand[e];
        io.stats[4 * e + 1] = (float)P;
        io.stats[4 * e + 2] = (float)nk;
        io.stats[4 * e + 3] = (float)mx;
    }
}

void launch_finalize(const ReduceIO &io, const ReduceParams &p, int sm_count, cudaStream_t s, const FinFork *fk) {
    if (io.E <= 0) return;
    k_patch_off<<<1, 1024, 0, s>>>(io.E, io.n_patch, io.patch_off, io.large_count, io.njob);
    k_patch_env<<<(unsigned)((io.E * 32 + 255) / 256), 256, 0, s>>>(io.E, p.N, io.n_patch, io.patch_off,
                                                                     io.member_offsets, io.wenv, io.large_list,
                                                                     io.large_count);
    const int64_t maxw = io.E * (int64_t)p.N;
    const size_t wsm = FW_BYTES_PER_WARP * FW_WARPS;
    // per device, and only once both raises succeeded (a failed raise leaves the launch
    // to report the error)
    static bool configured[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!configured[dev & 63] &&
        cudaFuncSetAttribute(k_fin_sort_warp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wsm) == cudaSuccess &&
        cudaFuncSetAttribute(k_fin_sort_block, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)FB_BYTES) == cudaSuccess)
        configured[dev & 63] = true;
    auto cap = [&](int64_t want, int64_t limit) { return (unsigned)(want < limit ? want : limit); };
    // The three stage-1 kernels are independent (k_patch_env wrote the work lists): with
    // a fork they run as concurrent branches (graph branches when captured), so the
    // CTA-per-patch sort and the sequential sums fill each other's tails. The chains
    // need both sorts; the sums join before the stats.
    cudaStream_t sb = s, sf = s;
    if (fk) {
        cudaEventRecord(fk->ev_fork, s);
        cudaStreamWaitEvent(fk->s_block, fk->ev_fork, 0);
        cudaStreamWaitEvent(fk->s_fold, fk->ev_fork, 0);
        sb = fk->s_block;
        sf = fk->s_fold;
    }
    // launch order (measured, graph replay): the CTA-per-patch sort first, then the
    // warp-per-patch sort, then the folds: 3.164 ms; folds / block / warp: 3.190 ms
    k_fin_sort_block<<<cap((int64_t)sm_count * 4 * FIN_GRID, maxw), FB_THREADS, FB_BYTES, sb>>>(io, p);
    k_fin_sort_warp<<<cap((int64_t)sm_count * 8 * FIN_GRID, (maxw + FW_WARPS - 1) / FW_WARPS), FW_WARPS * 32, wsm, s>>>(io, p);
    k_fin_fold_large<<<cap((int64_t)sm_count * 4 * FIN_GRID, (maxw + FL_WARPS - 1) / FL_WARPS), FL_WARPS * 32, 0, sf>>>(io, p);
    if (fk) {
        cudaEventRecord(fk->ev_block, sb);
        cudaStreamWaitEvent(s, fk->ev_block, 0);
    }
    k_fin_chain<<<cap((int64_t)sm_count * 8 * FIN_GRID_CHAIN, (maxw + CH_WARPS - 1) / CH_WARPS), CH_WARPS * 32, 0, s>>>(io, p);
    k_fin_kept<<<cap((int64_t)sm_count * 8 * FIN_GRID, (maxw + FK_WARPS - 1) / FK_WARPS), FK_WARPS * 32, 0, s>>>(io, p);
    if (fk) {
        cudaEventRecord(fk->ev_fold, sf);
        cudaStreamWaitEvent(s, fk->ev_fold, 0);
    }
    k_stats<<<(unsigned)((io.E * 32 + 255) / 256), 256, 0, s>>>(io, p);
}

}  // namespace cs
