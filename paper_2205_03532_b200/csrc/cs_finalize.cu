// Per-patch finalisation on sm_100a (reduction.py:146-236).
//
//   k_patch_off     exclusive scan of patch counts -> work list [E+1].
//   k_finalize<W>   ONE WARP PER PATCH for patches of <= FIN_SMALL members
//                   (~95% of patches): the (u, v, pos) sort keys and the chain
//                   stack live in this warp's slice of shared memory; member rows
//                   are read through the read-only path. Warps never block each
//                   other, so an SM keeps ~20 patches in flight and the inherently
//                   sequential parts (monotone chain, axis-0 folds) overlap.
//   k_finalize<B>   ONE CTA PER PATCH for larger patches (shared memory up to
//                   FIN_LARGE members, global scratch beyond).
//   k_stats         per env stats (the multi-GPU all-gather payload).
// Both paths run the same templated per-patch code (finalize_patch) over a
// "team" (warp or block) abstraction, so they produce identical bits.
#include <stdint.h>

#include "cs_reduce_util.cuh"

namespace cs {

constexpr int FIN_SMALL = 512;        // members per warp-path patch
constexpr int FIN_WARPS = 2;          // warp teams per CTA (small path)
constexpr int FIN_LARGE = 1024;       // members per CTA-path patch held in shared memory
constexpr int FIN_LARGE_THREADS = 256;

__global__ void k_patch_off(int64_t E, const int32_t *__restrict__ n_patch, int32_t *__restrict__ off,
                            int32_t *__restrict__ large_count) {
    __shared__ int ws[WS_INTS];
    if (threadIdx.x == 0) *large_count = 0;
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
    __device__ bool any(bool b) const { return __any_sync(0xffffffffu, b); }
    __device__ int bcast(int v) const { return __shfl_sync(0xffffffffu, v, 0); }
    __device__ double bcast(double v) const { return __shfl_sync(0xffffffffu, v, 0); }
    // best (bk, bd) under depth_before over the team
    __device__ void best_depth(int &bk, double &bd) const {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            int ok = __shfl_xor_sync(0xffffffffu, bk, o);
            double od = __shfl_xor_sync(0xffffffffu, bd, o);
            if (ok >= 0 && (bk < 0 || depth_before(od, ok, bd, bk))) { bk = ok; bd = od; }
        }
    }
    template <class Idx, class Pred>
    __device__ int compact(int m, Pred pred, Idx *out) const {
        const unsigned lt = (1u << rank()) - 1u;
        int running = 0;
        for (int c0 = 0; c0 < m; c0 += 32) {
            int k = c0 + rank();
            bool f = k < m && pred(k);
            unsigned b = __ballot_sync(0xffffffffu, f);
            if (f) out[running + __popc(b & lt)] = (Idx)k;
            running += __popc(b);
        }
        __syncwarp();
        return running;
    }
};

struct BlockTeam {
    int *misc;        // >= 4 ints
    ArgMax *am;       // 32 entries
    int *ws;          // WS_INTS
    double *dred;     // 32 doubles
    int *ired;        // 32 ints
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
    __device__ bool any(bool b) const { return __syncthreads_or(b) != 0; }
    __device__ int bcast(int v) const {
        if (threadIdx.x == 0) misc[3] = v;
        __syncthreads();
        int r = misc[3];
        __syncthreads();
        return r;
    }
    __device__ double bcast(double v) const {
        if (threadIdx.x == 0) dred[31] = v;
        __syncthreads();
        double r = dred[31];
        __syncthreads();
        return r;
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
    template <class Idx, class Pred>
    __device__ int compact(int m, Pred pred, Idx *out) const {
        int running = 0;
        for (int c0 = 0; c0 < m; c0 += blockDim.x) {
            int k = c0 + threadIdx.x;
            int f = (k < m && pred(k)) ? 1 : 0;
            int tot;
            int pos = running + block_excl_scan(f, ws, &tot);
            if (f) out[pos] = (Idx)k;
            running += tot;
        }
        return running;
    }
};

// All-ascending bitonic sort of m (u, v, pos) keys by a team (virtual +inf padding).
template <class Team, class Idx>
__device__ void team_sort(const Team &t, double *su, double *sv, Idx *sp, int m) {
    int P2 = 1, lg = 0;
    while (P2 < m) { P2 <<= 1; ++lg; }
    const int half = P2 >> 1;
    for (int lk = 1; lk <= lg; ++lk) {  // k = 2^lk
        const int k = 1 << lk, hk = k >> 1;
        for (int lj = lk - 1; lj >= 0; --lj) {  // jj = 2^lj
            const int jj = 1 << lj;
            for (int idx = t.rank(); idx < half; idx += t.size()) {
                int i, j;
                if (jj == hk) {  // first step of a merge: mirrored partner
                    const int blk = idx >> lj, off = idx & (jj - 1);
                    i = (blk << lk) + off;
                    j = (blk << lk) + k - 1 - off;
                } else {
                    const int blk = idx >> lj, off = idx & (jj - 1);
                    i = (blk << (lj + 1)) + off;
                    j = i + jj;
                }
                if (j < m) {
                    double ui = su[i], uj = su[j], vi = sv[i], vj = sv[j];
                    int pi = sp[i], pj = sp[j];
                    if (key_less(uj, vj, pj, ui, vi, pi)) {
                        su[i] = uj; su[j] = ui; sv[i] = vj; sv[j] = vi; sp[i] = (Idx)pj; sp[j] = (Idx)pi;
                    }
                }
            }
            t.sync();
        }
    }
}

// One half of Andrew's monotone chain (reduction.py:214-223) over the sorted keys:
// dir > 0 is the lower chain (ascending), dir < 0 the upper one (descending).
// The two stack-top points are cached in registers, so a step costs one cross
// product; the stack itself (indices) is only reloaded on a pop. Returns length.
template <class Idx>
__device__ int half_chain(const double *su, const double *sv, int m, int dir, Idx *h) {
    int top = 0;
    double ua = 0.0, va = 0.0, ub = 0.0, vb = 0.0;  // h[top-2], h[top-1]
    for (int t = 0; t < m; ++t) {
        const int s = dir > 0 ? t : m - 1 - t;
        const double us = su[s], vs = sv[s];
        while (top >= 2) {
            // cross(o, a, b) = (a.u - o.u)(b.v - o.v) - (a.v - o.v)(b.u - o.u), o = h[top-2], a = h[top-1]
            const double cr = (ub - ua) * (vs - va) - (vb - va) * (us - ua);
            if (cr > 0.0) break;
            --top;
            ub = ua; vb = va;
            if (top >= 2) { const int o = h[top - 2]; ua = su[o]; va = sv[o]; }
        }
        h[top] = (Idx)s;
        ua = ub; va = vb;
        ub = us; vb = vs;
        ++top;
    }
    return top;
}

// _monotone_hull: lower and upper chains run concurrently in ranks 0 and 1, then
// hull = lower[:-1] + upper[:-1] is assembled in h[0..H). h needs 2m + 4 entries.
template <class Team, class Idx>
__device__ int team_chain(const Team &t, const double *su, const double *sv, int m, Idx *h) {
    const int r = t.rank();
    int len = 0;
    if (r < 2) len = half_chain(su, sv, m, r == 0 ? 1 : -1, h + (r == 0 ? 0 : m + 1));
    if (r == 0) t.misc[1] = len;
    if (r == 1) t.misc[2] = len;
    t.sync();
    const int L = t.misc[1], U = t.misc[2];
    t.sync();
    if (r == 0)  // upper[:-1] after lower[:-1] (ascending copy: the ranges overlap downwards only)
        for (int j = 0; j < U - 1; ++j) h[L - 1 + j] = h[m + 1 + j];
    t.sync();
    return (L - 1) + (U - 1);
}

template <class Idx>
__device__ double chain_area(const double *su, const double *sv, const Idx *h, int H) {
    double d1 = ddot_x2(H, [&](int k) { return su[h[k]]; }, [&](int k) { return sv[h[(k + 1) % H]]; });
    double d2 = ddot_x2(H, [&](int k) { return sv[h[k]]; }, [&](int k) { return su[h[(k + 1) % H]]; });
    return 0.5 * fabs(d1 - d2);
}

// the member weights, for numpy's pairwise summation
struct WeightBuf {
    const double *d;  // staged member depths; the weight is max(depth, 0)
    __device__ double operator()(int k) const { return weight_of(d[k]); }
};

// One patch (reduction.py:146-199). su/sv/sp/sh/wbuf: team-private scratch of >= m
// (wbuf holds the member depths once gathered)
// entries (sh: >= 2m + 4; su: >= 9 x team size); chosen: MAX_KEPT ints.
template <class Team, class Idx>
__device__ void finalize_patch(const Team &t, const ReduceIO &io, const ReduceParams &p, int64_t e, int q,
                               double *su, double *sv, Idx *sp, Idx *sh, double *wbuf, int *chosen) {
    const int N = p.N, K = p.K;
    const int64_t base = io.cand_base[e];
    const int32_t *moffp = io.member_offsets + e * (N + 1);
    const int moff = moffp[q];
    const int m = moffp[q + 1] - moff;
    const int32_t *mem = io.members + base + moff;
    const int64_t pq = e * N + q;
    const double *P = io.point + 3 * base, *Nn = io.normal + 3 * base, *D = io.depth + base;
    auto dep = [&](int k) { return __ldg(D + mem[k]); };
    auto pt = [&](int k, int c) { return __ldg(P + 3 * (int64_t)mem[k] + c); };
    auto nr = [&](int k, int c) { return __ldg(Nn + 3 * (int64_t)mem[k] + c); };

    // deepest (first argmax), NaN-propagating max
    ArgMax am = {0.0, -1, 0};
    double mx = -INFINITY;
    bool anynan = false;
    for (int k = t.rank(); k < m; k += t.size()) {
        const double d = dep(k);
        wbuf[k] = d;
        am = argmax_combine(am, ArgMax{d, k, 1});
        anynan |= isnan(d);
        if (d > mx) mx = d;
    }
    am = t.argmax(am);
    const int deepest = am.i;
    mx = t.max(mx);
    anynan = t.any(anynan);

    double t1[3], t2[3];
    tangent_basis(io.patch_normal + 3 * pq, t1, t2);
    // base = touching members (depth >= 0) if >= 3 else all (reduction.py:183-184)
    t.sync();
    const int nt = t.compact(m, [&](int k) { return wbuf[k] >= 0.0; }, sp);
    const bool all_base = nt < 3 || nt == m;
    const int nb = nt < 3 ? m : nt;
    const bool need_sel = m > K;
    bool have_hull = false;
    int H = 0;
    if (need_sel || (m >= 3 && all_base)) {
        for (int j = t.rank(); j < nb; j += t.size()) {
            int k = (nt < 3) ? j : (int)sp[j];
            double x = pt(k, 0), y = pt(k, 1), z = pt(k, 2);
            su[j] = V3(x, y, z, t1[0], t1[1], t1[2]);  // _project_2d, n >= 2
            sv[j] = V3(x, y, z, t2[0], t2[1], t2[2]);
            sp[j] = (Idx)k;  // payload: member position (monotone in base order)
        }
        t.sync();
        team_sort(t, su, sv, sp, nb);
        H = team_chain(t, su, sv, nb, sh);
        have_hull = true;
    }
    double area = 0.0;
    if (t.rank() == 0 && m >= 3 && have_hull && all_base) area = H < 3 ? 0.0 : chain_area(su, sv, sh, H);
    // kept selection (reduction.py:172-199)
    int nc = 0;
    if (!need_sel) {
        for (int k = t.rank(); k < m; k += t.size()) chosen[k] = k;
        nc = m;
    } else {
        if (t.rank() == 0) {
            int nh = 0;  // hull -> member positions with the deepest excluded (in place)
            for (int h = 0; h < H; ++h) {
                int k = sp[sh[h]];
                if (k != deepest) sh[nh++] = (Idx)k;
            }
            chosen[0] = deepest;
            int c = 1;
            if (nh <= K - 1) {
                for (int h = 0; h < nh; ++h) chosen[c++] = sh[h];
            } else {  // picks = linspace(0, len(hull), K-1, endpoint=False).astype(int)
                double step = (double)nh / (double)(K - 1);
                for (int j = 0; j < K - 1; ++j) chosen[c++] = sh[(int)((double)j * step + 0.0)];
            }
            t.misc[0] = c;
        }
        t.sync();
        nc = t.misc[0];
        t.sync();
        while (nc < K) {  // fill by np.argsort(-depths, kind="stable"), skipping chosen
            int bk = -1;
            double bd = 0.0;
            for (int k = t.rank(); k < m; k += t.size()) {
                bool in = false;
                for (int j = 0; j < nc; ++j) in |= (chosen[j] == k);
                if (in) continue;
                const double d = wbuf[k];
                if (bk < 0 || depth_before(d, k, bd, bk)) { bk = k; bd = d; }
            }
            t.best_depth(bk, bd);
            if (bk < 0) break;
            if (t.rank() == 0) chosen[nc] = bk;
            t.sync();
            ++nc;
        }
    }
    t.sync();
    const int nk = nc < K ? nc : K;
    if (m >= 3 && !(have_hull && all_base)) {  // area hull over all members
        for (int j = t.rank(); j < m; j += t.size()) {
            double x = pt(j, 0), y = pt(j, 1), z = pt(j, 2);
            su[j] = V3(x, y, z, t1[0], t1[1], t1[2]);
            sv[j] = V3(x, y, z, t2[0], t2[1], t2[2]);
            sp[j] = (Idx)j;
        }
        t.sync();
        team_sort(t, su, sv, sp, m);
        const int h2 = team_chain(t, su, sv, m, sh);
        if (t.rank() == 0) area = h2 < 3 ? 0.0 : chain_area(su, sv, sh, h2);
    }
    // aggregates (reduction.py:153-168). The axis-0 sums are sequential folds (one
    // thread per component); the team streams the weighted products of each chunk
    // of members through a shared tile (su is free now) so the folds read shared
    // memory, and keeps the weights for the pairwise sum in wbuf.
    t.sync();
    const int r = t.rank(), CH = min(t.size(), 64);  // tile: 9 x CH doubles in su
    double s = 0.0;
    for (int c0 = 0; c0 < m; c0 += CH) {
        const int k = c0 + r;
        if (r < CH && k < m) {
            const double wk = weight_of(wbuf[k]);
            const double px = pt(k, 0), py = pt(k, 1), pz = pt(k, 2);
            const double nx = nr(k, 0), ny = nr(k, 1), nz = nr(k, 2);
            su[0 * CH + r] = px * wk; su[1 * CH + r] = py * wk; su[2 * CH + r] = pz * wk;
            su[3 * CH + r] = nx * wk; su[4 * CH + r] = ny * wk; su[5 * CH + r] = nz * wk;
            su[6 * CH + r] = (py * nz - pz * ny) * wk;  // np.cross(pts, norms) * w
            su[7 * CH + r] = (pz * nx - px * nz) * wk;
            su[8 * CH + r] = (px * ny - py * nx) * wk;
        }
        t.sync();
        if (r < 9) {
            const int cnt = min(CH, m - c0);
            const double *row = su + r * CH;
            for (int j = 0; j < cnt; ++j) s = (c0 + j == 0) ? row[j] : s + row[j];
        }
        t.sync();
    }
    if (r < 9) {
        const int kind = r / 3, c = r % 3;
        double *o = (kind == 0 ? io.wp_sum : kind == 1 ? io.wn_sum : io.wt_sum) + 3 * pq;
        o[c] = s;
    } else if (r == 9) {
        io.w_sum[pq] = 0.0 + pairwise(WeightBuf{wbuf}, 0, m);
    }
    if (r == 0) {
        io.max_depth[pq] = anynan ? (double)NAN : mx;
        io.area[pq] = area;
        io.patch_nkept[pq] = nk;
    }
    for (int j = r; j < K; j += t.size()) {
        const int64_t o = pq * K + j;
        if (j < nk) {
            const int k = chosen[j];
            const int i = mem[k];
            io.kept_cand[o] = i;
            io.kept_face[o] = io.face ? io.face[base + i] : -1;
            io.kept_depth[o] = wbuf[k];
            for (int c = 0; c < 3; ++c) {
                io.kept_point[3 * o + c] = pt(k, c);
                io.kept_normal[3 * o + c] = nr(k, c);
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

__device__ __forceinline__ int64_t env_of(const int32_t *patch_off, int64_t E, int w) {
    int64_t lo = 0, hi = E - 1;  // last e with patch_off[e] <= w
    while (lo < hi) {
        int64_t mid = (lo + hi + 1) >> 1;
        if (patch_off[mid] <= w) lo = mid; else hi = mid - 1;
    }
    return lo;
}

__device__ __forceinline__ int patch_size(const ReduceIO &io, int N, int64_t e, int q) {
    const int32_t *m = io.member_offsets + e * (N + 1);
    return m[q + 1] - m[q];
}

// Small patches: one warp each.
__global__ void __launch_bounds__(FIN_WARPS * 32, 10) k_finalize_warp(ReduceIO io, ReduceParams p) {
    __shared__ double s_u[FIN_WARPS][FIN_SMALL], s_v[FIN_WARPS][FIN_SMALL];
    __shared__ uint16_t s_p[FIN_WARPS][FIN_SMALL], s_h[FIN_WARPS][2 * FIN_SMALL + 4];
    __shared__ double s_w[FIN_WARPS][FIN_SMALL];
    __shared__ int s_chosen[FIN_WARPS][MAX_KEPT];
    __shared__ int s_misc[FIN_WARPS][4];
    const int wib = threadIdx.x >> 5;
    WarpTeam t{s_misc[wib]};
    const int64_t E = io.E;
    const int total = io.patch_off[E];
    for (int w = blockIdx.x * FIN_WARPS + wib; w < total; w += gridDim.x * FIN_WARPS) {
        const int64_t e = env_of(io.patch_off, E, w);
        const int q = w - io.patch_off[e];
        if (patch_size(io, p.N, e, q) > FIN_SMALL) {  // handed to the CTA path (order-free: patches are independent)
            if ((threadIdx.x & 31) == 0) io.large_list[atomicAdd(io.large_count, 1)] = w;
            continue;
        }
        finalize_patch(t, io, p, e, q, s_u[wib], s_v[wib], s_p[wib], s_h[wib], s_w[wib], s_chosen[wib]);
    }
}

// Large patches: one CTA each; shared memory up to FIN_LARGE members, global scratch beyond.
__global__ void __launch_bounds__(FIN_LARGE_THREADS) k_finalize_block(ReduceIO io, ReduceParams p) {
    extern __shared__ __align__(16) unsigned char dyn[];
    double *su = reinterpret_cast<double *>(dyn);
    double *sv = su + FIN_LARGE;
    double *sw = sv + FIN_LARGE;
    int *sp = reinterpret_cast<int *>(sw + FIN_LARGE);
    int *sh = sp + FIN_LARGE;  // 2 FIN_LARGE + 4
    __shared__ ArgMax s_am[32];
    __shared__ int s_ws[WS_INTS];
    __shared__ double s_dred[32];
    __shared__ int s_ired[32];
    __shared__ int s_misc[4];
    __shared__ int s_chosen[MAX_KEPT];
    BlockTeam t{s_misc, s_am, s_ws, s_dred, s_ired};
    const int64_t E = io.E;
    const int total = *io.large_count;
    for (int li = blockIdx.x; li < total; li += gridDim.x) {
        const int w = io.large_list[li];
        const int64_t e = env_of(io.patch_off, E, w);
        const int q = w - io.patch_off[e];
        const int m = patch_size(io, p.N, e, q);
        if (m <= FIN_LARGE) {
            finalize_patch(t, io, p, e, q, su, sv, sp, sh, sw, s_chosen);
        } else {
            const int64_t base = io.cand_base[e];
            const int moff = io.member_offsets[e * (p.N + 1) + q];
            finalize_patch(t, io, p, e, q, io.su + base + moff, io.sv + base + moff, io.sp + base + moff,
                           io.sh + 2 * base + e * (4 * (int64_t)p.N + 4) + 2 * (int64_t)moff + 4 * q,
                           io.gD + base + moff, s_chosen);
        }
    }
}

__global__ void k_stats(ReduceIO io, ReduceParams p) {
    int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= io.E) return;
    const int N = p.N, K = p.K;
    int P = io.n_patch[e], nk = 0;
    double mx = 0.0;  // StepReport.max_penetration = max(max(depth, 0)) (scene.py:160-161)
    for (int q = 0; q < P; ++q) {
        int k = io.patch_nkept[e * N + q];
        nk += k;
        for (int j = 0; j < k; ++j) {
            double d = io.kept_depth[(e * N + q) * K + j];
            if (d > mx) mx = d;
        }
    }
    io.n_kept[e] = nk;
    io.stats[4 * e + 0] = (float)io.n_cand[e];
    io.stats[4 * e + 1] = (float)P;
    io.stats[4 * e + 2] = (float)nk;
    io.stats[4 * e + 3] = (float)mx;
}

void launch_finalize(const ReduceIO &io, const ReduceParams &p, int sm_count, cudaStream_t s) {
    if (io.E <= 0) return;
    k_patch_off<<<1, 1024, 0, s>>>(io.E, io.n_patch, io.patch_off, io.large_count);
    const int64_t maxw = io.E * (int64_t)p.N;
    int64_t grid = (int64_t)sm_count * 12;
    int64_t need = (maxw + FIN_WARPS - 1) / FIN_WARPS;
    k_finalize_warp<<<(unsigned)(grid < need ? grid : need), FIN_WARPS * 32, 0, s>>>(io, p);
    const size_t smem = (size_t)FIN_LARGE * (8 + 8 + 8 + 4 + 8) + 16;
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(k_finalize_block, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        configured = true;
    }
    int64_t lgrid = (int64_t)sm_count * 4;
    k_finalize_block<<<(unsigned)(lgrid < maxw ? lgrid : maxw), FIN_LARGE_THREADS, smem, s>>>(io, p);
    k_stats<<<(unsigned)((io.E + 127) / 128), 128, 0, s>>>(io, p);
}

}  // namespace cs
