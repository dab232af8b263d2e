// Contact-patch reduction on sm_100a (reduction.py:45-236, Algorithm 1).
//
//   k_reduce    one CTA per env: batched Assign / FindDeepest / BinReduce /
//               AddPatch (append, merge, evict + fold) with the reference's
//               tie-breaks, then a stable counting sort of members by patch (CSR).
//   k_patch_off exclusive scan of patch counts (work list for finalize).
//   k_finalize  one CTA per patch (grid-stride over the work list): kept-contact
//               selection (deepest + monotone-chain hull), aggregates, hull area.
//   k_stats     per env stats (the multi-GPU all-gather payload).
#include <float.h>

#include "cs_reduce.cuh"

namespace cs {

// ------------------------------------------------------------------ helpers

// numpy argmax order: NaN beats everything (first NaN wins), else larger, ties -> lower index.
__device__ __forceinline__ bool amax_better(double v, int i, double bv, int bi) {
    bool vn = isnan(v), bn = isnan(bv);
    if (vn || bn) return vn && (!bn || i < bi);
    if (v != bv) return v > bv;
    return i < bi;
}

struct ArgMax {
    double v;
    int i;
    int cnt;
};

__device__ __forceinline__ ArgMax argmax_combine(ArgMax a, ArgMax b) {
    ArgMax r;
    r.cnt = a.cnt + b.cnt;
    if (b.i < 0) { r.v = a.v; r.i = a.i; return r; }
    if (a.i < 0) { r.v = b.v; r.i = b.i; return r; }
    if (amax_better(b.v, b.i, a.v, a.i)) { r.v = b.v; r.i = b.i; } else { r.v = a.v; r.i = a.i; }
    return r;
}

// Block-wide argmax with counts. smem: 32 ArgMax entries.
__device__ ArgMax block_argmax(ArgMax a, ArgMax *sm) {
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        ArgMax b;
        b.v = __shfl_down_sync(0xffffffffu, a.v, o);
        b.i = __shfl_down_sync(0xffffffffu, a.i, o);
        b.cnt = __shfl_down_sync(0xffffffffu, a.cnt, o);
        a = argmax_combine(a, b);
    }
    if (lane == 0) sm[wid] = a;
    __syncthreads();
    if (wid == 0) {
        ArgMax x = lane < nw ? sm[lane] : ArgMax{0.0, -1, 0};
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            ArgMax b;
            b.v = __shfl_down_sync(0xffffffffu, x.v, o);
            b.i = __shfl_down_sync(0xffffffffu, x.i, o);
            b.cnt = __shfl_down_sync(0xffffffffu, x.cnt, o);
            x = argmax_combine(x, b);
        }
        if (lane == 0) sm[0] = x;
    }
    __syncthreads();
    ArgMax r = sm[0];
    __syncthreads();
    return r;
}

// order-preserving encoding of doubles for integer atomicMax (NaN never stored)
__device__ __forceinline__ unsigned long long enc_d(double d) {
    unsigned long long u = (unsigned long long)__double_as_longlong(d);
    return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double dec_d(unsigned long long u) {
    u = (u & 0x8000000000000000ull) ? (u & 0x7fffffffffffffffull) : ~u;
    return __longlong_as_double((long long)u);
}

// tangent_basis (math3d.py:143-152)
__device__ __forceinline__ void tangent_basis(const double *n, double *t1, double *t2) {
    double a0, a1, a2;
    if (fabs(n[0]) < 0.57735) { a0 = 1.0; a1 = 0.0; a2 = 0.0; } else { a0 = 0.0; a1 = 1.0; a2 = 0.0; }
    double d = G3(a0, a1, a2, n[0], n[1], n[2]);  // np.dot -> ddot(3)
    a0 = a0 - n[0] * d; a1 = a1 - n[1] * d; a2 = a2 - n[2] * d;
    double nn = sqrt(G3(a0, a1, a2, a0, a1, a2));  // np.linalg.norm -> sqrt(ddot)
    t1[0] = a0 / nn; t1[1] = a1 / nn; t1[2] = a2 / nn;
    t2[0] = n[1] * t1[2] - n[2] * t1[1];  // np.cross
    t2[1] = n[2] * t1[0] - n[0] * t1[2];
    t2[2] = n[0] * t1[1] - n[1] * t1[0];
}

// lexsort((v, u)) is a stable sort by (u, v); with the original position as the
// last key it is a total order, so the bitonic network reproduces it exactly.
__device__ __forceinline__ bool key_less(double ua, double va, int pa, double ub, double vb, int pb) {
    if (ua != ub) return ua < ub;
    if (va != vb) return va < vb;
    return pa < pb;
}

// All-ascending bitonic sort of m keys with virtual +inf padding (block-cooperative).
__device__ void block_sort_uv(double *su, double *sv, int *sp, int m) {
    int P2 = 1;
    while (P2 < m) P2 <<= 1;
    int half = P2 >> 1;
    for (int k = 2; k <= P2; k <<= 1) {
        int hk = k >> 1;
        for (int idx = threadIdx.x; idx < half; idx += blockDim.x) {
            int blk = idx / hk, off = idx % hk;
            int i = blk * k + off, j = blk * k + k - 1 - off;
            if (j < m && key_less(su[j], sv[j], sp[j], su[i], sv[i], sp[i])) {
                double tu = su[i]; su[i] = su[j]; su[j] = tu;
                double tv = sv[i]; sv[i] = sv[j]; sv[j] = tv;
                int tp = sp[i]; sp[i] = sp[j]; sp[j] = tp;
            }
        }
        __syncthreads();
        for (int jj = hk >> 1; jj >= 1; jj >>= 1) {
            for (int idx = threadIdx.x; idx < half; idx += blockDim.x) {
                int blk = idx / jj, off = idx % jj;
                int i = blk * 2 * jj + off, j = i + jj;
                if (j < m && key_less(su[j], sv[j], sp[j], su[i], sv[i], sp[i])) {
                    double tu = su[i]; su[i] = su[j]; su[j] = tu;
                    double tv = sv[i]; sv[i] = sv[j]; sv[j] = tv;
                    int tp = sp[i]; sp[i] = sp[j]; sp[j] = tp;
                }
            }
            __syncthreads();
        }
    }
}

__device__ __forceinline__ double cross2(const double *su, const double *sv, int o, int a, int b) {
    return (su[a] - su[o]) * (sv[b] - sv[o]) - (sv[a] - sv[o]) * (su[b] - su[o]);
}

// _monotone_hull (reduction.py:207-224) over sorted keys; single thread.
// Writes hull as sorted-indices into h (capacity m + 2); returns length.
__device__ int monotone_chain(const double *su, const double *sv, int m, int *h) {
    int top = 0;
    for (int s = 0; s < m; ++s) {
        while (top >= 2 && cross2(su, sv, h[top - 2], h[top - 1], s) <= 0.0) --top;
        h[top++] = s;
    }
    int L = top;  // lower = h[0..L); hull keeps h[0..L-1)
    int base = L - 1;
    top = base;
    for (int s = m - 1; s >= 0; --s) {
        while (top - base >= 2 && cross2(su, sv, h[top - 2], h[top - 1], s) <= 0.0) --top;
        h[top++] = s;
    }
    return top - 1;  // (L-1) + (U-1)
}

// OpenBLAS ddot with inc_x = 2 (the strided (H,2) column) and contiguous y.
template <class FX, class FY>
__device__ __forceinline__ double ddot_x2(int n, FX x, FY y) {
    double t1 = 0.0, t2 = 0.0;
    int i = 0, n1 = n & -4;
    while (i < n1) {
        double m3 = y(i + 2) * x(i + 2);
        double m4 = y(i + 3) * x(i + 3);
        t1 = t1 + __fma_rn(y(i), x(i), m3);
        t2 = t2 + __fma_rn(y(i + 1), x(i + 1), m4);
        i += 4;
    }
    while (i < n) { t1 = __fma_rn(y(i), x(i), t1); ++i; }
    return t1 + t2;
}

// _hull_area tail (reduction.py:234-236) given hull (sorted indices) of length H >= 3.
__device__ double hull_area_of(const double *su, const double *sv, const int *h, int H) {
    double d1 = ddot_x2(H, [&](int k) { return su[h[k]]; }, [&](int k) { return sv[h[(k + 1) % H]]; });
    double d2 = ddot_x2(H, [&](int k) { return sv[h[k]]; }, [&](int k) { return su[h[(k + 1) % H]]; });
    return 0.5 * fabs(d1 - d2);
}

// numpy pairwise summation (umath loops), as add.reduce on a contiguous array: 0 + pw.
template <class F>
__device__ double pairwise(F a, int off, int n) {
    if (n < 8) {
        double r = 0.0;
        for (int i = 0; i < n; ++i) r += a(off + i);
        return r;
    } else if (n <= 128) {
        double r[8];
        for (int j = 0; j < 8; ++j) r[j] = a(off + j);
        int i;
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; ++j) r[j] += a(off + i + j);
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; ++i) res += a(off + i);
        return res;
    }
    int n2 = n / 2;
    n2 -= n2 % 8;
    return pairwise(a, off, n2) + pairwise(a, off + n2, n - n2);  // depth <= log2(n / 128)
}

// ------------------------------------------------------------------ k_reduce

// ------------------------------------------------------------------ k_reduce

struct RedShared {
    ArgMax am[32];
    int ws[WS_INTS];
    int P;         // number of builders
    int decision;  // 0 append, 1 merge, 2 evict
    int target;
    double pmax;
    double t1[3], t2[3];
    double area;
    int victim;
    unsigned long long pmax_enc;
};

// Ordered compaction of env candidates with label == L into idx[0..m) (ascending).
__device__ int block_collect_label(const int32_t *lab, int C, int L, int *idx, int *ws) {
    int running = 0;
    for (int c0 = 0; c0 < C; c0 += blockDim.x) {
        int i = c0 + threadIdx.x;
        int f = (i < C && lab[i] == L) ? 1 : 0;
        int tot;
        int pos = running + block_excl_scan(f, ws, &tot);
        if (f) idx[pos] = i;
        running += tot;
    }
    return running;
}

// _hull_area (reduction.py:227-236) of the candidates labelled L; block-cooperative.
// Scratch: su/sv/sp >= C entries, sh >= 2C + 2 entries.
__device__ double block_hull_area_label(const int32_t *lab, int C, int L, const double *pts, const double *normal,
                                        double *su, double *sv, int *sp, int *sh, RedShared &S) {
    int m = block_collect_label(lab, C, L, sh, S.ws);
    if (m < 3) return 0.0;
    if (threadIdx.x == 0) tangent_basis(normal, S.t1, S.t2);
    __syncthreads();
    for (int k = threadIdx.x; k < m; k += blockDim.x) {
        const double *p = pts + 3 * (int64_t)sh[k];
        su[k] = V3(p[0], p[1], p[2], S.t1[0], S.t1[1], S.t1[2]);  // (m,3) @ (3,), m >= 2
        sv[k] = V3(p[0], p[1], p[2], S.t2[0], S.t2[1], S.t2[2]);
        sp[k] = k;
    }
    __syncthreads();
    block_sort_uv(su, sv, sp, m);
    if (threadIdx.x == 0) {
        int H = monotone_chain(su, sv, m, sh);
        S.area = H < 3 ? 0.0 : hull_area_of(su, sv, sh, H);
    }
    __syncthreads();
    double a = S.area;
    __syncthreads();
    return a;
}

__device__ __forceinline__ double cosv(bool v3, const double *a, const double *b) {
    return v3 ? V3(a[0], a[1], a[2], b[0], b[1], b[2]) : G3(a[0], a[1], a[2], b[0], b[1], b[2]);
}

__global__ void __launch_bounds__(REDUCE_BLOCK) k_reduce(ReduceIO io, ReduceParams p, int SB) {
    __shared__ RedShared S;
    extern __shared__ __align__(16) unsigned char dyn[];
    const int N = p.N;
    double *bn = reinterpret_cast<double *>(dyn);                               // [N][3]
    unsigned long long *bmx = reinterpret_cast<unsigned long long *>(bn + 3 * N);  // [N]
    double *cosb = reinterpret_cast<double *>(bmx + N);                         // [N]
    int *hcnt = reinterpret_cast<int *>(cosb + N);                              // [N]
    int *wc = hcnt + N;                                                         // [nwarps][N]
    uint8_t *st = reinterpret_cast<uint8_t *>(wc + (REDUCE_BLOCK / 32) * N);    // [SB]

    const int e = blockIdx.x;
    const int64_t base = io.cand_base[e];
    const int C = io.n_cand[e];
    const double *nrm = io.normal + 3 * base;
    const double *dep = io.depth + base;
    const double *pts = io.point + 3 * base;
    int32_t *ord = io.order + base;
    int32_t *lab = io.label + base;
    const int64_t hb = 2 * base + (int64_t)e * (4 * N + 4);
    double *su = io.su + base, *sv = io.sv + base;
    int *sp = io.sp + base, *sh = io.sh + hb;
    const int tid = threadIdx.x, T = blockDim.x;

    for (int i = tid; i < C; i += T) lab[i] = -1;
    // order = candidates passing min_depth (reduction.py:50-53), ascending
    const bool has_md = io.env_min_depth ? true : (p.has_min_depth != 0);
    const double md = io.env_min_depth ? io.env_min_depth[e] : p.min_depth;
    int n_order = 0;
    for (int c0 = 0; c0 < C; c0 += T) {
        int i = c0 + tid;
        int f = 0;
        if (i < C) f = (!has_md || dep[i] >= md) ? 1 : 0;
        int tot;
        int pos = n_order + block_excl_scan(f, S.ws, &tot);
        if (f) ord[pos] = i;
        n_order += tot;
    }
    if (tid == 0) S.P = 0;
    __syncthreads();

    for (int start = 0; start < n_order; start += p.batch_size) {
        const int bsz = min(p.batch_size, n_order - start);
        const int32_t *bo = ord + start;
        int P = S.P;
        // _assign_to_existing (reduction.py:78-88): normals[batch] @ reps.T
        {
            const bool v3 = !((bsz >= 2 && P >= 2) || (bsz == 1 && P == 1));
            for (int k = tid; k < bsz; k += T) {
                uint8_t s = 0;
                if (P > 0) {
                    int i = bo[k];
                    const double *a = nrm + 3 * (int64_t)i;
                    int best = 0;
                    double bc = cosv(v3, a, bn);
                    for (int q = 1; q < P; ++q) {
                        double c = cosv(v3, a, bn + 3 * q);
                        if (amax_better(c, q, bc, best)) { bc = c; best = q; }
                    }
                    if (bc >= p.cone) {
                        lab[i] = best;
                        s = 1;
                        double d = dep[i];
                        if (!isnan(d)) atomicMax(&bmx[best], enc_d(d));
                    }
                }
                st[k] = s;
            }
        }
        __syncthreads();
        for (;;) {
            // FindDeepest: first argmax of depth over the unassigned (reduction.py:64)
            ArgMax a = {0.0, -1, 0};
            for (int k = tid; k < bsz; k += T)
                if (st[k] == 0) a = argmax_combine(a, ArgMax{dep[bo[k]], k, 1});
            a = block_argmax(a, S.am);
            const int nu = a.cnt;
            if (nu == 0) break;
            const int dp = a.i;
            const int seed = bo[dp];
            const double sn[3] = {nrm[3 * (int64_t)seed], nrm[3 * (int64_t)seed + 1], nrm[3 * (int64_t)seed + 2]};
            const double sd = dep[seed];
            // BinReduce: normals[unassigned] @ seed_normal, seed forced in (reduction.py:67-69)
            const bool v3 = nu >= 2;
            for (int k = tid; k < bsz; k += T) {
                if (st[k] != 0) continue;
                double c = cosv(v3, nrm + 3 * (int64_t)bo[k], sn);
                if (c >= p.cone || k == dp) st[k] = 2;
            }
            if (isnan(sd)) {  // patch.max_depth = max over non-NaN members (absorb uses strict >)
                if (tid == 0) S.pmax_enc = enc_d(-INFINITY);
                __syncthreads();
                for (int k = tid; k < bsz; k += T)
                    if (st[k] == 2 && !isnan(dep[bo[k]])) atomicMax(&S.pmax_enc, enc_d(dep[bo[k]]));
                __syncthreads();
                if (tid == 0) S.pmax = dec_d(S.pmax_enc);
            } else if (tid == 0) {
                S.pmax = sd;
            }
            // _add_patch decision (reduction.py:91-110)
            if (tid < 32) {
                int best = -1;
                double bc = 0.0;
                if (P > 0) {
                    const bool v3b = P >= 2;  // reps @ patch.normal
                    for (int q = tid; q < P; q += 32) {
                        double c = cosv(v3b, bn + 3 * q, sn);
                        cosb[q] = c;
                        if (best < 0 || amax_better(c, q, bc, best)) { bc = c; best = q; }
                    }
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) {
                        double obc = __shfl_down_sync(0xffffffffu, bc, o);
                        int ob = __shfl_down_sync(0xffffffffu, best, o);
                        if (ob >= 0 && (best < 0 || amax_better(obc, ob, bc, best))) { bc = obc; best = ob; }
                    }
                }
                if (tid == 0) {
                    bool similar = P > 0 && bc >= p.cone;
                    if (similar && (bc >= MERGE_COS || P >= N)) { S.decision = 1; S.target = best; }
                    else if (P < N) { S.decision = 0; S.target = P; }
                    else { S.decision = 2; S.target = -1; }
                }
            }
            __syncthreads();
            const int dec = S.decision;
            if (dec == 0) {  // append
                if (tid == 0) {
                    bn[3 * P] = sn[0]; bn[3 * P + 1] = sn[1]; bn[3 * P + 2] = sn[2];
                    bmx[P] = enc_d(S.pmax);
                    S.P = P + 1;
                }
                for (int k = tid; k < bsz; k += T)
                    if (st[k] == 2) { lab[bo[k]] = P; st[k] = 1; }
            } else if (dec == 1) {  // merge: keep the deeper patch's normal, union members
                const int t = S.target;
                if (tid == 0 && S.pmax > dec_d(bmx[t])) { bn[3 * t] = sn[0]; bn[3 * t + 1] = sn[1]; bn[3 * t + 2] = sn[2]; }
                __syncthreads();
                for (int k = tid; k < bsz; k += T)
                    if (st[k] == 2) {
                        int i = bo[k];
                        lab[i] = t;
                        st[k] = 1;
                        if (!isnan(dep[i])) atomicMax(&bmx[t], enc_d(dep[i]));
                    }
            } else {  // evict the lowest-priority patch (reduction.py:111-126)
                for (int k = tid; k < bsz; k += T)
                    if (st[k] == 2) lab[bo[k]] = -2;
                __syncthreads();
                // areas of every builder, then victim = max(score) in slot order
                for (int q = 0; q < P; ++q) {
                    double ar = block_hull_area_label(lab, C, q, pts, bn + 3 * q, su, sv, sp, sh, S);
                    if (tid == 0) cosb[q] = ar;
                    __syncthreads();
                }
                double parea = block_hull_area_label(lab, C, -2, pts, sn, su, sv, sp, sh, S);
                if (tid == 0) {
                    double gm = dec_d(bmx[0]);
                    for (int q = 1; q < P; ++q) { double v = dec_d(bmx[q]); if (v > gm) gm = v; }
                    int victim = -1, vprot = 0;
                    double vd = 0.0, va = 0.0;
                    for (int q = 0; q < P; ++q) {
                        double d = dec_d(bmx[q]), ar = cosb[q];
                        int prot = d >= gm;
                        bool better;
                        if (victim < 0) better = true;
                        else if ((prot ? 0 : 1) != (vprot ? 0 : 1)) better = (prot ? 0 : 1) > (vprot ? 0 : 1);
                        else if (-d != -vd) better = -d > -vd;
                        else if (-ar != -va) better = -ar > -va;
                        else better = false;
                        if (better) { victim = q; vprot = prot; vd = d; va = ar; }
                    }
                    const double pm = S.pmax;
                    bool replace = (pm > vd) || (pm == vd && parea > va);
                    double fn[3];
                    if (replace) {
                        fn[0] = bn[3 * victim]; fn[1] = bn[3 * victim + 1]; fn[2] = bn[3 * victim + 2];
                        bn[3 * victim] = sn[0]; bn[3 * victim + 1] = sn[1]; bn[3 * victim + 2] = sn[2];
                        bmx[victim] = enc_d(pm);
                    } else {
                        fn[0] = sn[0]; fn[1] = sn[1]; fn[2] = sn[2];
                    }
                    // _fold_members: nearest normal among builders (reps @ folded.normal)
                    const bool v3b = P >= 2;
                    int tgt = -1;
                    double tc = 0.0;
                    for (int q = 0; q < P; ++q) {
                        double c = (replace && q == victim) ? -INFINITY : cosv(v3b, bn + 3 * q, fn);
                        if (tgt < 0 || amax_better(c, q, tc, tgt)) { tc = c; tgt = q; }
                    }
                    S.decision = replace ? 3 : 4;
                    S.target = tgt;
                    S.victim = victim;
                }
                __syncthreads();
                const int tgt = S.target;
                const int victim = S.victim;
                if (S.decision == 3) {
                    // victim's old members -> tgt (stay put when tgt == victim), then new members -> victim
                    for (int i = tid; i < C; i += T)
                        if (lab[i] == victim) {
                            if (tgt != victim) lab[i] = tgt;
                            if (!isnan(dep[i])) atomicMax(&bmx[tgt], enc_d(dep[i]));
                        }
                    __syncthreads();
                    for (int i = tid; i < C; i += T)
                        if (lab[i] == -2) lab[i] = victim;
                } else {
                    for (int i = tid; i < C; i += T)
                        if (lab[i] == -2) {
                            lab[i] = tgt;
                            if (!isnan(dep[i])) atomicMax(&bmx[tgt], enc_d(dep[i]));
                        }
                }
                for (int k = tid; k < bsz; k += T)
                    if (st[k] == 2) st[k] = 1;
            }
            __syncthreads();
            P = S.P;
        }
    }
    __syncthreads();
    const int P = S.P;
    // builders -> outputs
    for (int q = tid; q < N; q += T) {
        double *o = io.patch_normal + 3 * ((int64_t)e * N + q);
        if (q < P) { o[0] = bn[3 * q]; o[1] = bn[3 * q + 1]; o[2] = bn[3 * q + 2]; }
        else { o[0] = 0.0; o[1] = 0.0; o[2] = 0.0; }
        io.builder_maxd[(int64_t)e * N + q] = q < P ? dec_d(bmx[q]) : 0.0;
        hcnt[q] = 0;
    }
    for (int w = 0; w < T / 32; ++w)
        for (int q = tid; q < N; q += T) wc[w * N + q] = 0;
    if (tid == 0) io.n_patch[e] = P;
    __syncthreads();
    // CSR: stable counting sort of candidate indices by patch
    for (int i = tid; i < C; i += T) {
        int l = lab[i];
        if (l >= 0) atomicAdd(&hcnt[l], 1);
    }
    __syncthreads();
    int32_t *moff = io.member_offsets + (int64_t)e * (N + 1);
    if (tid == 0) {
        int run = 0;
        for (int q = 0; q < N; ++q) {
            moff[q] = run;
            int c = q < P ? hcnt[q] : 0;
            hcnt[q] = run;  // running base
            run += c;
        }
        moff[N] = run;
    }
    __syncthreads();
    int32_t *mem = io.members + base;
    const int wid = tid >> 5, lane = tid & 31;
    const unsigned lt = (1u << lane) - 1u;
    for (int c0 = 0; c0 < C; c0 += T) {
        int i = c0 + tid;
        int l = (i < C) ? lab[i] : -1;
        unsigned peers = __match_any_sync(0xffffffffu, l);
        int rank = __popc(peers & lt);
        if (l >= 0 && rank == 0) wc[wid * N + l] = __popc(peers);
        __syncthreads();
        if (l >= 0) {
            int pos = hcnt[l] + rank;
            for (int w = 0; w < wid; ++w) pos += wc[w * N + l];
            mem[pos] = i;
        }
        __syncthreads();
        for (int q = tid; q < P; q += T) {
            int s = 0;
            for (int w = 0; w < T / 32; ++w) { s += wc[w * N + q]; wc[w * N + q] = 0; }
            hcnt[q] += s;
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------ finalize

__global__ void k_patch_off(int64_t E, const int32_t *__restrict__ n_patch, int32_t *__restrict__ off) {
    __shared__ int ws[WS_INTS];
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

struct FinShared {
    ArgMax am[32];
    int ws[WS_INTS];
    double t1[3], t2[3];
    int H, nkept;
    double area;
    int chosen[MAX_KEPT];
};

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

struct WeightAt {
    const double *d;
    __device__ double operator()(int k) const { return weight_of(d[k]); }
};

// Member data of one patch, staged in shared memory when it fits.
struct PatchView {
    const double *P, *Nn, *D;  // [m,3], [m,3], [m]
};

__global__ void __launch_bounds__(FINALIZE_BLOCK) k_finalize(ReduceIO io, ReduceParams p) {
    __shared__ FinShared S;
    extern __shared__ __align__(16) unsigned char dyn[];
    const int FSP = FINALIZE_SMEM_POINTS;
    double *cP = reinterpret_cast<double *>(dyn);  // [FSP,3]
    double *cN = cP + 3 * FSP;                     // [FSP,3]
    double *cD = cN + 3 * FSP;                     // [FSP]
    double *c_u = cD + FSP, *c_v = c_u + FSP;      // [FSP]
    int *c_p = reinterpret_cast<int *>(c_v + FSP);  // [FSP]
    int *c_h = c_p + FSP;                           // [2 FSP + 4]
    const int N = p.N, K = p.K;
    const int64_t E = io.E;
    const int total = io.patch_off[E];
    const int tid = threadIdx.x, T = blockDim.x;
    for (int w = blockIdx.x; w < total; w += gridDim.x) {
        int64_t lo = 0, hi = E - 1;  // env of work item w: last e with patch_off[e] <= w
        while (lo < hi) {
            int64_t mid = (lo + hi + 1) >> 1;
            if (io.patch_off[mid] <= w) lo = mid; else hi = mid - 1;
        }
        const int64_t e = lo;
        const int q = w - io.patch_off[e];
        const int64_t base = io.cand_base[e];
        const int32_t *moffp = io.member_offsets + e * (N + 1);
        const int moff = moffp[q];
        const int m = moffp[q + 1] - moff;
        const int32_t *mem = io.members + base + moff;
        const double *gpts = io.point + 3 * base;
        const double *gnrm = io.normal + 3 * base;
        const double *gdep = io.depth + base;
        const int64_t pq = e * N + q;
        const double *rn = io.patch_normal + 3 * pq;
        double *su, *sv;
        int *sp, *sh;
        PatchView V;
        if (m <= FSP) {
            for (int k = tid; k < m; k += T) {
                int i = mem[k];
                cD[k] = gdep[i];
                for (int c = 0; c < 3; ++c) { cP[3 * k + c] = gpts[3 * (int64_t)i + c]; cN[3 * k + c] = gnrm[3 * (int64_t)i + c]; }
            }
            V.P = cP; V.Nn = cN; V.D = cD;
            su = c_u; sv = c_v; sp = c_p; sh = c_h;
        } else {  // large patch: member rows gathered into global scratch
            double *gP = io.gP + 3 * (base + moff), *gN = io.gN + 3 * (base + moff), *gD = io.gD + base + moff;
            for (int k = tid; k < m; k += T) {
                int i = mem[k];
                gD[k] = gdep[i];
                for (int c = 0; c < 3; ++c) { gP[3 * k + c] = gpts[3 * (int64_t)i + c]; gN[3 * k + c] = gnrm[3 * (int64_t)i + c]; }
            }
            V.P = gP; V.Nn = gN; V.D = gD;
            su = io.su + base + moff; sv = io.sv + base + moff; sp = io.sp + base + moff;
            sh = io.sh + 2 * base + e * (4 * N + 4) + 2 * moff + 4 * q;
        }
        __syncthreads();
        // deepest = first argmax over members (reduction.py:182)
        ArgMax a = {0.0, -1, 0};
        for (int k = tid; k < m; k += T) a = argmax_combine(a, ArgMax{V.D[k], k, 1});
        a = block_argmax(a, S.am);
        const int deepest = a.i;
        if (tid == 0) tangent_basis(rn, S.t1, S.t2);
        // base: touching members (depth >= 0) if >= 3 else all (reduction.py:183-184)
        int nt = 0;
        for (int c0 = 0; c0 < m; c0 += T) {
            int k = c0 + tid;
            int f = (k < m && V.D[k] >= 0.0) ? 1 : 0;
            int tot;
            int pos = nt + block_excl_scan(f, S.ws, &tot);
            if (f) sp[pos] = k;
            nt += tot;
        }
        const bool all_base = nt < 3 || nt == m;
        const int nb = nt < 3 ? m : nt;
        const bool need_sel = m > K;
        // hull over the selection base; payload = member position (monotone in base order)
        bool have_hull = false;
        if (need_sel || (m >= 3 && all_base)) {
            for (int j = tid; j < nb; j += T) {
                int k = (nt < 3) ? j : sp[j];
                const double *pp = V.P + 3 * k;
                su[j] = V3(pp[0], pp[1], pp[2], S.t1[0], S.t1[1], S.t1[2]);  // _project_2d, n >= 2
                sv[j] = V3(pp[0], pp[1], pp[2], S.t2[0], S.t2[1], S.t2[2]);
                sp[j] = k;
            }
            __syncthreads();
            block_sort_uv(su, sv, sp, nb);
            if (tid == 0) S.H = monotone_chain(su, sv, nb, sh);
            __syncthreads();
            have_hull = true;
        }
        if (tid == 0) {
            // area over all members (reduction.py:167): reuse the hull when base == members
            if (m < 3) S.area = 0.0;
            else if (have_hull && all_base) S.area = S.H < 3 ? 0.0 : hull_area_of(su, sv, sh, S.H);
            // kept selection (reduction.py:172-199)
            int nc = 0;
            if (!need_sel) {
                for (int k = 0; k < m; ++k) S.chosen[nc++] = k;
            } else {
                S.chosen[nc++] = deepest;
                const int H = S.H;
                int nh = 0;
                for (int h = 0; h < H; ++h) nh += (sp[sh[h]] != deepest);
                if (nh <= K - 1) {
                    for (int h = 0; h < H; ++h) {
                        int k = sp[sh[h]];
                        if (k != deepest) S.chosen[nc++] = k;
                    }
                    while (nc < K) {  // fill by np.argsort(-depths, kind="stable")
                        int bk = -1;
                        double bd = 0.0;
                        for (int k = 0; k < m; ++k) {
                            bool in = false;
                            for (int j = 0; j < nc; ++j) in |= (S.chosen[j] == k);
                            if (in) continue;
                            double d = V.D[k];
                            if (bk < 0 || depth_before(d, k, bd, bk)) { bk = k; bd = d; }
                        }
                        if (bk < 0) break;
                        S.chosen[nc++] = bk;
                    }
                } else {  // picks = linspace(0, len(hull), K-1, endpoint=False).astype(int)
                    double step = (double)nh / (double)(K - 1);
                    int j = 0, cnt = -1;
                    int pk = (int)((double)j * step + 0.0);
                    for (int h = 0; h < H && j < K - 1; ++h) {
                        int k = sp[sh[h]];
                        if (k == deepest) continue;
                        ++cnt;
                        while (j < K - 1 && cnt == pk) {
                            S.chosen[nc++] = k;
                            ++j;
                            pk = (int)((double)j * step + 0.0);
                        }
                    }
                }
            }
            S.nkept = nc < K ? nc : K;
        }
        __syncthreads();
        if (m >= 3 && !(have_hull && all_base)) {  // area hull over all members
            for (int j = tid; j < m; j += T) {
                const double *pp = V.P + 3 * j;
                su[j] = V3(pp[0], pp[1], pp[2], S.t1[0], S.t1[1], S.t1[2]);
                sv[j] = V3(pp[0], pp[1], pp[2], S.t2[0], S.t2[1], S.t2[2]);
                sp[j] = j;
            }
            __syncthreads();
            block_sort_uv(su, sv, sp, m);
            if (tid == 0) {
                int H = monotone_chain(su, sv, m, sh);
                S.area = H < 3 ? 0.0 : hull_area_of(su, sv, sh, H);
            }
        }
        // aggregates (reduction.py:153-168): sequential axis-0 sums, one lane per component
        const int wid = tid >> 5, lane = tid & 31;
        if (wid == 0 && lane < 9) {
            const int kind = lane / 3, c = lane % 3;
            double s = 0.0;
            for (int k = 0; k < m; ++k) {
                const double *pp = V.P + 3 * k, *nn = V.Nn + 3 * k;
                double wk = weight_of(V.D[k]), x;
                if (kind == 0) x = pp[c] * wk;
                else if (kind == 1) x = nn[c] * wk;
                else {
                    int c1 = (c + 1) % 3, c2 = (c + 2) % 3;  // np.cross component c
                    x = (pp[c1] * nn[c2] - pp[c2] * nn[c1]) * wk;
                }
                s = (k == 0) ? x : s + x;
            }
            double *o = (kind == 0 ? io.wp_sum : kind == 1 ? io.wn_sum : io.wt_sum) + 3 * pq;
            o[c] = s;
        } else if (wid == 1 && lane == 0) {
            io.w_sum[pq] = 0.0 + pairwise(WeightAt{V.D}, 0, m);
        } else if (wid == 1 && lane == 1) {
            double mx = V.D[0];
            for (int k = 1; k < m; ++k) {
                double d = V.D[k];
                if (isnan(d) || isnan(mx)) mx = NAN;
                else if (d > mx) mx = d;
            }
            io.max_depth[pq] = mx;
        }
        __syncthreads();
        const int nk = S.nkept;
        if (tid == 0) { io.patch_nkept[pq] = nk; io.area[pq] = S.area; }
        for (int j = tid; j < K; j += T) {
            const int64_t o = pq * K + j;
            if (j < nk) {
                int k = S.chosen[j];
                int i = mem[k];
                io.kept_cand[o] = i;
                io.kept_face[o] = io.face ? io.face[base + i] : -1;
                io.kept_depth[o] = V.D[k];
                for (int c = 0; c < 3; ++c) {
                    io.kept_point[3 * o + c] = V.P[3 * k + c];
                    io.kept_normal[3 * o + c] = V.Nn[3 * k + c];
                }
            } else {
                io.kept_cand[o] = -1;
                io.kept_face[o] = -1;
                io.kept_depth[o] = 0.0;
                for (int c = 0; c < 3; ++c) { io.kept_point[3 * o + c] = 0.0; io.kept_normal[3 * o + c] = 0.0; }
            }
        }
        __syncthreads();
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

// ------------------------------------------------------------------ launchers

size_t reduce_smem_bytes(int N, int SB) {
    return (size_t)N * (3 * 8 + 8 + 8 + 4) + (size_t)(REDUCE_BLOCK / 32) * N * 4 + (size_t)SB + 16;
}

size_t finalize_smem_bytes() { return (size_t)FINALIZE_SMEM_POINTS * (7 * 8 + 2 * 8 + 4 + 8) + 16; }

void launch_reduce(const ReduceIO &io, const ReduceParams &p, int64_t max_batch, cudaStream_t s) {
    if (io.E <= 0) return;
    int SB = (int)max_batch;
    size_t smem = reduce_smem_bytes(p.N, SB);
    static size_t configured = 0;
    if (smem > 48 * 1024 && smem > configured) {
        cudaFuncSetAttribute(k_reduce, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        configured = smem;
    }
    k_reduce<<<(unsigned)io.E, REDUCE_BLOCK, smem, s>>>(io, p, SB);
}

void launch_finalize(const ReduceIO &io, const ReduceParams &p, int sm_count, cudaStream_t s) {
    if (io.E <= 0) return;
    k_patch_off<<<1, 1024, 0, s>>>(io.E, io.n_patch, io.patch_off);
    int64_t maxw = io.E * (int64_t)p.N;
    int64_t grid = (int64_t)sm_count * 8;
    if (grid > maxw) grid = maxw;
    k_finalize<<<(unsigned)grid, FINALIZE_BLOCK, finalize_smem_bytes(), s>>>(io, p);
    k_stats<<<(unsigned)((io.E + 127) / 128), 128, 0, s>>>(io, p);
}

}  // namespace cs
