// Device helpers shared by the reduction kernels (cs_reduce.cu, cs_finalize.cu):
// numpy-order argmax, tangent basis, (u, v, pos) bitonic sorts, the monotone
// chain, the OpenBLAS strided ddot and numpy pairwise summation.
#pragma once
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
__device__ inline ArgMax block_argmax(ArgMax a, ArgMax *sm) {
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
// last key it is a total order, so the bitonic network reproduces it exactly. Per
// key numpy orders NaN after every number and NaNs as equal (npy_sort's
// LT(a, b) = a < b || (b != b && a == a)). NANS = false: keys known to be free of NaN.
template <bool NANS = true>
__device__ __forceinline__ bool key_less(double ua, double va, int pa, double ub, double vb, int pb) {
    if (!NANS) {
        if (ua != ub) return ua < ub;
        if (va != vb) return va < vb;
        return pa < pb;
    }
    if (ua != ub) {
        if (ua < ub) return true;
        if (ub < ua) return false;
        if (isnan(ua) != isnan(ub)) return isnan(ub);  // one NaN: the number first
    }
    if (va != vb) {
        if (va < vb) return true;
        if (vb < va) return false;
        if (isnan(va) != isnan(vb)) return isnan(vb);
    }
    return pa < pb;
}

// All-ascending bitonic sort of m keys with virtual +inf padding (block-cooperative).
__device__ inline void block_sort_uv(double *su, double *sv, int *sp, int m) {
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
__device__ inline int monotone_chain(const double *su, const double *sv, int m, int *h) {
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
__device__ inline double hull_area_of(const double *su, const double *sv, const int *h, int H) {
    double d1 = ddot_x2(H, [&](int k) { return su[h[k]]; }, [&](int k) { return sv[h[(k + 1) % H]]; });
    double d2 = ddot_x2(H, [&](int k) { return sv[h[k]]; }, [&](int k) { return su[h[(k + 1) % H]]; });
    return 0.5 * fabs(d1 - d2);
}

// numpy pairwise summation (umath loops, PW_BLOCKSIZE 128): leaves of <= 128
// elements use eight interleaved accumulators; larger ranges split at
// n/2 rounded down to a multiple of 8 and add left + right.
template <class F>
__device__ __forceinline__ double pairwise_leaf(F a, int off, int n) {
    if (n < 8) {
        double r = 0.0;
        for (int i = 0; i < n; ++i) r += a(off + i);
        return r;
    }
    double r0 = a(off), r1 = a(off + 1), r2 = a(off + 2), r3 = a(off + 3);
    double r4 = a(off + 4), r5 = a(off + 5), r6 = a(off + 6), r7 = a(off + 7);
    int i;
    for (i = 8; i < n - (n % 8); i += 8) {
        r0 += a(off + i); r1 += a(off + i + 1); r2 += a(off + i + 2); r3 += a(off + i + 3);
        r4 += a(off + i + 4); r5 += a(off + i + 5); r6 += a(off + i + 6); r7 += a(off + i + 7);
    }
    double res = ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7));
    for (; i < n; ++i) res += a(off + i);
    return res;
}

// Iterative post-order walk of the split tree (no device recursion: the call
// stack of large patches would overflow the per-thread stack).
template <class F>
__device__ double pairwise(F a, int off, int n) {
    if (n <= 128) return pairwise_leaf(a, off, n);
    int s_off[32], s_n[32];
    unsigned char s_state[32];
    double s_left[32];
    int sp = 0;
    double ret = 0.0;
    s_off[0] = off; s_n[0] = n; s_state[0] = 0; sp = 1;
    while (sp > 0) {
        const int t = sp - 1;
        const int fo = s_off[t], fn = s_n[t];
        if (fn <= 128) { ret = pairwise_leaf(a, fo, fn); --sp; continue; }
        int n2 = fn / 2;
        n2 -= n2 % 8;
        if (s_state[t] == 0) {
            s_state[t] = 1;
            s_off[sp] = fo; s_n[sp] = n2; s_state[sp] = 0; ++sp;
        } else if (s_state[t] == 1) {
            s_left[t] = ret;
            s_state[t] = 2;
            s_off[sp] = fo + n2; s_n[sp] = fn - n2; s_state[sp] = 0; ++sp;
        } else {
            ret = s_left[t] + ret;
            --sp;
        }
    }
    return ret;
}

// ------------------------------------------------------------------ warp-level variants

__device__ __forceinline__ ArgMax warp_argmax(ArgMax a) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        ArgMax b;
        b.v = __shfl_xor_sync(0xffffffffu, a.v, o);
        b.i = __shfl_xor_sync(0xffffffffu, a.i, o);
        b.cnt = __shfl_xor_sync(0xffffffffu, a.cnt, o);
        a = argmax_combine(a, b);
    }
    return a;
}

// All-ascending bitonic sort of m (u, v, pos) keys by one warp (virtual +inf padding).
__device__ inline void warp_sort_uv(double *su, double *sv, int *sp, int m) {
    const int lane = threadIdx.x & 31;
    int P2 = 1;
    while (P2 < m) P2 <<= 1;
    const int half = P2 >> 1;
    for (int k = 2; k <= P2; k <<= 1) {
        const int hk = k >> 1;
        for (int jj = hk; jj >= 1; jj >>= 1) {
            for (int idx = lane; idx < half; idx += 32) {
                int i, j;
                if (jj == hk) {  // first step of a merge: mirrored partner
                    int blk = idx / hk, off = idx % hk;
                    i = blk * k + off;
                    j = blk * k + k - 1 - off;
                } else {
                    int blk = idx / jj, off = idx % jj;
                    i = blk * 2 * jj + off;
                    j = i + jj;
                }
                if (j < m) {
                    double ui = su[i], uj = su[j], vi = sv[i], vj = sv[j];
                    int pi = sp[i], pj = sp[j];
                    if (key_less(uj, vj, pj, ui, vi, pi)) {
                        su[i] = uj; su[j] = ui; sv[i] = vj; sv[j] = vi; sp[i] = pj; sp[j] = pi;
                    }
                }
            }
            __syncwarp();
        }
    }
}

// Ordered compaction by one warp: writes k for every k in [0, m) with pred(k)
// into out[] in ascending order, returns the count.
template <class Pred>
__device__ __forceinline__ int warp_compact(int m, Pred pred, int *out) {
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    int running = 0;
    for (int c0 = 0; c0 < m; c0 += 32) {
        int k = c0 + lane;
        bool f = k < m && pred(k);
        unsigned b = __ballot_sync(0xffffffffu, f);
        if (f) out[running + __popc(b & lt)] = k;
        running += __popc(b);
    }
    __syncwarp();
    return running;
}

}  // namespace cs
