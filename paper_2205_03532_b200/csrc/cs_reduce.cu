// Contact-patch reduction on sm_100a (reduction.py:45-143, Algorithm 1).
//
//   k_reduce   one CTA (RED_T threads) per env.
//     * Assign (reduction.py:78-88): every batch position against every builder,
//       in parallel over the CTA.
//     * FindDeepest / BinReduce / AddPatch (reduction.py:63-73, 91-126): a
//       sequential loop (one step per created patch, ~35 per env), each step
//       spread over the CTA: an order-preserving list of the still unassigned
//       positions (block-scan compaction, ping-pong buffers); one pass over it
//       bins against the seed AND finds the next seed (first argmax of depth
//       among the survivors); the builder decision is a block argmax. The cold
//       eviction path (reduction.py:111-126) runs in warp 0.
//     * Members -> CSR by a stable counting sort (__match_any_sync) in warp 0.
//   Builders (normals, order-encoded max depths) and the batch state live in
//   shared memory; candidates are read through the read-only path.
// Per-patch finalisation lives in cs_finalize.cu.
#include <float.h>
#include <climits>

#include "cs_reduce_util.cuh"

namespace cs {

constexpr int RED_T = 128;

// Shared memory of one env: builders [N][3] f64, max depth [N] u64, counts [N] i32,
// batch depths [SB] f64 (normals are read through L1), batch -> candidate [SB] i32,
// unassigned lists [2][SB] i32, binned list [SB] i32, flags [SB] u8.
__host__ __device__ inline size_t red_smem_bytes(int N, int SB) {
    return (((size_t)N * (3 * 8 + 8 + 4) + 15) & ~(size_t)15) + (size_t)SB * (8 + 16) +
           (((size_t)SB + 15) & ~(size_t)15);
}

__device__ __forceinline__ double cosv(bool v3, const double *a, const double *b) {
    return v3 ? V3(a[0], a[1], a[2], b[0], b[1], b[2]) : G3(a[0], a[1], a[2], b[0], b[1], b[2]);
}

// numpy argmax over q = 0, 1, ...: strictly larger wins, the first NaN wins
__device__ __forceinline__ bool seq_better(double c, double bc) { return c > bc || (c != c && bc == bc); }

// _hull_area (reduction.py:227-236) of the env's candidates labelled L, by one warp
// over global scratch (only used on the eviction path).
__device__ double warp_hull_area_label(const int32_t *lab, int C, int L, const double *pts, const double *normal,
                                       double *su, double *sv, int *sp, int *sh) {
    const int lane = threadIdx.x & 31;
    int m = warp_compact(C, [&](int i) { return lab[i] == L; }, sh);
    if (m < 3) return 0.0;
    double t1[3], t2[3];
    tangent_basis(normal, t1, t2);
    for (int k = lane; k < m; k += 32) {
        const double *p = pts + 3 * (int64_t)sh[k];
        su[k] = V3(p[0], p[1], p[2], t1[0], t1[1], t1[2]);  // (m,3) @ (3,), m >= 2
        sv[k] = V3(p[0], p[1], p[2], t2[0], t2[1], t2[2]);
        sp[k] = k;
    }
    __syncwarp();
    warp_sort_uv(su, sv, sp, m);
    double area = 0.0;
    if (lane == 0) {
        int H = monotone_chain(su, sv, m, sh);
        area = H < 3 ? 0.0 : hull_area_of(su, sv, sh, H);
    }
    area = __shfl_sync(0xffffffffu, area, 0);
    __syncwarp();
    return area;
}

#ifdef RED_PROF
__device__ unsigned long long g_red_prof[8];
#define RED_MARK(i) do { if (threadIdx.x == 0) { const long long t_ = clock64(); atomicAdd(&g_red_prof[i], (unsigned long long)(t_ - t_red)); t_red = t_; } } while (0)
extern "C" int cs_debug_red_prof(unsigned long long *out) { return (int)cudaMemcpyFromSymbol(out, g_red_prof, sizeof(g_red_prof)); }
#else
#define RED_MARK(i) do {} while (0)
#endif

// Builders -> outputs, then the members CSR: a stable counting sort of candidate
// indices by patch label. With room in the (now idle) batch staging `scratch`, the four
// warps take contiguous quarters of the candidates: per-warp label counts give every
// (warp, patch) its base, so each patch's members stay in ascending candidate order;
// else warp 0 alone. Called by all RED_T threads after a barrier.
__device__ void write_patches_csr(const ReduceIO &io, int N, int P, const double *bn, const unsigned long long *bmx,
                                  int *hcnt, int *scratch, size_t scratch_bytes, const int32_t *lab, int C) {
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const unsigned FULL = 0xffffffffu, lt = (1u << lane) - 1u;
    __shared__ int s_ws2[WS_INTS];
    const int64_t e = blockIdx.x;
    const int64_t base = io.cand_base[e];
    for (int q = tid; q < N; q += RED_T) {
        double *o = io.patch_normal + 3 * (e * N + q);
        if (q < P) { o[0] = bn[3 * q]; o[1] = bn[3 * q + 1]; o[2] = bn[3 * q + 2]; }
        else { o[0] = 0.0; o[1] = 0.0; o[2] = 0.0; }
        io.builder_maxd[e * N + q] = q < P ? dec_d(bmx[q]) : 0.0;
        hcnt[q] = 0;
    }
    if (tid == 0) io.n_patch[e] = P;
    __syncthreads();
    int32_t *moff = io.member_offsets + e * (N + 1);
    int32_t *mem = io.members + base;
    const bool par = scratch_bytes >= (size_t)16 * N;
    int *hw = par ? scratch : hcnt;  // [4][N] counts, then bases (par)
    if (par) {
        for (int q = tid; q < 4 * N; q += RED_T) hw[q] = 0;
        __syncthreads();
    }
    const int qlen = par ? (C + 3) / 4 : C;
    const int i0 = par ? min(C, wid * qlen) : 0, i1 = par ? min(C, i0 + qlen) : C;
    if (par) {
        for (int i = i0 + lane; i < i1; i += 32) {
            const int l = lab[i];
            if (l >= 0) atomicAdd(&hw[wid * N + l], 1);
        }
    } else {
        for (int i = tid; i < C; i += RED_T) {
            const int l = lab[i];
            if (l >= 0) atomicAdd(&hcnt[l], 1);
        }
    }
    __syncthreads();
    if (par) {
        int run = 0;
        for (int q0 = 0; q0 < N; q0 += RED_T) {
            const int q = q0 + tid;
            int c[4] = {0, 0, 0, 0};
            if (q < P)
                for (int w = 0; w < 4; ++w) c[w] = hw[w * N + q];
            int tot;
            const int x = run + block_excl_scan(c[0] + c[1] + c[2] + c[3], s_ws2, &tot);
            if (q < N) {
                moff[q] = x;
                int b = x;
                for (int w = 0; w < 4; ++w) { hw[w * N + q] = b; b += c[w]; }
            }
            run += tot;
        }
        if (tid == 0) moff[N] = run;
        __syncthreads();
    } else {
        if (wid != 0) return;
        if (lane == 0) {
            int run = 0;
            for (int q = 0; q < N; ++q) {
                moff[q] = run;
                const int c = q < P ? hcnt[q] : 0;
                hcnt[q] = run;  // running base
                run += c;
            }
            moff[N] = run;
        }
        __syncwarp();
    }
    int *cnt = par ? hw + wid * N : hcnt;  // this warp's running bases
    constexpr int PF = 8;  // labels prefetched per lane: keeps 8 loads in flight per round
    for (int c0 = i0; c0 < i1; c0 += 32 * PF) {
        int lb[PF];
#pragma unroll
        for (int u = 0; u < PF; ++u) {
            const int i = c0 + 32 * u + lane;
            lb[u] = (i < i1) ? lab[i] : -1;
        }
#pragma unroll
        for (int u = 0; u < PF; ++u) {
            const int i = c0 + 32 * u + lane;
            const int l = lb[u];
            const unsigned peers = __match_any_sync(FULL, l);
            const int rank = __popc(peers & lt);
            if (l >= 0) mem[cnt[l] + rank] = i;
            __syncwarp();
            if (l >= 0 && rank == 0) cnt[l] += __popc(peers);
            __syncwarp();
        }
    }
}

__global__ void __launch_bounds__(RED_T) k_reduce(ReduceIO io, ReduceParams p, int SB) {
    // keep at <= 72 registers (7 CTAs per SM: 1036 >= 1024 envs in one wave); 80 registers measured
    // 13% slower, and a (RED_T, 7) bound makes ptxas spill
#ifdef RED_PROF
    long long t_red = clock64();
#endif
    extern __shared__ __align__(16) unsigned char dyn[];
    __shared__ int s_P;
    __shared__ int s_ws[WS_INTS];
    __shared__ ArgMax s_am[32];
    __shared__ double s_dred[32];
    const int N = p.N;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const unsigned FULL = 0xffffffffu, lt = (1u << lane) - 1u;
    double *bn = reinterpret_cast<double *>(dyn);                                  // [N][3]
    unsigned long long *bmx = reinterpret_cast<unsigned long long *>(bn + 3 * N);  // [N]
    int *hcnt = reinterpret_cast<int *>(bmx + N);                                  // [N]
    double *bdep = reinterpret_cast<double *>(dyn + (((size_t)N * 36 + 15) & ~(size_t)15));  // [SB]
    int32_t *sbo = reinterpret_cast<int32_t *>(bdep + SB);                         // [SB]
    int32_t *ul = sbo + SB;                                                        // [SB] unassigned positions
    int32_t *bl = ul + SB;                                                         // [SB] binned positions
    int32_t *ul2 = bl + SB;                                                        // [SB] unassigned (ping-pong)
    uint8_t *st = reinterpret_cast<uint8_t *>(ul2 + SB);                           // [SB]

    const int64_t e = blockIdx.x;
    if (io.red_slow && io.red_slow[e] == 0) return;  // k_reduce_fast finished this env
    const int64_t base = io.cand_base[e];
    const int C = io.n_cand[e];
    const double *nrm = io.normal + 3 * base;
    const double *dep = io.depth + base;
    const double *pts = io.point + 3 * base;
    int32_t *ord = io.order + base;
    int32_t *lab = io.label + base;
    const int64_t hb = 2 * base + e * (4 * (int64_t)N + 4);
    double *su = io.su + base, *sv = io.sv + base;
    int *sp = io.sp + base, *sh = io.sh + hb;

    for (int i = tid; i < C; i += RED_T) lab[i] = -1;
    // order = candidates passing min_depth (reduction.py:50-53), ascending
    const bool has_md = io.env_min_depth ? true : (p.has_min_depth != 0);
    const double md = io.env_min_depth ? io.env_min_depth[e] : p.min_depth;
    // Generated candidates always pass (phi <= cd  =>  depth >= -cd), so check that
    // in parallel first and keep the identity order; compact only when some fail.
    bool any_fail = false;
    if (has_md)
        for (int i = tid; i < C; i += RED_T) any_fail |= !(__ldg(dep + i) >= md);
    const bool identity = !__syncthreads_or(any_fail);
    int n_order = C;
    if (!identity) {
        if (wid == 0) n_order = warp_compact(C, [&](int i) { return !has_md || __ldg(dep + i) >= md; }, ord);
        if (tid == 0) s_P = n_order;
        __syncthreads();
        n_order = s_P;
        __syncthreads();
    }

    int P = 0;  // builders; uniform across the CTA at every barrier
    RED_MARK(0);
    for (int start = 0; start < n_order; start += p.batch_size) {
        const int bsz = min(p.batch_size, n_order - start);
        // stage the batch: candidate index, normal and depth per position (read many times below)
        for (int k = tid; k < bsz; k += RED_T) {
            const int i = identity ? start + k : ord[start + k];
            sbo[k] = i;
            bdep[k] = __ldg(dep + i);
        }
        __syncthreads();
        // _assign_to_existing: normals[batch] @ reps.T, first argmax, >= cone
        {
            const bool v3 = !((bsz >= 2 && P >= 2) || (bsz == 1 && P == 1));
            for (int k = tid; k < bsz; k += RED_T) {
                uint8_t s = 0;
                if (P > 0) {
                    const int i = sbo[k];
                    const double a[3] = {__ldg(nrm + 3 * (int64_t)i), __ldg(nrm + 3 * (int64_t)i + 1),
                                         __ldg(nrm + 3 * (int64_t)i + 2)};
                    int best = 0;
                    double bc = cosv(v3, a, bn);
                    for (int q = 1; q < P; ++q) {
                        const double c = cosv(v3, a, bn + 3 * q);
                        if (seq_better(c, bc)) { bc = c; best = q; }
                    }
                    if (bc >= p.cone) {
                        lab[i] = best;
                        s = 1;
                        const double d = bdep[k];
                        if (!isnan(d)) atomicMax(&bmx[best], enc_d(d));
                    }
                }
                st[k] = s;
            }
        }
        __syncthreads();
        // Seed / BinReduce / AddPatch (reduction.py:63-73, 91-126), one step per created
        // patch, each step spread over the CTA: the unassigned batch positions are kept
        // as an ascending list (ordered block-scan compaction), so "first argmax" is
        // numpy's, and the next seed comes out of the same pass as the bin.
        RED_MARK(1);
        int nu, dp;
        {
            int run = 0;
            ArgMax am = {0.0, -1, 0};
            for (int r0 = 0; r0 < bsz; r0 += 32 * RED_T) {
                const int rn = min(bsz - r0, 32 * RED_T);
                const int c = (rn + RED_T - 1) / RED_T;
                const int k0 = r0 + tid * c, k1 = min(k0 + c, r0 + rn);
                int n = 0;
                for (int k = k0; k < k1; ++k) n += st[k] == 0 ? 1 : 0;
                int tot;
                int pos = run + block_excl_scan(n, s_ws, &tot);
                for (int k = k0; k < k1; ++k)
                    if (st[k] == 0) {
                        am = argmax_combine(am, ArgMax{bdep[k], pos, 1});
                        ul[pos++] = k;
                    }
                run += tot;
            }
            am = block_argmax(am, s_am);
            nu = run;
            dp = am.i;
        }
        int32_t *ua = ul, *ub = ul2;
        while (nu > 0) {
            // FindDeepest: dp indexes ua (ascending positions)
            const int sk = ua[dp];
            const int64_t si = sbo[sk];
            const double sn[3] = {__ldg(nrm + 3 * si), __ldg(nrm + 3 * si + 1), __ldg(nrm + 3 * si + 2)};
            const double sd = bdep[sk];
            // BinReduce (reduction.py:67-69) fused with the next FindDeepest. Each thread
            // owns a contiguous span of the list (at most 32 positions per round of
            // 32 RED_T), flags it in registers, and one block scan orders the writes.
            const bool v3 = nu >= 2;
            int keep = 0, nbin = 0;
            double lmax = -INFINITY;
            ArgMax nx = {0.0, -1, 0};
            for (int r0 = 0; r0 < nu; r0 += 32 * RED_T) {
                const int rn = min(nu - r0, 32 * RED_T);
                const int c = (rn + RED_T - 1) / RED_T;
                const int j0 = r0 + tid * c, j1 = min(j0 + c, r0 + rn);
                unsigned bmask = 0;  // bit i: position j0 + i is binned
                int nk = 0, nb = 0;
                for (int j = j0; j < j1; ++j) {
                    const int k = ua[j];
                    const int64_t i = sbo[k];
                    const double n3[3] = {__ldg(nrm + 3 * i), __ldg(nrm + 3 * i + 1), __ldg(nrm + 3 * i + 2)};
                    const bool binned = cosv(v3, n3, sn) >= p.cone || j == dp;
                    bmask |= (binned ? 1u : 0u) << (j - j0);
                    nb += binned ? 1 : 0;
                    nk += binned ? 0 : 1;
                }
                int tot;
                const int pk = block_excl_scan(nk | (nb << 16), s_ws, &tot);
                int kp = keep + (pk & 0xffff), bp = nbin + (pk >> 16);
                for (int j = j0; j < j1; ++j) {
                    const int k = ua[j];
                    const double d = bdep[k];
                    if ((bmask >> (j - j0)) & 1u) {
                        bl[bp++] = k;
                        st[k] = 2;
                        if (d > lmax) lmax = d;  // patch.max_depth: strict > over members, NaN ignored
                    } else {
                        nx = argmax_combine(nx, ArgMax{d, kp, 1});
                        ub[kp++] = k;
                    }
                }
                keep += tot & 0xffff;
                nbin += tot >> 16;
            }
            nx = block_argmax(nx, s_am);
            double pmax = sd;
            if (isnan(sd)) {
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) lmax = fmax(lmax, __shfl_xor_sync(FULL, lmax, o));
                if (lane == 0) s_dred[wid] = lmax;
                __syncthreads();
                pmax = -INFINITY;
                for (int i = 0; i < RED_T / 32; ++i) pmax = fmax(pmax, s_dred[i]);
                __syncthreads();
            }
            // _add_patch decision (reduction.py:91-110): reps @ patch.normal, first argmax
            ArgMax bq = {0.0, -1, 0};
            if (P > 0) {
                const bool v3b = P >= 2;
                for (int q = tid; q < P; q += RED_T) bq = argmax_combine(bq, ArgMax{cosv(v3b, bn + 3 * q, sn), q, 1});
                bq = block_argmax(bq, s_am);
            }
            const int best = bq.i;
            const double bc = bq.v;
            const bool similar = P > 0 && bc >= p.cone;
            if (similar && (bc >= MERGE_COS || P >= N)) {  // merge: deeper patch's normal, union members
                const int t = best;
                if (tid == 0 && pmax > dec_d(bmx[t])) { bn[3 * t] = sn[0]; bn[3 * t + 1] = sn[1]; bn[3 * t + 2] = sn[2]; }
                __syncthreads();
                for (int x = tid; x < nbin; x += RED_T) {
                    const int k = bl[x], i = sbo[k];
                    lab[i] = t;
                    st[k] = 1;
                    const double d = bdep[k];
                    if (!isnan(d)) atomicMax(&bmx[t], enc_d(d));
                }
            } else if (P < N) {  // append
                if (tid == 0) {
                    bn[3 * P] = sn[0]; bn[3 * P + 1] = sn[1]; bn[3 * P + 2] = sn[2];
                    bmx[P] = enc_d(pmax);
                }
                for (int x = tid; x < nbin; x += RED_T) {
                    const int k = bl[x];
                    lab[sbo[k]] = P;
                    st[k] = 1;
                }
                ++P;
            } else if (wid == 0) {  // evict the lowest-priority patch (reduction.py:111-126): cold, warp 0
                    for (int x = lane; x < nbin; x += 32) lab[sbo[bl[x]]] = -2;
                    __syncwarp();
                    double gm = dec_d(bmx[0]);
                    for (int q = 1; q < P; ++q) { const double v = dec_d(bmx[q]); if (v > gm) gm = v; }
                    int victim = -1, vprot = 0;
                    double vd = 0.0, va = 0.0;
                    for (int q = 0; q < P; ++q) {  // victim = max(score) in slot order
                        const double ar = warp_hull_area_label(lab, C, q, pts, bn + 3 * q, su, sv, sp, sh);
                        const double d = dec_d(bmx[q]);
                        const int prot = d >= gm;
                        bool better;
                        if (victim < 0) better = true;
                        else if ((prot ? 0 : 1) != (vprot ? 0 : 1)) better = (prot ? 0 : 1) > (vprot ? 0 : 1);
                        else if (-d != -vd) better = -d > -vd;
                        else if (-ar != -va) better = -ar > -va;
                        else better = false;
                        if (better) { victim = q; vprot = prot; vd = d; va = ar; }
                    }
                    const double parea = warp_hull_area_label(lab, C, -2, pts, sn, su, sv, sp, sh);
                    const bool replace = (pmax > vd) || (pmax == vd && parea > va);
                    double fn[3];
                    if (replace) {
                        fn[0] = bn[3 * victim]; fn[1] = bn[3 * victim + 1]; fn[2] = bn[3 * victim + 2];
                        __syncwarp();
                        if (lane == 0) {
                            bn[3 * victim] = sn[0]; bn[3 * victim + 1] = sn[1]; bn[3 * victim + 2] = sn[2];
                            bmx[victim] = enc_d(pmax);
                        }
                    } else {
                        fn[0] = sn[0]; fn[1] = sn[1]; fn[2] = sn[2];
                    }
                    __syncwarp();
                    // _fold_members: nearest normal among builders (reps @ folded.normal)
                    const bool v3b = P >= 2;
                    int tgt = -1;
                    double tc = 0.0;
                    for (int q = 0; q < P; ++q) {
                        const double c = (replace && q == victim) ? -INFINITY : cosv(v3b, bn + 3 * q, fn);
                        if (tgt < 0 || amax_better(c, q, tc, tgt)) { tc = c; tgt = q; }
                    }
                    if (replace) {
                        // victim's old members -> tgt (stay when tgt == victim), then new members -> victim
                        for (int i = lane; i < C; i += 32)
                            if (lab[i] == victim) {
                                if (tgt != victim) lab[i] = tgt;
                                const double d = __ldg(dep + i);
                                if (!isnan(d)) atomicMax(&bmx[tgt], enc_d(d));
                            }
                        __syncwarp();
                        for (int i = lane; i < C; i += 32)
                            if (lab[i] == -2) lab[i] = victim;
                    } else {
                        for (int i = lane; i < C; i += 32)
                            if (lab[i] == -2) {
                                lab[i] = tgt;
                                const double d = __ldg(dep + i);
                                if (!isnan(d)) atomicMax(&bmx[tgt], enc_d(d));
                            }
                    }
                    for (int x = lane; x < nbin; x += 32) st[bl[x]] = 1;
            }
            __syncthreads();
            int32_t *tmp = ua; ua = ub; ub = tmp;
            nu = keep;
            dp = nx.i;
        }
        __syncthreads();
        RED_MARK(3);
    }
    RED_MARK(2);
    write_patches_csr(io, N, P, bn, bmx, hcnt, reinterpret_cast<int *>(bdep), (size_t)25 * SB, lab, C);
    RED_MARK(5);
}


// ------------------------------------------------------------------ fast path
//
// k_reduce_fast: the same Algorithm 1 for envs whose candidates all pass min_depth
// and carry no NaN depth or normal (every generated candidate), as long as no patch
// has to be evicted; any other env is flagged (red_slow[e] = 1) and redone from
// scratch by k_reduce. Differences from k_reduce are in the schedule only:
//   * the batch positions stay in place (no ordered compaction of the unassigned
//     list): with no NaN, numpy's first argmax over the unassigned list in position
//     order is the (depth, -position) maximum over the unassigned positions, so
//     each seed comes out of an order-independent block argmax;
//   * the _add_patch decision for a seed is known before its bin is formed (it
//     depends only on the seed normal and the builders): every warp computes it
//     redundantly (no barrier), so bin members get their final label in the binning
//     pass itself, and a bin's max depth is the seed's depth (bin members are
//     unassigned, hence not deeper than the seed);
//   * one step = one pass over the batch + one block argmax: two barriers.
// The assign pass is specialised on its BLAS pattern (G3 / V3) and, without NaN,
// numpy's argmax is a strict > scan.

// Block argmax over (v, i) without NaN: larger v, ties -> lower i; plus the count of
// contributing entries. Each thread brings its local best (i < 0: none). A warp finds
// its max v by shuffles, then the lowest index holding it and the count by one
// reduction each; lane 0 of every warp posts to `part`, and after the barrier every
// thread combines the RED_T / 32 posts the same way.
struct BestD {
    double v;
    int i, cnt;
};

__device__ __forceinline__ BestD warp_best(double v, int i, int cnt) {
    // the max by 32-bit reductions over the order-preserving encoding (hi word, then
    // lo word among the hi-word maxima); v + 0.0 maps -0.0 to +0.0 (numpy: equal)
    const unsigned FULL = 0xffffffffu;
    const unsigned long long enc = i >= 0 ? enc_d(v + 0.0) : 0ull;  // 0: below every encoding
    const unsigned hi = (unsigned)(enc >> 32), lo = (unsigned)enc;
    const unsigned mh = __reduce_max_sync(FULL, hi);
    const unsigned ml = __reduce_max_sync(FULL, hi == mh ? lo : 0u);
    const bool top = i >= 0 && hi == mh && lo == ml;
    const int bi = (int)__reduce_min_sync(FULL, top ? (unsigned)i : 0xffffffffu);
    const int c = __reduce_add_sync(FULL, cnt);
    return BestD{dec_d(((unsigned long long)mh << 32) | ml), bi, c};
}

__device__ __forceinline__ BestD block_best(BestD w, BestD *part) {
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = w;
    __syncthreads();
    BestD r = part[0];
#pragma unroll
    for (int k = 1; k < RED_T / 32; ++k) {
        const BestD b = part[k];
        r.cnt += b.cnt;
        if (b.i >= 0 && (r.i < 0 || b.v > r.v || (b.v == r.v && b.i < r.i))) { r.v = b.v; r.i = b.i; }
    }
    return r;
}

// first argmax over q < P of cos(reps[q], n) (reps @ n: gemv, V3 when P >= 2), per warp
__device__ __forceinline__ BestD warp_best_builder(const double *bn, int P, double n0, double n1, double n2) {
    const int lane = threadIdx.x & 31;
    double bv = -INFINITY;
    int bi = -1;
    for (int q = lane; q < P; q += 32) {  // ascending q per lane: strict > keeps the first
        const double *b = bn + 3 * q;
        const double c = P >= 2 ? V3(b[0], b[1], b[2], n0, n1, n2) : G3(b[0], b[1], b[2], n0, n1, n2);
        if (bi < 0 || c > bv) { bv = c; bi = q; }
    }
    return warp_best(bv, bi, 0);
}

// normals[batch] @ reps.T for U entries at once: first argmax over the builders
// (strict >, no NaN), each builder normal loaded once for the U entries
template <bool GEMM, int U>
__device__ __forceinline__ void assign_best(const double *bn, int P, const double (&a)[U][3], double (&bc)[U],
                                            int (&best)[U]) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
        bc[u] = GEMM ? G3(a[u][0], a[u][1], a[u][2], bn[0], bn[1], bn[2]) : V3(a[u][0], a[u][1], a[u][2], bn[0], bn[1], bn[2]);
        best[u] = 0;
    }
    for (int q = 1; q < P; ++q) {
        const double b0 = bn[3 * q], b1 = bn[3 * q + 1], b2 = bn[3 * q + 2];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const double c = GEMM ? G3(a[u][0], a[u][1], a[u][2], b0, b1, b2) : V3(a[u][0], a[u][1], a[u][2], b0, b1, b2);
            if (c > bc[u]) { bc[u] = c; best[u] = q; }
        }
    }
}

constexpr int AU = 2;  // assign-pass entries per thread per builder sweep

__global__ void __launch_bounds__(RED_T, 7) k_reduce_fast(ReduceIO io, ReduceParams p, int SB) {
    extern __shared__ __align__(16) unsigned char dyn[];
    __shared__ BestD s_part[RED_T / 32];
    const int N = p.N;
    const int tid = threadIdx.x;
    double *bn = reinterpret_cast<double *>(dyn);                                  // [N][3]
    unsigned long long *bmx = reinterpret_cast<unsigned long long *>(bn + 3 * N);  // [N]
    int *hcnt = reinterpret_cast<int *>(bmx + N);                                  // [N]
    double *bdep = reinterpret_cast<double *>(dyn + (((size_t)N * 36 + 15) & ~(size_t)15));  // [SB]
    uint8_t *st = reinterpret_cast<uint8_t *>(bdep + SB);                          // [SB] 1: assigned

    const int64_t e = blockIdx.x;
    const int64_t base = io.cand_base[e];
    const int C = io.n_cand[e];
    const double *nrm = io.normal + 3 * base;
    const double *dep = io.depth + base;
    int32_t *lab = io.label + base;
    const bool has_md = io.env_min_depth ? true : (p.has_min_depth != 0);
    const double md = io.env_min_depth ? io.env_min_depth[e] : p.min_depth;
    int P = 0;  // builders; uniform across the CTA
    for (int start = 0; start < C; start += p.batch_size) {
        const int bsz = min(p.batch_size, C - start);
        // stage depths; eligibility (every candidate passes min_depth, no NaN); the assign
        // pass (_assign_to_existing); the first seed
        const bool gemm = (bsz >= 2 && P >= 2) || (bsz == 1 && P == 1);
        bool bad = false;
        double lv = 0.0;
        int li = -1, lc = 0;
        for (int k0 = 0; k0 < bsz; k0 += AU * RED_T) {
            double a[AU][3], d[AU], bc[AU];
            int best[AU];
#pragma unroll
            for (int u = 0; u < AU; ++u) {
                const int k = k0 + u * RED_T + tid;
                const int64_t i = start + min(k, bsz - 1);
                d[u] = __ldg(dep + i);
                a[u][0] = __ldg(nrm + 3 * i); a[u][1] = __ldg(nrm + 3 * i + 1); a[u][2] = __ldg(nrm + 3 * i + 2);
                bad |= isnan(d[u]) || isnan(a[u][0]) || isnan(a[u][1]) || isnan(a[u][2]) || (has_md && !(d[u] >= md));
            }
            if (P > 0) {
                if (gemm) assign_best<true, AU>(bn, P, a, bc, best);
                else assign_best<false, AU>(bn, P, a, bc, best);
            }
#pragma unroll
            for (int u = 0; u < AU; ++u) {
                const int k = k0 + u * RED_T + tid;
                if (k >= bsz) continue;
                bdep[k] = d[u];
                const bool s = P > 0 && bc[u] >= p.cone;
                st[k] = s ? 1 : 0;
                if (s) {
                    lab[start + k] = best[u];
                    atomicMax(&bmx[best[u]], enc_d(d[u]));
                } else {
                    lab[start + k] = -1;
                    if (li < 0 || d[u] > lv) { lv = d[u]; li = k; }  // ascending k: first max
                    ++lc;
                }
            }
        }
        if (__syncthreads_or(bad)) {  // the general kernel redoes this env
            if (tid == 0) io.red_slow[e] = 1;
            return;
        }
        BestD nx = block_best(warp_best(lv, li, lc), s_part);
        int nu = nx.cnt, sk = nx.i;
        __syncthreads();
        // seed / bin / add-patch steps (reduction.py:63-73, 91-110)
        while (nu > 0) {
            const int64_t si = start + sk;
            const double s0 = __ldg(nrm + 3 * si), s1 = __ldg(nrm + 3 * si + 1), s2 = __ldg(nrm + 3 * si + 2);
            const double sd = bdep[sk];
            int label;
            bool merge = false;
            {
                const BestD bq = P > 0 ? warp_best_builder(bn, P, s0, s1, s2) : BestD{0.0, -1, 0};
                const bool similar = P > 0 && bq.v >= p.cone;
                merge = similar && (bq.v >= MERGE_COS || P >= N);
                if (!merge && P >= N) {  // eviction: the general kernel redoes this env
                    if (tid == 0) io.red_slow[e] = 1;
                    return;
                }
                label = merge ? bq.i : P;
            }
            // BinReduce: cos = normals[unassigned] @ seed_normal (V3: the list holds the seed
            // and, when it has other entries, >= 2 rows), the seed forced in
            lv = 0.0; li = -1; lc = 0;
            for (int k = tid; k < bsz; k += RED_T) {
                if (st[k]) continue;
                const int64_t i = start + k;
                const double c = V3(__ldg(nrm + 3 * i), __ldg(nrm + 3 * i + 1), __ldg(nrm + 3 * i + 2), s0, s1, s2);
                if (c >= p.cone || k == sk) {
                    st[k] = 1;
                    lab[i] = label;
                } else {
                    const double d = bdep[k];
                    if (li < 0 || d > lv) { lv = d; li = k; }
                    ++lc;
                }
            }
            nx = block_best(warp_best(lv, li, lc), s_part);
            if (tid == 0) {
                if (merge) {  // the deeper patch's normal; max depth over the union
                    const unsigned long long ed = enc_d(sd);
                    if (sd > dec_d(bmx[label])) { bn[3 * label] = s0; bn[3 * label + 1] = s1; bn[3 * label + 2] = s2; }
                    if (ed > bmx[label]) bmx[label] = ed;
                } else {
                    bn[3 * label] = s0; bn[3 * label + 1] = s1; bn[3 * label + 2] = s2;
                    bmx[label] = enc_d(sd);
                }
            }
            P += merge ? 0 : 1;
            nu = nx.cnt;
            sk = nx.i;
            __syncthreads();
        }
    }
    if (tid == 0) io.red_slow[e] = 0;
    __syncthreads();
    write_patches_csr(io, N, P, bn, bmx, hcnt, reinterpret_cast<int *>(bdep), (size_t)9 * SB, lab, C);
}

size_t reduce_smem_bytes(int N, int SB) { return red_smem_bytes(N, SB); }

// k_reduce_fast's layout: builders [N] (36 B each), batch depths [SB] f64, flags [SB] u8.
// Less than k_reduce's, so the L1 left beside 7 CTAs per SM holds the batch normals
// the seed steps re-read.
static size_t red_fast_smem_bytes(int N, int SB) { return (((size_t)N * 36 + 15) & ~(size_t)15) + (size_t)SB * 9; }

void launch_reduce(const ReduceIO &io, const ReduceParams &p, int64_t max_batch, cudaStream_t s) {
    if (io.E <= 0) return;
    const int SB = (int)max_batch;
    const size_t smem = reduce_smem_bytes(p.N, SB);
    // per device: the attribute is raised only when the call succeeds (a failed raise
    // leaves the launch to report the error)
    static size_t configured[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    static size_t configured_fast[64] = {};
    size_t &cfg = configured[dev & 63], &cfg_fast = configured_fast[dev & 63];
    if (smem > 48 * 1024 && smem > cfg &&
        cudaFuncSetAttribute(k_reduce, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) == cudaSuccess)
        cfg = smem;
    const size_t fsmem = red_fast_smem_bytes(p.N, SB);
    if (fsmem > 48 * 1024 && fsmem > cfg_fast &&
        cudaFuncSetAttribute(k_reduce_fast, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsmem) == cudaSuccess)
        cfg_fast = fsmem;
    if (io.red_slow) k_reduce_fast<<<(unsigned)io.E, RED_T, fsmem, s>>>(io, p, SB);
    k_reduce<<<(unsigned)io.E, RED_T, smem, s>>>(io, p, SB);
}

}  // namespace cs
