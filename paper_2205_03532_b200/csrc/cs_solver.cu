// Contact solver kernels (cs_solver.cuh). Compiled with -fmad=false like the rest
// of the library: numba's sweep kernel has no FMA contraction, and the numpy
// products of ContactConstraints.build are OpenBLAS kernels whose rounding is
// written out with explicit fma (measured against the reference in this
// container; oracle/cs_oracle_solver.c carries the same formulas and is pinned to
// the reference's outputs).
//
// The sweep is sequential within a system (every row reads the velocities the
// previous row wrote), so a system is one thread: its body velocities and
// impulses live in registers (two-body systems) or the thread's column of shared
// memory, its mobility matrices in shared memory, and the next row's constraint
// data and accumulators are loaded while the current row is solved, which takes
// the L2 latency off the dependency chain. Systems are independent and run side
// by side.
#include <cuda_pipeline.h>

#include "cs_solver.cuh"

namespace cs {

namespace {

// math3d.py:143-152
__device__ __forceinline__ void tangent_basis(const double n[3], double t1[3], double t2[3]) {
    double a[3];
    if (fabs(n[0]) < 0.57735) { a[0] = 1.0; a[1] = 0.0; a[2] = 0.0; }
    else { a[0] = 0.0; a[1] = 1.0; a[2] = 0.0; }
    const double d = G3(a[0], a[1], a[2], n[0], n[1], n[2]);
    for (int k = 0; k < 3; ++k) a[k] = a[k] - n[k] * d;
    const double nn = sqrt(G3(a[0], a[1], a[2], a[0], a[1], a[2]));
    for (int k = 0; k < 3; ++k) t1[k] = a[k] / nn;
    t2[0] = n[1] * t1[2] - n[2] * t1[1];
    t2[1] = n[2] * t1[0] - n[0] * t1[2];
    t2[2] = n[0] * t1[1] - n[1] * t1[0];
}

// g @ W @ g for g = [d, r x d] (solver.py:128-131). g @ W is numpy -> cblas_dgemv ->
// OpenBLAS dgemv_n on the transposed view: its 4-row vector block pairs products
// (1, 0) and (5, 4) and fuses the rest; the two leftover rows are an fma chain.
// The final (6,) @ (6,) is ddot: an fma chain from the first product.
__device__ double quad_form(const double d[3], const double r[3], const double *__restrict__ W) {
    double g[6];
    g[0] = d[0]; g[1] = d[1]; g[2] = d[2];
    g[3] = r[1] * d[2] - r[2] * d[1];
    g[4] = r[2] * d[0] - r[0] * d[2];
    g[5] = r[0] * d[1] - r[1] * d[0];
    double v[6];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        double t = __fma_rn(g[0], __ldg(W + j), __dmul_rn(g[1], __ldg(W + 6 + j)));
        t = __fma_rn(g[2], __ldg(W + 12 + j), t);
        t = __fma_rn(g[3], __ldg(W + 18 + j), t);
        const double u = __fma_rn(g[4], __ldg(W + 24 + j), __dmul_rn(g[5], __ldg(W + 30 + j)));
        v[j] = t + u;
    }
#pragma unroll
    for (int j = 4; j < 6; ++j) {
        double t = __dmul_rn(g[0], __ldg(W + j));
#pragma unroll
        for (int i = 1; i < 6; ++i) t = __fma_rn(g[i], __ldg(W + 6 * i + j), t);
        v[j] = t;
    }
    double q = __dmul_rn(v[0], g[0]);
#pragma unroll
    for (int i = 1; i < 6; ++i) q = __fma_rn(v[i], g[i], q);
    return q;
}

// ContactConstraints.build for one row c of system s
__device__ __forceinline__ void build_row(int64_t s, int nb, const SysRows &rows, const BuildIO &io, int64_t c) {
    const int64_t b0 = s * nb;
    const int64_t ia = b0 + io.body_a[c], ib = b0 + io.body_b[c];
    double p[3], n[3], a[3], b[3], t1[3], t2[3];
    for (int k = 0; k < 3; ++k) {
        p[k] = io.point[rows.vec(c, k)];
        n[k] = io.normal[rows.vec(c, k)];
        a[k] = p[k] - io.ref[3 * ia + k];
        b[k] = p[k] - io.ref[3 * ib + k];
    }
    tangent_basis(n, t1, t2);
    for (int k = 0; k < 3; ++k) {
        io.ra[rows.vec(c, k)] = a[k]; io.rb[rows.vec(c, k)] = b[k];
        io.tan1[rows.vec(c, k)] = t1[k]; io.tan2[rows.vec(c, k)] = t2[k];
    }
    const double *Wa = io.w_mat + 36 * ia, *Wb = io.w_mat + 36 * ib;
    const double kq0 = quad_form(n, a, Wa) + quad_form(n, b, Wb);
    const double kq1 = quad_form(t1, a, Wa) + quad_form(t1, b, Wb);
    const double kq2 = quad_form(t2, a, Wa) + quad_form(t2, b, Wb);
    io.kn[c] = kq0 > 1e-12 ? 1.0 / kq0 : 0.0;
    io.kt1[c] = kq1 > 1e-12 ? 1.0 / kq1 : 0.0;
    io.kt2[c] = kq2 > 1e-12 ? 1.0 / kq2 : 0.0;
    const double dep = io.depth[c], sl = io.slop[c];
    double bt = 0.0;
    if (dep > sl) bt = io.bias_factor * (dep - sl) / io.h;
    else if (dep < 0.0) bt = dep / io.h;
    io.bias_target[c] = bt;
    // _normal_velocity (solver.py:166-171): v + w x r (numpy cross), then ddot
    const double *vb = io.vel + 6 * ib, *va = io.vel + 6 * ia;
    const double ub0 = vb[0] + (vb[4] * b[2] - vb[5] * b[1]);
    const double ub1 = vb[1] + (vb[5] * b[0] - vb[3] * b[2]);
    const double ub2 = vb[2] + (vb[3] * b[1] - vb[4] * b[0]);
    const double ua0 = va[0] + (va[4] * a[2] - va[5] * a[1]);
    const double ua1 = va[1] + (va[5] * a[0] - va[3] * a[2]);
    const double ua2 = va[2] + (va[3] * a[1] - va[4] * a[0]);
    const double vn0 = G3(ub0 - ua0, ub1 - ua1, ub2 - ua2, n[0], n[1], n[2]);
    const double neg = -vn0;
    const double v_impact = (0.0 > neg) ? 0.0 : neg;  // Python max(-vn0, 0.0)
    const double e = v_impact > 0.5 ? io.restitution[c] : 0.0;  // RESTITUTION_THRESHOLD (solver.py:21)
    io.restitution_target[c] = e * v_impact;
}

// Rows are independent. CSR layout: a warp per system, lanes over its rows;
// interleaved layout: a thread per row slot (a warp covers one row of 32 systems).
__global__ void k_constraints_build(int64_t S, int nb, SysRows rows, BuildIO io) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (rows.off) {
        const int64_t s = t >> 5;
        if (s >= S) return;
        const int64_t n = rows.n(s);
        for (int64_t j = t & 31; j < n; j += 32) build_row(s, nb, rows, io, rows.row(s, j));
    } else {
        const int64_t blk = (t >> 5) / rows.stride, j = (t >> 5) % rows.stride, s = blk * 32 + (t & 31);
        if (s >= S || j >= rows.n(s)) return;
        build_row(s, nb, rows, io, t);
    }
}

#ifndef SW_T_DEF
#define SW_T_DEF 1
#endif
// Systems per sweep block, one thread each. The sweep is issue-bound per warp, so
// a few systems per warp spread the systems over more warps and schedulers.
constexpr int SW_T = SW_T_DEF;

// Body state of one system. Two-body systems (every collide plan: SDF body, mesh
// body) keep velocities and impulses in registers; other sizes use the thread's
// column of shared memory. W (36 per body) is always the thread's shared column:
// one system per lane makes global loads of W 32-way uncoalesced.
struct RegState2 {
    double v0[6], v1[6], i0[6], i1[6];
    const double *W;  // shared, element j of the system at W[j * SW_T]
    bool z0, z1;      // body frozen (see frozen_body)
    __device__ __forceinline__ double v(int body, int k) const { return body ? v1[k] : v0[k]; }
    __device__ __forceinline__ bool frozen(int body) const { return body ? z1 : z0; }
    __device__ __forceinline__ void add_v(int body, const double t[6]) {
        if (body) {
#pragma unroll
            for (int k = 0; k < 6; ++k) v1[k] += t[k];
        } else {
#pragma unroll
            for (int k = 0; k < 6; ++k) v0[k] += t[k];
        }
    }
    __device__ __forceinline__ void add_i(int body, const double g[6]) {
        if (body) {
#pragma unroll
            for (int k = 0; k < 6; ++k) i1[k] += g[k];
        } else {
#pragma unroll
            for (int k = 0; k < 6; ++k) i0[k] += g[k];
        }
    }
};

// Up to four bodies in registers (multi-pair scenes): body indices are per row, so
// every access selects among the NB register sets with compile-time indices.
template <int NB>
struct RegStateN {
    double v_[NB][6], i_[NB][6];
    const double *W;
    bool z_[NB];
    __device__ __forceinline__ double v(int body, int k) const {
        double r = v_[0][k];
#pragma unroll
        for (int b = 1; b < NB; ++b) r = body == b ? v_[b][k] : r;
        return r;
    }
    __device__ __forceinline__ bool frozen(int body) const {
        bool r = z_[0];
#pragma unroll
        for (int b = 1; b < NB; ++b) r = body == b ? z_[b] : r;
        return r;
    }
    __device__ __forceinline__ void add_v(int body, const double t[6]) {
#pragma unroll
        for (int b = 0; b < NB; ++b)
            if (body == b) {
#pragma unroll
                for (int k = 0; k < 6; ++k) v_[b][k] += t[k];
            }
    }
    __device__ __forceinline__ void add_i(int body, const double g[6]) {
#pragma unroll
        for (int b = 0; b < NB; ++b)
            if (body == b) {
#pragma unroll
                for (int k = 0; k < 6; ++k) i_[b][k] += g[k];
            }
    }
};

struct SmemState {
    double *V, *I;  // shared, element j at [j * SW_T]
    const double *W;
    __device__ __forceinline__ double v(int body, int k) const { return V[(6 * body + k) * SW_T]; }
    __device__ __forceinline__ bool frozen(int) const { return false; }
    __device__ __forceinline__ void add_v(int body, const double t[6]) {
#pragma unroll
        for (int k = 0; k < 6; ++k) V[(6 * body + k) * SW_T] += t[k];
    }
    __device__ __forceinline__ void add_i(int body, const double g[6]) {
#pragma unroll
        for (int k = 0; k < 6; ++k) I[(6 * body + k) * SW_T] += g[k];
    }
};

// A body whose 36 mobility entries are all zero (static bodies, chain-driven
// bodies: solver.py:60-62) and whose velocity is finite without -0.0 components:
// every impulse adds w * g == +-0 per term to it, and v + (+-0) == v, so its
// velocity never changes and the 36 products can be skipped while its impulses
// are finite (checked per call). Exact: skipped updates are identities.
__device__ __forceinline__ bool frozen_body(const double *W, const double *v) {
    bool z = true;
    for (int j = 0; j < 36; ++j) z &= W[j * SW_T] == 0.0;
    for (int k = 0; k < 6; ++k) z &= isfinite(v[k]) && !(v[k] == 0.0 && signbit(v[k]));
    return z;
}

// _kernels.py:16-37
template <class St>
__device__ __forceinline__ void apply_impulse(St &st, int body, double jx, double jy, double jz, double rx, double ry,
                                              double rz, double sign) {
    double g[6];
    g[0] = jx * sign; g[1] = jy * sign; g[2] = jz * sign;
    g[3] = (ry * jz - rz * jy) * sign;
    g[4] = (rz * jx - rx * jz) * sign;
    g[5] = (rx * jy - ry * jx) * sign;
    if (!st.frozen(body) || !isfinite(((g[0] + g[1]) + (g[2] + g[3])) + (g[4] + g[5]))) {
        const double *w = st.W + 36 * body * SW_T;
        double t[6];
#pragma unroll
        for (int k = 0; k < 6; ++k)
            t[k] = w[(6 * k) * SW_T] * g[0] + w[(6 * k + 1) * SW_T] * g[1] + w[(6 * k + 2) * SW_T] * g[2] +
                   w[(6 * k + 3) * SW_T] * g[3] + w[(6 * k + 4) * SW_T] * g[4] + w[(6 * k + 5) * SW_T] * g[5];
        st.add_v(body, t);
    }
    st.add_i(body, g);
}

// _kernels.py:40-49
template <class St>
__device__ __forceinline__ double rel_vel(const St &st, int ia, int ib, const double a[3], const double b[3],
                                          double dx, double dy, double dz) {
    const double ubx = st.v(ib, 0) + st.v(ib, 4) * b[2] - st.v(ib, 5) * b[1];
    const double uby = st.v(ib, 1) + st.v(ib, 5) * b[0] - st.v(ib, 3) * b[2];
    const double ubz = st.v(ib, 2) + st.v(ib, 3) * b[1] - st.v(ib, 4) * b[0];
    const double uax = st.v(ia, 0) + st.v(ia, 4) * a[2] - st.v(ia, 5) * a[1];
    const double uay = st.v(ia, 1) + st.v(ia, 5) * a[0] - st.v(ia, 3) * a[2];
    const double uaz = st.v(ia, 2) + st.v(ia, 3) * a[1] - st.v(ia, 4) * a[0];
    return (ubx - uax) * dx + (uby - uay) * dy + (ubz - uaz) * dz;
}

// Row staging. Each system thread streams its rows through a ring of RING slots
// in shared memory with per-thread asynchronous copies (cp.async), RING - 1 rows
// ahead of the row being solved, so no load latency sits on the sweep's chain
// and no registers hold rows in flight. The accumulators (lam_n of the phase,
// lam_t1, lam_t2) of systems up to LAM_CAP rows live in shared memory for the
// whole call.
constexpr int RING = 8;
constexpr int ROW_F = 22;  // a[3] b[3] n[3] t1[3] t2[3] kn kt1 kt2 target mu body_a body_b
constexpr int LAM_CAP = 1024;

__host__ __device__ inline size_t sweep_smem_doubles(int nb, bool two) {
    if (nb > SOLVER_SMEM_BODIES) return (size_t)RING * ROW_F + 3 * (size_t)LAM_CAP;  // MODE 1: state in global
    return (size_t)36 * nb + (two ? 0 : (size_t)12 * nb) + (size_t)RING * ROW_F + 3 * (size_t)LAM_CAP;
}

template <bool FIX>
__device__ __forceinline__ void stage_row(double *slot, const SweepIO &io, const SweepPhase &ph, const SysRows &rows,
                                          int64_t c) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const int64_t v = rows.vec(c, k);
        __pipeline_memcpy_async(slot + (0 + k) * SW_T, io.ra + v, 8);
        __pipeline_memcpy_async(slot + (3 + k) * SW_T, io.rb + v, 8);
        __pipeline_memcpy_async(slot + (6 + k) * SW_T, io.nrm + v, 8);
        __pipeline_memcpy_async(slot + (9 + k) * SW_T, io.tan1 + v, 8);
        __pipeline_memcpy_async(slot + (12 + k) * SW_T, io.tan2 + v, 8);
    }
    __pipeline_memcpy_async(slot + 15 * SW_T, io.kn + c, 8);
    __pipeline_memcpy_async(slot + 16 * SW_T, io.kt1 + c, 8);
    __pipeline_memcpy_async(slot + 17 * SW_T, io.kt2 + c, 8);
    __pipeline_memcpy_async(slot + 18 * SW_T, ph.target + c, 8);
    __pipeline_memcpy_async(slot + 19 * SW_T, io.mu + c, 8);
    if (!FIX) {
        __pipeline_memcpy_async(slot + 20 * SW_T, io.body_a + c, 8);
        __pipeline_memcpy_async(slot + 21 * SW_T, io.body_b + c, 8);
    }
}

// One row of the sweep (_kernels.py:71-115) on the system state st; the row's
// accumulators are read and written through pln / plt1 / plt2.
template <class St>
__device__ __forceinline__ void solve_row(St &st, int ia, int ib, const double a[3], const double b[3],
                                          const double n[3], const double t1[3], const double t2[3], double kn,
                                          double kt1, double kt2, double tg, double mu, double *pln, double *plt1,
                                          double *plt2, int with_friction) {
    double ln = *pln;
    if (kn > 0.0) {
        const double vn = rel_vel(st, ia, ib, a, b, n[0], n[1], n[2]);
        double dl = kn * (tg - vn);
        double new_l = ln + dl;
        if (new_l < 0.0) new_l = 0.0;
        dl = new_l - ln;
        ln = new_l;
        *pln = new_l;
        if (dl != 0.0) {
            const double jx = dl * n[0], jy = dl * n[1], jz = dl * n[2];
            apply_impulse(st, ib, jx, jy, jz, b[0], b[1], b[2], 1.0);
            apply_impulse(st, ia, jx, jy, jz, a[0], a[1], a[2], -1.0);
        }
    }
    if (with_friction && mu > 0.0 && ln > 0.0) {
        const double lt1 = *plt1, lt2 = *plt2;
        double d1 = 0.0, d2 = 0.0;
        if (kt1 > 0.0) d1 = -kt1 * rel_vel(st, ia, ib, a, b, t1[0], t1[1], t1[2]);
        if (kt2 > 0.0) d2 = -kt2 * rel_vel(st, ia, ib, a, b, t2[0], t2[1], t2[2]);
        double new1 = lt1 + d1, new2 = lt2 + d2;
        const double limit = mu * ln;
        const double mag = sqrt(new1 * new1 + new2 * new2);
        if (mag > limit) {
            const double scale = limit / mag;
            new1 *= scale;
            new2 *= scale;
        }
        d1 = new1 - lt1;
        d2 = new2 - lt2;
        *plt1 = new1;
        *plt2 = new2;
        if (d1 != 0.0 || d2 != 0.0) {
            const double jx = d1 * t1[0] + d2 * t2[0];
            const double jy = d1 * t1[1] + d2 * t2[1];
            const double jz = d1 * t1[2] + d2 * t2[2];
            apply_impulse(st, ib, jx, jy, jz, b[0], b[1], b[2], 1.0);
            apply_impulse(st, ia, jx, jy, jz, a[0], a[1], a[2], -1.0);
        }
    }
}

// The phases of one system, its rows in sweep order. FIX: every row has
// body_a = 0, body_b = 1 (plan rows, scene.py:228-243), so body indices are
// compile-time constants.
template <bool FIX, class St>
__device__ __forceinline__ void sweep_system(St &st, const SweepIO &io, const SweepPhase *phs, int n_phases,
                                             const SysRows &rows, int64_t s, double *ring, double *lam) {
    const int m = (int)rows.n(s);
    if (m <= 0) return;
    const int64_t base = rows.row(s, 0), step = rows.off ? 1 : 32;
    const bool lam_sm = m <= LAM_CAP;
    double *lt1s = lam + LAM_CAP * SW_T, *lt2s = lam + 2 * LAM_CAP * SW_T;
    if (lam_sm)  // accumulators in: asynchronous copies, one wait (no per-row round trip)
        for (int j = 0; j < m; ++j) {
            __pipeline_memcpy_async(lt1s + j * SW_T, io.lam_t1 + base + step * j, 8);
            __pipeline_memcpy_async(lt2s + j * SW_T, io.lam_t2 + base + step * j, 8);
        }
    for (int phi = 0; phi < n_phases; ++phi) {
        const SweepPhase ph = phs[phi];
        if (ph.iters <= 0) continue;
        if (lam_sm) {
            for (int j = 0; j < m; ++j) __pipeline_memcpy_async(lam + j * SW_T, ph.lam_n + base + step * j, 8);
            __pipeline_commit();
            __pipeline_wait_prior(0);
        }
        const int64_t T = ph.iters * (int64_t)m;
        // prologue: steps 0 .. RING - 2, one commit group per step
        int js = 0;  // row of the next step to stage
        for (int p = 0; p < RING - 1; ++p) {
            if (p < T) stage_row<FIX>(ring + p * ROW_F * SW_T, io, ph, rows, base + step * js);
            __pipeline_commit();
            if (++js == m) js = 0;
        }
        int j = 0;
        for (int64_t q = 0; q < T; ++q) {
            __pipeline_wait_prior(RING - 2);  // step q's row has landed
            const double *r = ring + (int)(q % RING) * ROW_F * SW_T;
            double a[3], b[3], n[3], t1[3], t2[3];
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                a[k] = r[k * SW_T]; b[k] = r[(3 + k) * SW_T]; n[k] = r[(6 + k) * SW_T];
                t1[k] = r[(9 + k) * SW_T]; t2[k] = r[(12 + k) * SW_T];
            }
            const double kn = r[15 * SW_T], kt1 = r[16 * SW_T], kt2 = r[17 * SW_T], tg = r[18 * SW_T],
                         mu = r[19 * SW_T];
            const int ia = FIX ? 0 : (int)__double_as_longlong(r[20 * SW_T]);
            const int ib = FIX ? 1 : (int)__double_as_longlong(r[21 * SW_T]);
            // refill the slot consumed by the previous step (its reads are complete)
            if (q + RING - 1 < T)
                stage_row<FIX>(ring + (int)((q + RING - 1) % RING) * ROW_F * SW_T, io, ph, rows, base + step * js);
            __pipeline_commit();
            if (++js == m) js = 0;
            const int64_t c = base + step * j;
            double *pln = lam_sm ? lam + j * SW_T : ph.lam_n + c;
            double *plt1 = lam_sm ? lt1s + j * SW_T : io.lam_t1 + c;
            double *plt2 = lam_sm ? lt2s + j * SW_T : io.lam_t2 + c;
            solve_row(st, ia, ib, a, b, n, t1, t2, kn, kt1, kt2, tg, mu, pln, plt1, plt2, ph.with_friction);
            if (++j == m) j = 0;
        }
        __pipeline_wait_prior(0);
        if (lam_sm)
            for (int jj = 0; jj < m; ++jj) ph.lam_n[base + step * jj] = lam[jj * SW_T];
    }
    __pipeline_commit();
    __pipeline_wait_prior(0);
    if (lam_sm)
        for (int jj = 0; jj < m; ++jj) {
            io.lam_t1[base + step * jj] = lt1s[jj * SW_T];
            io.lam_t2[base + step * jj] = lt2s[jj * SW_T];
        }
}

// gauss_seidel_sweeps (_kernels.py:52-115), one system per thread, 1-2 phases.
// TWO: the two-body register path (nb == 2).
template <int MODE, bool FIX>
__global__ void __launch_bounds__(SW_T) k_sweeps(int64_t S, int nb, SysRows rows, SweepIO io, SweepPhase p0,
                                                 SweepPhase p1, int n_phases) {
    extern __shared__ double sm[];
    const int64_t s = blockIdx.x * (int64_t)SW_T + threadIdx.x;
    if (s >= S) return;
    const int nv = 6 * nb;
    constexpr bool GLOBAL = MODE == 1;  // systems above SOLVER_SMEM_BODIES: the state stays in global memory
    static_assert(!GLOBAL || SW_T == 1, "global body state is addressed with the shared columns' stride");
    const double *Ws = GLOBAL ? io.w_mat + s * 36 * nb : sm + threadIdx.x;  // [36 nb][SW_T]
    if (!GLOBAL)
        for (int j = 0; j < 36 * nb; ++j) sm[threadIdx.x + j * SW_T] = __ldg(io.w_mat + s * 36 * nb + j);
    constexpr bool TWO = MODE == 2;
    double *after_w = GLOBAL ? sm : sm + (size_t)36 * nb * SW_T + (MODE ? 0 : (size_t)12 * nb * SW_T);
    double *ring = after_w + threadIdx.x;
    double *lam = after_w + (size_t)RING * ROW_F * SW_T + threadIdx.x;
    const SweepPhase phs[2] = {p0, p1};
    if (TWO) {
        RegState2 st;
        st.W = Ws;
#pragma unroll
        for (int k = 0; k < 6; ++k) {
            st.v0[k] = io.vel[s * 12 + k]; st.v1[k] = io.vel[s * 12 + 6 + k];
            st.i0[k] = io.imp[s * 12 + k]; st.i1[k] = io.imp[s * 12 + 6 + k];
        }
        st.z0 = frozen_body(Ws, st.v0);
        st.z1 = frozen_body(Ws + 36 * SW_T, st.v1);
        sweep_system<FIX>(st, io, phs, n_phases, rows, s, ring, lam);
#pragma unroll
        for (int k = 0; k < 6; ++k) {
            io.vel[s * 12 + k] = st.v0[k]; io.vel[s * 12 + 6 + k] = st.v1[k];
            io.imp[s * 12 + k] = st.i0[k]; io.imp[s * 12 + 6 + k] = st.i1[k];
        }
    } else if (MODE == 4) {
        RegStateN<4> st;
        st.W = Ws;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
#pragma unroll
            for (int k = 0; k < 6; ++k) {
                st.v_[b][k] = b < nb ? io.vel[s * nv + 6 * b + k] : 0.0;
                st.i_[b][k] = b < nb ? io.imp[s * nv + 6 * b + k] : 0.0;
            }
            st.z_[b] = b < nb ? frozen_body(Ws + 36 * b * SW_T, st.v_[b]) : true;
        }
        sweep_system<false>(st, io, phs, n_phases, rows, s, ring, lam);
#pragma unroll
        for (int b = 0; b < 4; ++b)
            if (b < nb)
#pragma unroll
                for (int k = 0; k < 6; ++k) {
                    io.vel[s * nv + 6 * b + k] = st.v_[b][k];
                    io.imp[s * nv + 6 * b + k] = st.i_[b][k];
                }
    } else if (GLOBAL) {  // velocities and impulses updated in place (one thread owns the system)
        SmemState st;
        st.W = Ws;
        st.V = io.vel + s * nv;
        st.I = io.imp + s * nv;
        sweep_system<false>(st, io, phs, n_phases, rows, s, ring, lam);
    } else {
        SmemState st;
        st.W = Ws;
        st.V = sm + 36 * nb * SW_T + threadIdx.x;
        st.I = st.V + nv * SW_T;
        for (int j = 0; j < nv; ++j) {
            st.V[j * SW_T] = io.vel[s * nv + j];
            st.I[j * SW_T] = io.imp[s * nv + j];
        }
        sweep_system<false>(st, io, phs, n_phases, rows, s, ring, lam);
        for (int j = 0; j < nv; ++j) {
            io.vel[s * nv + j] = st.V[j * SW_T];
            io.imp[s * nv + j] = st.I[j * SW_T];
        }
    }
}

// ------------------------------------------------------------------ packed rows + bulk copies
//
// The plan paths (cs_plan_solve, cs_multipair_solve) pack each row's sweep fields
// into one 176-byte record after the build; the sweep then streams chunks of
// PK_CH records of its system into a shared-memory double buffer with one TMA
// bulk copy (cp.async.bulk, mbarrier completion) per chunk instead of 20 8-byte
// asynchronous copies per row (LDGSTS: 8 issue cycles each).
constexpr int PK_F = 22;  // a[3] b[3] n[3] t1[3] t2[3] kn kt1 kt2 target(pos) target(vel) mu ids(2 x i32)
constexpr int PK_CH = 8;  // rows per bulk copy

__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void bulk_load(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT%=;\n}" ::"r"(
            smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// rows (interleaved) -> records packed[(s stride + j) PK_F + f]; a thread per row slot
__global__ void k_pack_rows(int64_t S, SysRows rows, SweepIO io, const double *tg_pos, const double *tg_vel,
                            double *__restrict__ packed) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= rows.planes) return;
    const int64_t blk = (t >> 5) / rows.stride, j = (t >> 5) % rows.stride, s = blk * 32 + (t & 31);
    if (s >= S || j >= rows.n(s)) return;
    double *o = packed + (s * rows.stride + j) * PK_F;
    for (int k = 0; k < 3; ++k) {
        const int64_t v = rows.vec(t, k);
        o[k] = io.ra[v]; o[3 + k] = io.rb[v]; o[6 + k] = io.nrm[v]; o[9 + k] = io.tan1[v]; o[12 + k] = io.tan2[v];
    }
    o[15] = io.kn[t]; o[16] = io.kt1[t]; o[17] = io.kt2[t];
    o[18] = tg_pos[t]; o[19] = tg_vel[t]; o[20] = io.mu[t];
    const int2 ids = make_int2((int)io.body_a[t], (int)io.body_b[t]);
    o[21] = __longlong_as_double(((long long)(unsigned)ids.y << 32) | (unsigned)ids.x);
}

template <bool FIX, class St>
__device__ __forceinline__ void sweep_packed(St &st, const SweepIO &io, const SweepPhase *phs, int n_phases,
                                             const SysRows &rows, int64_t s, const double *packed, double *buf,
                                             uint64_t *bar, double *lam) {
    const int m = (int)rows.n(s);
    if (m <= 0) return;
    const int64_t base = rows.row(s, 0), step = 32;  // accumulators stay in the interleaved layout
    const double *src = packed + s * rows.stride * PK_F;
    const bool lam_sm = m <= LAM_CAP;
    double *lt1s = lam + LAM_CAP * SW_T, *lt2s = lam + 2 * LAM_CAP * SW_T;
    if (lam_sm)
        for (int j = 0; j < m; ++j) {
            __pipeline_memcpy_async(lt1s + j * SW_T, io.lam_t1 + base + step * j, 8);
            __pipeline_memcpy_async(lt2s + j * SW_T, io.lam_t2 + base + step * j, 8);
        }
    const int nch = (m + PK_CH - 1) / PK_CH;
    unsigned use0 = 0, use1 = 0;  // completed phases of each buffer's barrier
    auto issue = [&](int k, int b) {
        const int r0 = k * PK_CH, nr = min(PK_CH, m - r0);
        fence_proxy_async();  // the buffer's previous rows were read through the generic proxy
        bulk_load(buf + b * PK_CH * PK_F, src + (int64_t)r0 * PK_F, (unsigned)(nr * PK_F * sizeof(double)), bar + b);
    };
    for (int phi = 0; phi < n_phases; ++phi) {
        const SweepPhase ph = phs[phi];
        if (ph.iters <= 0) continue;
        if (lam_sm) {
            for (int j = 0; j < m; ++j) __pipeline_memcpy_async(lam + j * SW_T, ph.lam_n + base + step * j, 8);
            __pipeline_commit();
            __pipeline_wait_prior(0);
        }
        const bool pos = phi == 0;  // targets: phase 0 the bias, phase 1 the restitution (record fields 18 / 19)
        const int64_t T = ph.iters * (int64_t)nch;
        issue(0, 0);
        for (int64_t q = 0; q < T; ++q) {
            const int b = (int)(q & 1), k = (int)(q % nch);
            if (q + 1 < T) issue((int)((q + 1) % nch), b ^ 1);
            mbar_wait(bar + b, b ? (use1++ & 1) : (use0++ & 1));
            const double *rb = buf + b * PK_CH * PK_F;
            const int r0 = k * PK_CH, nr = min(PK_CH, m - r0);
            for (int r = 0; r < nr; ++r) {
                const double2 *w2 = reinterpret_cast<const double2 *>(rb + r * PK_F);
                double f[PK_F];
#pragma unroll
                for (int i = 0; i < PK_F / 2; ++i) { const double2 x = w2[i]; f[2 * i] = x.x; f[2 * i + 1] = x.y; }
                const double a[3] = {f[0], f[1], f[2]}, bb[3] = {f[3], f[4], f[5]}, n[3] = {f[6], f[7], f[8]};
                const double t1[3] = {f[9], f[10], f[11]}, t2[3] = {f[12], f[13], f[14]};
                const long long ids = __double_as_longlong(f[21]);
                const int ia = FIX ? 0 : (int)(ids & 0xffffffff), ib = FIX ? 1 : (int)(ids >> 32);
                const int j = r0 + r;
                const int64_t c = base + step * j;
                double *pln = lam_sm ? lam + j * SW_T : ph.lam_n + c;
                double *plt1 = lam_sm ? lt1s + j * SW_T : io.lam_t1 + c;
                double *plt2 = lam_sm ? lt2s + j * SW_T : io.lam_t2 + c;
                solve_row(st, ia, ib, a, bb, n, t1, t2, f[15], f[16], f[17], pos ? f[18] : f[19], f[20], pln, plt1, plt2,
                          ph.with_friction);
            }
        }
        if (lam_sm)
            for (int jj = 0; jj < m; ++jj) ph.lam_n[base + step * jj] = lam[jj * SW_T];
    }
    __pipeline_commit();
    __pipeline_wait_prior(0);
    if (lam_sm)
        for (int jj = 0; jj < m; ++jj) {
            io.lam_t1[base + step * jj] = lt1s[jj * SW_T];
            io.lam_t2[base + step * jj] = lt2s[jj * SW_T];
        }
}

__host__ __device__ inline size_t packed_smem_doubles(int nb, bool regs) {
    if (nb > SOLVER_SMEM_BODIES) return (size_t)2 * PK_CH * PK_F + 3 * (size_t)LAM_CAP;
    return (size_t)36 * nb + (regs ? 0 : (size_t)12 * nb) + (size_t)2 * PK_CH * PK_F + 3 * (size_t)LAM_CAP;
}

// The plan paths' sweeps (interleaved rows, packed records): one system per
// thread (SW_T == 1 block), MODE as k_sweeps.
template <int MODE, bool FIX>
__global__ void __launch_bounds__(SW_T) k_sweeps_packed(int64_t S, int nb, SysRows rows, SweepIO io,
                                                        const double *__restrict__ packed, SweepPhase p0,
                                                        SweepPhase p1, int n_phases) {
    extern __shared__ __align__(16) double sm[];
    __shared__ uint64_t bar[2];
    const int64_t s = blockIdx.x * (int64_t)SW_T + threadIdx.x;
    if (s >= S) return;
    static_assert(SW_T == 1, "the packed sweep runs one system per block");
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
    fence_proxy_async();
    const int nv = 6 * nb;
    constexpr bool GLOBAL = MODE == 1;  // as k_sweeps
    const double *Ws = GLOBAL ? io.w_mat + s * 36 * nb : sm;
    if (!GLOBAL)
        for (int j = 0; j < 36 * nb; ++j) sm[j] = __ldg(io.w_mat + s * 36 * nb + j);
    double *after_w = GLOBAL ? sm : sm + (size_t)36 * nb + (MODE ? 0 : (size_t)12 * nb);
    double *buf = after_w;  // 16-byte aligned: 36 nb (+ 12 nb) doubles are a multiple of 2
    double *lam = after_w + 2 * PK_CH * PK_F;
    const SweepPhase phs[2] = {p0, p1};
    if (MODE == 2) {
        RegState2 st;
        st.W = Ws;
#pragma unroll
        for (int k = 0; k < 6; ++k) {
            st.v0[k] = io.vel[s * 12 + k]; st.v1[k] = io.vel[s * 12 + 6 + k];
            st.i0[k] = io.imp[s * 12 + k]; st.i1[k] = io.imp[s * 12 + 6 + k];
        }
        st.z0 = frozen_body(Ws, st.v0);
        st.z1 = frozen_body(Ws + 36 * SW_T, st.v1);
        sweep_packed<FIX>(st, io, phs, n_phases, rows, s, packed, buf, bar, lam);
#pragma unroll
        for (int k = 0; k < 6; ++k) {
            io.vel[s * 12 + k] = st.v0[k]; io.vel[s * 12 + 6 + k] = st.v1[k];
            io.imp[s * 12 + k] = st.i0[k]; io.imp[s * 12 + 6 + k] = st.i1[k];
        }
    } else if (MODE == 4) {
        RegStateN<4> st;
        st.W = Ws;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
#pragma unroll
            for (int k = 0; k < 6; ++k) {
                st.v_[b][k] = b < nb ? io.vel[s * nv + 6 * b + k] : 0.0;
                st.i_[b][k] = b < nb ? io.imp[s * nv + 6 * b + k] : 0.0;
            }
            st.z_[b] = b < nb ? frozen_body(Ws + 36 * b * SW_T, st.v_[b]) : true;
        }
        sweep_packed<FIX>(st, io, phs, n_phases, rows, s, packed, buf, bar, lam);
#pragma unroll
        for (int b = 0; b < 4; ++b)
            if (b < nb)
#pragma unroll
                for (int k = 0; k < 6; ++k) {
                    io.vel[s * nv + 6 * b + k] = st.v_[b][k];
                    io.imp[s * nv + 6 * b + k] = st.i_[b][k];
                }
    } else if (GLOBAL) {
        SmemState st;
        st.W = Ws;
        st.V = io.vel + s * nv;
        st.I = io.imp + s * nv;
        sweep_packed<FIX>(st, io, phs, n_phases, rows, s, packed, buf, bar, lam);
    } else {
        SmemState st;
        st.W = Ws;
        st.V = sm + 36 * nb;
        st.I = st.V + nv;
        for (int j = 0; j < nv; ++j) {
            st.V[j] = io.vel[s * nv + j];
            st.I[j] = io.imp[s * nv + j];
        }
        sweep_packed<FIX>(st, io, phs, n_phases, rows, s, packed, buf, bar, lam);
        for (int j = 0; j < nv; ++j) {
            io.vel[s * nv + j] = st.V[j];
            io.imp[s * nv + j] = st.I[j];
        }
    }
}

// ContactConstraints.body_wrenches (solver.py:154-163). A warp per system: the lanes
// compute the rows' terms (j/h, (r x j)/h) in parallel into shared memory, then
// one lane per output element accumulates them in row order (b's terms before a's
// within a row, as the reference's four statements run).
constexpr int WR_WARPS = 4, WR_TILE = 32;

__global__ void __launch_bounds__(WR_WARPS * 32) k_body_wrenches(int64_t S, int nb, SysRows rows, WrenchIO io) {
    __shared__ double tb[WR_WARPS][WR_TILE][6], ta[WR_WARPS][WR_TILE][6];
    __shared__ int bi[WR_WARPS][WR_TILE][2];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t s = blockIdx.x * (int64_t)WR_WARPS + w;
    if (s >= S) return;
    const int nv = 6 * nb;  // elements in groups of 64: lane owns e0 + lane and e0 + lane + 32
    const int64_t m = rows.n(s);
    const double h = io.h;
    for (int e0 = 0; e0 < nv; e0 += 64) {  // one group up to 10 bodies; larger systems recompute the row terms
    double acc0 = 0.0, acc1 = 0.0;
    for (int64_t t0 = 0; t0 < m; t0 += WR_TILE) {
        if (t0 + lane < m) {
            const int64_t c = rows.row(s, t0 + lane);
            const double lam = io.lam_n[c] + io.lam_vel[c];
            const double l1 = io.lam_t1[c], l2 = io.lam_t2[c];
            double j[3], a[3], b[3];
            for (int k = 0; k < 3; ++k) {
                const int64_t v = rows.vec(c, k);
                j[k] = (lam * io.nrm[v] + l1 * io.tan1[v]) + l2 * io.tan2[v];
                a[k] = io.ra[v];
                b[k] = io.rb[v];
            }
            const double cb[3] = {b[1] * j[2] - b[2] * j[1], b[2] * j[0] - b[0] * j[2], b[0] * j[1] - b[1] * j[0]};
            const double ca[3] = {a[1] * j[2] - a[2] * j[1], a[2] * j[0] - a[0] * j[2], a[0] * j[1] - a[1] * j[0]};
            for (int k = 0; k < 3; ++k) {
                const double jh = j[k] / h;
                tb[w][lane][k] = jh;
                ta[w][lane][k] = jh;
                tb[w][lane][3 + k] = cb[k] / h;
                ta[w][lane][3 + k] = ca[k] / h;
            }
            bi[w][lane][0] = (int)io.body_b[c];
            bi[w][lane][1] = (int)io.body_a[c];
        }
        __syncwarp();
        const int n = m - t0 < WR_TILE ? (int)(m - t0) : WR_TILE;
        for (int q = 0; q < 2; ++q) {
            const int el = e0 + lane + 32 * q;
            if (el >= nv) break;
            const int body = el / 6, k = el - 6 * body;
            double acc = q ? acc1 : acc0;
            for (int i = 0; i < n; ++i) {
                if (bi[w][i][0] == body) acc += tb[w][i][k];
                if (bi[w][i][1] == body) acc -= ta[w][i][k];
            }
            if (q) acc1 = acc; else acc0 = acc;
        }
        __syncwarp();
    }
    if (e0 + lane < nv) io.out[s * nv + e0 + lane] = acc0;
    if (e0 + lane + 32 < nv) io.out[s * nv + e0 + lane + 32] = acc1;
    }
}

// Scene rows of a plan's reduced contacts: warp per system; its pair slots in
// order, each slot's patches (up to n_patch: later slots are stale) in slot order
__global__ void k_plan_rows(int64_t S, PlanRowsIO io) {
    const int64_t s = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (s >= S) return;
    const int N = io.N, K = io.K;
    const int64_t t0 = io.slot_off ? io.slot_off[s] : s, t1 = io.slot_off ? io.slot_off[s + 1] : s + 1;
    int run = 0;
    for (int64_t e = t0; e < t1; ++e) {
        const double mu = io.env_mu[e], rest = io.env_restitution[e], slop = io.env_slop[e];
        const int64_t ba = io.slot_a ? io.slot_a[e] : 0, bb = io.slot_b ? io.slot_b[e] : 1;
        const int np = io.n_patch[e];
        for (int p0 = 0; p0 < np; p0 += 32) {
            const int p = p0 + lane;
            const int nk = p < np ? io.patch_nkept[e * N + p] : 0;
            int inc = nk;
            for (int o = 1; o < 32; o <<= 1) {
                const int v = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += v;
            }
            const int64_t base = run + inc - nk;
            for (int k = 0; k < nk; ++k) {
                const int64_t src = ((int64_t)e * N + p) * K + k, r = io.rows.row(s, base + k);
                io.body_a[r] = ba;
                io.body_b[r] = bb;
                for (int q = 0; q < 3; ++q) {
                    io.point[io.rows.vec(r, q)] = io.kept_point[3 * src + q];
                    io.normal[io.rows.vec(r, q)] = io.kept_normal[3 * src + q];
                }
                io.depth[r] = io.kept_depth[src];
                io.mu[r] = mu;
                io.restitution[r] = rest;
                io.slop[r] = slop;
            }
            run += __shfl_sync(0xffffffffu, inc, 31);
        }
    }
    if (io.count_out && lane == 0) io.count_out[s] = run;
}

}  // namespace

void launch_constraints_build(int64_t n_sys, int nb, const SysRows &rows, const BuildIO &io, cudaStream_t s) {
    if (n_sys <= 0) return;
    const int64_t threads = rows.off ? n_sys * 32 : rows.planes;
    k_constraints_build<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(n_sys, nb, rows, io);
}

void launch_sweeps(int64_t n_sys, int nb, const SysRows &rows, const SweepIO &io, const SweepPhase *phases,
                   int n_phases, cudaStream_t s, bool fixed_bodies) {
    if (n_sys <= 0 || n_phases <= 0) return;
    const unsigned grid = (unsigned)((n_sys + SW_T - 1) / SW_T);
    const SweepPhase p1 = n_phases > 1 ? phases[1] : phases[0];
    const bool two = nb == 2, regs = nb <= 4;
    const size_t smem = sweep_smem_doubles(nb, regs) * SW_T * sizeof(double);
    auto go = [&](auto kern) {
        if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<grid, SW_T, smem, s>>>(n_sys, nb, rows, io, phases[0], p1, n_phases);
    };
    if (two && fixed_bodies) go(k_sweeps<2, true>);
    else if (two) go(k_sweeps<2, false>);
    else if (regs) go(k_sweeps<4, false>);
    else if (nb > SOLVER_SMEM_BODIES) go(k_sweeps<1, false>);
    else go(k_sweeps<0, false>);
}

void launch_sweeps_packed(int64_t n_sys, int nb, const SysRows &rows, const SweepIO &io, const SweepPhase *phases,
                          int n_phases, double *packed, cudaStream_t s, bool fixed_bodies) {
    if (n_sys <= 0 || n_phases <= 0) return;
    k_pack_rows<<<(unsigned)((rows.planes + 255) / 256), 256, 0, s>>>(n_sys, rows, io, phases[0].target,
                                                                       n_phases > 1 ? phases[1].target
                                                                                    : phases[0].target,
                                                                       packed);
    const unsigned grid = (unsigned)((n_sys + SW_T - 1) / SW_T);
    const SweepPhase p1 = n_phases > 1 ? phases[1] : phases[0];
    const bool two = nb == 2, regs = nb <= 4;
    const size_t smem = packed_smem_doubles(nb, regs) * sizeof(double);
    auto go = [&](auto kern) {
        if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<grid, SW_T, smem, s>>>(n_sys, nb, rows, io, packed, phases[0], p1, n_phases);
    };
    if (two && fixed_bodies) go(k_sweeps_packed<2, true>);
    else if (two) go(k_sweeps_packed<2, false>);
    else if (regs) go(k_sweeps_packed<4, false>);
    else if (nb > SOLVER_SMEM_BODIES) go(k_sweeps_packed<1, false>);
    else go(k_sweeps_packed<0, false>);
}

void launch_body_wrenches(int64_t n_sys, int nb, const SysRows &rows, const WrenchIO &io, cudaStream_t s) {
    if (n_sys <= 0) return;
    k_body_wrenches<<<(unsigned)((n_sys + WR_WARPS - 1) / WR_WARPS), WR_WARPS * 32, 0, s>>>(n_sys, nb, rows, io);
}

void launch_plan_rows(int64_t S, const PlanRowsIO &io, cudaStream_t s) {
    if (S <= 0) return;
    k_plan_rows<<<(unsigned)((S * 32 + 255) / 256), 256, 0, s>>>(S, io);
}

}  // namespace cs
