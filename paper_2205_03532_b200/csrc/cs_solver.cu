// Contact solver kernels (cs_solver.cuh). Compiled with -fmad=false like the rest
// of the library: numba's sweep kernel has no FMA contraction, and the numpy
// products of ContactConstraints.build are OpenBLAS kernels whose rounding is
// written out with explicit fma (measured against the reference in this
// container; oracle/cs_oracle_solver.c carries the same formulas and is pinned to
// the reference's outputs).
//
// The sweep is sequential within a system (every row reads the velocities the
// previous row wrote), so a system is one thread: its body velocities and
// impulses live in shared memory (row-independent layout, conflict-free), and
// the next row's constraint data and accumulators are loaded while the current
// row is solved, which takes the L2 latency off the dependency chain. Systems
// are independent and run side by side.
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

// ContactConstraints.build: rows are independent; a warp per system, lanes over rows.
__global__ void k_constraints_build(int64_t S, int nb, SysRows rows, BuildIO io) {
    const int64_t s = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (s >= S) return;
    const int64_t r0 = rows.begin(s), r1 = rows.end(s);
    const int64_t b0 = s * nb;
    for (int64_t c = r0 + lane; c < r1; c += 32) {
        const int64_t ia = b0 + io.body_a[c], ib = b0 + io.body_b[c];
        double p[3], n[3], a[3], b[3], t1[3], t2[3];
        for (int k = 0; k < 3; ++k) {
            p[k] = io.point[3 * c + k];
            n[k] = io.normal[3 * c + k];
            a[k] = p[k] - io.ref[3 * ia + k];
            b[k] = p[k] - io.ref[3 * ib + k];
        }
        tangent_basis(n, t1, t2);
        for (int k = 0; k < 3; ++k) {
            io.ra[3 * c + k] = a[k]; io.rb[3 * c + k] = b[k];
            io.tan1[3 * c + k] = t1[k]; io.tan2[3 * c + k] = t2[k];
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
}

constexpr int SW_T = 32;  // systems per sweep block, one thread each

struct Row {
    int ia, ib;
    double a[3], b[3], n[3], t1[3], t2[3];
    double kn, kt1, kt2, tg, mu;
    double ln, lt1, lt2;
};

__device__ __forceinline__ void load_row(Row &r, const SweepIO &io, const SweepPhase &ph, int64_t c) {
    r.ia = (int)__ldg(io.body_a + c);
    r.ib = (int)__ldg(io.body_b + c);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        r.a[k] = __ldg(io.ra + 3 * c + k);
        r.b[k] = __ldg(io.rb + 3 * c + k);
        r.n[k] = __ldg(io.nrm + 3 * c + k);
        r.t1[k] = __ldg(io.tan1 + 3 * c + k);
        r.t2[k] = __ldg(io.tan2 + 3 * c + k);
    }
    r.kn = __ldg(io.kn + c);
    r.kt1 = __ldg(io.kt1 + c);
    r.kt2 = __ldg(io.kt2 + c);
    r.tg = __ldg(ph.target + c);
    r.mu = __ldg(io.mu + c);
    // accumulators: written by this kernel, so plain (coherent) loads
    r.ln = ph.lam_n[c];
    r.lt1 = io.lam_t1[c];
    r.lt2 = io.lam_t2[c];
}

// _kernels.py:16-37 on the thread's shared-memory state (element j of the
// system's [nb][6] arrays at V[j * SW_T])
__device__ __forceinline__ void apply_impulse(const double *__restrict__ W, double *V, double *I, int body, double jx,
                                              double jy, double jz, double rx, double ry, double rz, double sign) {
    const double gx = jx * sign, gy = jy * sign, gz = jz * sign;
    const double tx = (ry * jz - rz * jy) * sign;
    const double ty = (rz * jx - rx * jz) * sign;
    const double tz = (rx * jy - ry * jx) * sign;
    const double *w = W + 36 * body;
#pragma unroll
    for (int k = 0; k < 6; ++k) {
        const double t = __ldg(w + 6 * k) * gx + __ldg(w + 6 * k + 1) * gy + __ldg(w + 6 * k + 2) * gz +
                         __ldg(w + 6 * k + 3) * tx + __ldg(w + 6 * k + 4) * ty + __ldg(w + 6 * k + 5) * tz;
        V[(6 * body + k) * SW_T] += t;
    }
    I[(6 * body) * SW_T] += gx;
    I[(6 * body + 1) * SW_T] += gy;
    I[(6 * body + 2) * SW_T] += gz;
    I[(6 * body + 3) * SW_T] += tx;
    I[(6 * body + 4) * SW_T] += ty;
    I[(6 * body + 5) * SW_T] += tz;
}

// _kernels.py:40-49
__device__ __forceinline__ double rel_vel(const double *V, int ia, int ib, const double a[3], const double b[3],
                                          double dx, double dy, double dz) {
    const double *vb = V + 6 * ib * SW_T, *va = V + 6 * ia * SW_T;
    const double vb0 = vb[0], vb1 = vb[SW_T], vb2 = vb[2 * SW_T], vb3 = vb[3 * SW_T], vb4 = vb[4 * SW_T],
                 vb5 = vb[5 * SW_T];
    const double va0 = va[0], va1 = va[SW_T], va2 = va[2 * SW_T], va3 = va[3 * SW_T], va4 = va[4 * SW_T],
                 va5 = va[5 * SW_T];
    const double ubx = vb0 + vb4 * b[2] - vb5 * b[1];
    const double uby = vb1 + vb5 * b[0] - vb3 * b[2];
    const double ubz = vb2 + vb3 * b[1] - vb4 * b[0];
    const double uax = va0 + va4 * a[2] - va5 * a[1];
    const double uay = va1 + va5 * a[0] - va3 * a[2];
    const double uaz = va2 + va3 * a[1] - va4 * a[0];
    return (ubx - uax) * dx + (uby - uay) * dy + (ubz - uaz) * dz;
}

// gauss_seidel_sweeps (_kernels.py:52-115), one system per thread, 1-2 phases
__global__ void __launch_bounds__(SW_T) k_sweeps(int64_t S, int nb, SysRows rows, SweepIO io, SweepPhase p0,
                                                 SweepPhase p1, int n_phases) {
    extern __shared__ double sm[];
    const int64_t s = blockIdx.x * (int64_t)SW_T + threadIdx.x;
    if (s >= S) return;
    const int nv = 6 * nb;
    double *V = sm + threadIdx.x, *I = sm + nv * SW_T + threadIdx.x;
    for (int j = 0; j < nv; ++j) {
        V[j * SW_T] = io.vel[s * nv + j];
        I[j * SW_T] = io.imp[s * nv + j];
    }
    const double *W = io.w_mat + s * nb * 36;
    const int64_t r0 = rows.begin(s), r1 = rows.end(s);
    if (r1 > r0) {
        for (int phi = 0; phi < n_phases; ++phi) {
            const SweepPhase ph = phi ? p1 : p0;
            if (ph.iters <= 0) continue;
            Row cur, nxt;
            load_row(cur, io, ph, r0);
            for (int64_t it = 0; it < ph.iters; ++it) {
                for (int64_t c = r0; c < r1; ++c) {
                    // next row of the sweep (wrapping into the next iteration)
                    const int64_t cn = c + 1 < r1 ? c + 1 : r0;
                    const bool more = c + 1 < r1 || it + 1 < ph.iters;
                    if (more) load_row(nxt, io, ph, cn);
                    if (cur.kn > 0.0) {
                        const double vn = rel_vel(V, cur.ia, cur.ib, cur.a, cur.b, cur.n[0], cur.n[1], cur.n[2]);
                        double dl = cur.kn * (cur.tg - vn);
                        double new_l = cur.ln + dl;
                        if (new_l < 0.0) new_l = 0.0;
                        dl = new_l - cur.ln;
                        cur.ln = new_l;
                        ph.lam_n[c] = new_l;
                        if (dl != 0.0) {
                            const double jx = dl * cur.n[0], jy = dl * cur.n[1], jz = dl * cur.n[2];
                            apply_impulse(W, V, I, cur.ib, jx, jy, jz, cur.b[0], cur.b[1], cur.b[2], 1.0);
                            apply_impulse(W, V, I, cur.ia, jx, jy, jz, cur.a[0], cur.a[1], cur.a[2], -1.0);
                        }
                    }
                    if (ph.with_friction && cur.mu > 0.0 && cur.ln > 0.0) {
                        double d1 = 0.0, d2 = 0.0;
                        if (cur.kt1 > 0.0)
                            d1 = -cur.kt1 * rel_vel(V, cur.ia, cur.ib, cur.a, cur.b, cur.t1[0], cur.t1[1], cur.t1[2]);
                        if (cur.kt2 > 0.0)
                            d2 = -cur.kt2 * rel_vel(V, cur.ia, cur.ib, cur.a, cur.b, cur.t2[0], cur.t2[1], cur.t2[2]);
                        double new1 = cur.lt1 + d1, new2 = cur.lt2 + d2;
                        const double limit = cur.mu * cur.ln;
                        const double mag = sqrt(new1 * new1 + new2 * new2);
                        if (mag > limit) {
                            const double scale = limit / mag;
                            new1 *= scale;
                            new2 *= scale;
                        }
                        d1 = new1 - cur.lt1;
                        d2 = new2 - cur.lt2;
                        cur.lt1 = new1;
                        cur.lt2 = new2;
                        io.lam_t1[c] = new1;
                        io.lam_t2[c] = new2;
                        if (d1 != 0.0 || d2 != 0.0) {
                            const double jx = d1 * cur.t1[0] + d2 * cur.t2[0];
                            const double jy = d1 * cur.t1[1] + d2 * cur.t2[1];
                            const double jz = d1 * cur.t1[2] + d2 * cur.t2[2];
                            apply_impulse(W, V, I, cur.ib, jx, jy, jz, cur.b[0], cur.b[1], cur.b[2], 1.0);
                            apply_impulse(W, V, I, cur.ia, jx, jy, jz, cur.a[0], cur.a[1], cur.a[2], -1.0);
                        }
                    }
                    if (more) {
                        if (cn == c) {  // a one-row system: the prefetch predates this row's writes
                            nxt.ln = cur.ln;
                            nxt.lt1 = cur.lt1;
                            nxt.lt2 = cur.lt2;
                        }
                        cur = nxt;
                    }
                }
            }
        }
    }
    for (int j = 0; j < nv; ++j) {
        io.vel[s * nv + j] = V[j * SW_T];
        io.imp[s * nv + j] = I[j * SW_T];
    }
}

// ContactConstraints.body_wrenches (solver.py:154-163), rows in order per system
__global__ void __launch_bounds__(SW_T) k_body_wrenches(int64_t S, int nb, SysRows rows, WrenchIO io) {
    extern __shared__ double sm[];
    const int64_t s = blockIdx.x * (int64_t)SW_T + threadIdx.x;
    if (s >= S) return;
    const int nv = 6 * nb;
    double *O = sm + threadIdx.x;
    for (int j = 0; j < nv; ++j) O[j * SW_T] = 0.0;
    const int64_t r0 = rows.begin(s), r1 = rows.end(s);
    const double h = io.h;
    for (int64_t c = r0; c < r1; ++c) {
        const double lam = io.lam_n[c] + io.lam_vel[c];
        const double l1 = io.lam_t1[c], l2 = io.lam_t2[c];
        double j[3], a[3], b[3];
        for (int k = 0; k < 3; ++k) {
            j[k] = (lam * io.nrm[3 * c + k] + l1 * io.tan1[3 * c + k]) + l2 * io.tan2[3 * c + k];
            a[k] = io.ra[3 * c + k];
            b[k] = io.rb[3 * c + k];
        }
        const double cb[3] = {b[1] * j[2] - b[2] * j[1], b[2] * j[0] - b[0] * j[2], b[0] * j[1] - b[1] * j[0]};
        const double ca[3] = {a[1] * j[2] - a[2] * j[1], a[2] * j[0] - a[0] * j[2], a[0] * j[1] - a[1] * j[0]};
        const int ib = (int)io.body_b[c], ia = (int)io.body_a[c];
        for (int k = 0; k < 3; ++k) {
            O[(6 * ib + k) * SW_T] += j[k] / h;
            O[(6 * ib + 3 + k) * SW_T] += cb[k] / h;
            O[(6 * ia + k) * SW_T] -= j[k] / h;
            O[(6 * ia + 3 + k) * SW_T] -= ca[k] / h;
        }
    }
    for (int j = 0; j < nv; ++j) io.out[s * nv + j] = O[j * SW_T];
}

// Scene rows of a plan's reduced contacts: warp per env, patches scanned in slot order
__global__ void k_plan_rows(int64_t E, PlanRowsIO io) {
    const int64_t e = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (e >= E) return;
    const int N = io.N, K = io.K;
    const double mu = io.env_mu[e], rest = io.env_restitution[e], slop = io.env_slop[e];
    int run = 0;
    for (int p0 = 0; p0 < N; p0 += 32) {
        const int p = p0 + lane;
        const int nk = p < N ? io.patch_nkept[e * N + p] : 0;
        int inc = nk;
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += v;
        }
        const int64_t base = e * io.stride + run + inc - nk;
        for (int k = 0; k < nk; ++k) {
            const int64_t src = ((int64_t)e * N + p) * K + k, r = base + k;
            io.body_a[r] = 0;
            io.body_b[r] = 1;
            for (int q = 0; q < 3; ++q) {
                io.point[3 * r + q] = io.kept_point[3 * src + q];
                io.normal[3 * r + q] = io.kept_normal[3 * src + q];
            }
            io.depth[r] = io.kept_depth[src];
            io.mu[r] = mu;
            io.restitution[r] = rest;
            io.slop[r] = slop;
        }
        run += __shfl_sync(0xffffffffu, inc, 31);
    }
}

}  // namespace

void launch_constraints_build(int64_t n_sys, int nb, const SysRows &rows, const BuildIO &io, cudaStream_t s) {
    if (n_sys <= 0) return;
    const int64_t threads = n_sys * 32;
    k_constraints_build<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(n_sys, nb, rows, io);
}

void launch_sweeps(int64_t n_sys, int nb, const SysRows &rows, const SweepIO &io, const SweepPhase *phases,
                   int n_phases, cudaStream_t s) {
    if (n_sys <= 0 || n_phases <= 0) return;
    const size_t smem = (size_t)2 * 6 * nb * SW_T * sizeof(double);
    k_sweeps<<<(unsigned)((n_sys + SW_T - 1) / SW_T), SW_T, smem, s>>>(n_sys, nb, rows, io, phases[0],
                                                                       n_phases > 1 ? phases[1] : phases[0], n_phases);
}

void launch_body_wrenches(int64_t n_sys, int nb, const SysRows &rows, const WrenchIO &io, cudaStream_t s) {
    if (n_sys <= 0) return;
    const size_t smem = (size_t)6 * nb * SW_T * sizeof(double);
    k_body_wrenches<<<(unsigned)((n_sys + SW_T - 1) / SW_T), SW_T, smem, s>>>(n_sys, nb, rows, io);
}

void launch_plan_rows(int64_t E, const PlanRowsIO &io, cudaStream_t s) {
    if (E <= 0) return;
    k_plan_rows<<<(unsigned)((E * 32 + 255) / 256), 256, 0, s>>>(E, io);
}

}  // namespace cs
