#pragma once
// Contact solver: the consumer of the reduced contacts.
//   ContactConstraints.build     dynamics/solver.py:105-141
//   gauss_seidel_sweeps          dynamics/_kernels.py:52-115
//   body_wrenches                dynamics/solver.py:154-163
// Batched over independent systems. System s owns the rows [begin(s), end(s)) in
// sweep order and the bodies [s nb, (s + 1) nb) of the state arrays; row body ids
// are local to the system.
#include "cs_common.cuh"

namespace cs {

// Systems up to SOLVER_SMEM_BODIES bodies keep the 6x6 mobility blocks and the body
// state on chip (registers / shared memory); larger ones (MODE 1 of the sweeps) read
// and update them in global memory. The reference has no limit; the bound below
// only keeps the element indices in 32 bits.
constexpr int SOLVER_SMEM_BODIES = 8;
constexpr int SOLVER_MAX_BODIES = 1 << 20;

struct SysRows {
    const int64_t *off;    // [S + 1] CSR offsets (the reference's layout: rows of a system
                           // contiguous, 3-vectors as (row, 3)); or null: the interleaved
                           // layout of plan rows, where ...
    int64_t stride;        // ... every system has `stride` row slots and count[s] rows, ...
    const int32_t *count;
    int64_t planes;        // ... slot j of system s is element ((s / 32 * stride + j) * 32 + s % 32)
                           // of each field, 3-vectors as 3 planes of `planes` elements: one
                           // system per lane reads a row of 32 systems as one coalesced line
    __device__ __forceinline__ int64_t n(int64_t s) const { return off ? off[s + 1] - off[s] : count[s]; }
    __device__ __forceinline__ int64_t row(int64_t s, int64_t j) const {
        return off ? off[s] + j : (((s >> 5) * stride + j) << 5) + (s & 31);
    }
    __device__ __forceinline__ int64_t vec(int64_t r, int q) const { return planes ? r + q * planes : 3 * r + q; }
};

struct BuildIO {
    const int64_t *body_a, *body_b;
    const double *point, *normal, *depth, *restitution, *slop;
    const double *ref, *w_mat, *vel;  // state [S nb (3 | 36 | 6)]
    double h, bias_factor;
    double *ra, *rb, *tan1, *tan2, *kn, *kt1, *kt2, *bias_target, *restitution_target;
};

// One sweep phase: `iters` in-order sweeps toward `target` accumulating into lam_n
// (position phase: bias targets with friction; velocity phase: restitution targets).
struct SweepPhase {
    int64_t iters;
    const double *target;
    double *lam_n;
    int with_friction;
};

struct SweepIO {
    const int64_t *body_a, *body_b;
    const double *ra, *rb, *nrm, *tan1, *tan2, *kn, *kt1, *kt2, *mu;
    double *lam_t1, *lam_t2;
    const double *w_mat;
    double *vel, *imp;  // [S nb 6] in/out
};

struct WrenchIO {
    const int64_t *body_a, *body_b;
    const double *ra, *rb, *nrm, *tan1, *tan2, *lam_n, *lam_vel, *lam_t1, *lam_t2;
    double h;
    double *out;  // [S nb 6], overwritten
};

void launch_constraints_build(int64_t n_sys, int nb, const SysRows &rows, const BuildIO &io, cudaStream_t s);
// fixed_bodies: every row has body_a = 0, body_b = 1 (plan rows)
void launch_sweeps(int64_t n_sys, int nb, const SysRows &rows, const SweepIO &io, const SweepPhase *phases,
                   int n_phases, cudaStream_t s, bool fixed_bodies = false);
// Interleaved plan rows only: packs the sweep fields of every row (phase 0's and
// phase 1's targets included) into `packed` [n_sys * stride * 22] and sweeps from
// the records with bulk copies.
void launch_sweeps_packed(int64_t n_sys, int nb, const SysRows &rows, const SweepIO &io, const SweepPhase *phases,
                          int n_phases, double *packed, cudaStream_t s, bool fixed_bodies = false);
void launch_body_wrenches(int64_t n_sys, int nb, const SysRows &rows, const WrenchIO &io, cudaStream_t s);

// Plan rows: system s's rows are the kept contacts of its pair slots (plan envs)
// [slot_off[s], slot_off[s + 1]) (one slot e = s when slot_off is null), slot by
// slot, each in (patch slot, k) order (scene.py:228-243), with body_a / body_b the
// slot's SDF / mesh body within the system (0 / 1 when null), in the interleaved
// layout of `rows`. count_out (optional) receives each system's row count.
struct PlanRowsIO {
    const int32_t *patch_nkept, *n_patch;                 // [E N], [E]
    const double *kept_point, *kept_normal, *kept_depth;  // [E N K (3)]
    const double *env_mu, *env_restitution, *env_slop;    // [E] per pair slot
    const int64_t *slot_off, *slot_a, *slot_b;            // [S + 1], [E], [E] or null
    int32_t N, K;
    SysRows rows;
    int32_t *count_out;
    int64_t *body_a, *body_b;
    double *point, *normal, *depth, *mu, *restitution, *slop;
};
void launch_plan_rows(int64_t E, const PlanRowsIO &io, cudaStream_t s);

}  // namespace cs
