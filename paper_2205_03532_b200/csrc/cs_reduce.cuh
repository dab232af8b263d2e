#pragma once
#include "cs_generate.cuh"

namespace cs {

constexpr int REDUCE_BLOCK = 256;
constexpr int FINALIZE_BLOCK = 128;
constexpr int FINALIZE_SMEM_POINTS = 512;  // patches up to this many members are staged in shared memory
constexpr int MAX_KEPT = 64;               // per_patch_cap limit of the GPU path
constexpr double MERGE_COS = 0.9961946980917455;  // float(np.cos(np.radians(5.0))) (reduction.py:25)

struct ReduceParams {
    int N, K, batch_size, has_min_depth;
    double cone, min_depth;
};

struct ReduceIO {
    int64_t E;
    const int64_t *cand_base;
    int32_t *n_cand;
    const double *env_min_depth;  // [E] or null: per-env cull (Scene passes -cd, scene.py:219-223)
    const double *point, *normal, *depth;
    const int32_t *face;
    // workspace (rows indexed like candidates)
    int32_t *order, *label;
    double *su, *sv;   // sort keys
    int32_t *sp;       // sort payload
    int32_t *sh;       // hull/stack scratch: env e uses [2 cand_base(e) + e (4N + 4), + 2 cap_e + 4N + 4)
    // finalisation scratch (cs_finalize.cu); rows like candidates unless stated
    double2 *suv;        // sorted (u, v) of every patch's members (rows), with sp the member (~k: not touching)
    double2 *tuv;        // the touching members' sorted (u, v), compacted (rows) ...
    int32_t *tpos;       // ... and their positions in the sorted rows
    double *tu, *tv;     // second sort buffer of patches too large for shared memory
    double *fw;          // member weights of k_fin_fold_large's patches above FL_W (it runs beside the sort)
    int32_t *tk;
    int32_t *hj;         // [4 rows] chain stacks: sorted positions (the hull output) ...
    double *hu, *hv;     // ... and their (u, v) (backing store of the shared-memory window)
    int32_t *hlen;       // [E N 4] chain lengths per patch and job
    int32_t *pdeep;      // [E N] per patch (work index): deepest member position
    int32_t *pnt;        // [E N] touching members (depth >= 0)
    int32_t *wenv;       // [E N] env of each work index
    int32_t *jobs;       // [64][4 E N] chain jobs (4 w + kind) bucketed by chain length
    int32_t *njob;       // [65] per-bucket counts, claimed
    int32_t *patch_off;  // [E+1]
    int32_t *red_slow;   // [E] k_reduce_fast left env e to k_reduce (NaN, min_depth cull, eviction)
    int32_t *large_list, *large_count;  // patches above the warp path's size limit
    // outputs
    int32_t *n_patch, *n_kept;
    double *patch_normal, *builder_maxd;
    int32_t *member_offsets, *members;
    int32_t *patch_nkept, *kept_cand, *kept_face;
    double *kept_point, *kept_normal, *kept_depth;
    double *w_sum, *wp_sum, *wn_sum, *wt_sum, *area, *max_depth;
    float *stats;
};

void launch_reduce(const ReduceIO &io, const ReduceParams &p, int64_t max_batch, cudaStream_t s);
size_t reduce_smem_bytes(int N, int SB);  // k_reduce dynamic shared memory per env
// Side streams and events of a plan: launch_finalize forks its independent kernels
// onto them (concurrent graph branches when the collide is captured).
struct FinFork {
    cudaStream_t s_block, s_fold;
    cudaEvent_t ev_fork, ev_block, ev_fold;
};
void launch_finalize(const ReduceIO &io, const ReduceParams &p, int sm_count, cudaStream_t s,
                     const FinFork *fk = nullptr);

}  // namespace cs
