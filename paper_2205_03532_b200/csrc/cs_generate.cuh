#pragma once
#include "cs_common.cuh"

namespace cs {

// register budgets / grids of the descent wavefront (measured best, round 1); plans with
// per-env grids (UNIFORM false) take one CTA per SM less: no spills (config 3: 1% faster)
#ifndef FIRST_MINB
#define FIRST_MINB 4  // 64 registers (spills 128 B; measured: 3 -> descent 1.033 ms, 4 -> 1.008, 2 -> 1.151, 5 -> 1.125)
#endif
#ifndef GRAD_MINB
#define GRAD_MINB 4  // 64 registers (with the stage-0 corner test: 4 -> descent 0.941 ms, 5 -> 1.008; without it 5 was best)
#endif
#ifndef GRAD_MINB_NU
#define GRAD_MINB_NU (GRAD_MINB - 1)  // plans with per-env grids (config 3: 2 -> 7.81 ms, 3 -> 7.42, 4 -> 7.59)
#endif
#ifndef REST_MINB
#define REST_MINB 6  // measured: 4 -> 1.033 ms (with FIRST_MINB 3), 6 -> 1.020, 3 -> 1.038, 8 -> worse than 6
#endif
#ifndef WAVE_GRID
#define WAVE_GRID 32  // CTAs per SM of the grad / first wave kernels (grid-stride loops): measured best
                      // (8: +0.05 ms, 64: +0.02 ms; many small CTAs balance the tail)
#endif
#ifndef REST_GRID
#define REST_GRID 8
#endif
#ifndef PREP_MINB
#define PREP_MINB 6  // 40 registers (re-measured in round 2: 4 -> prep 0.979 ms, 5 -> 0.874, 6 -> 0.870)
#endif
constexpr int PGD_GRAB = 64;  // work items a warp claims per atomic
#ifndef COMPACT_BLOCK_DEF
#define COMPACT_BLOCK_DEF 256
#endif
#ifndef COMPACT_MINB
#define COMPACT_MINB 3  // 85 registers (measured: 1 -> 0.178 ms, 2 -> 0.179, 3 -> 0.169, 4 -> 0.197)
#endif
constexpr int COMPACT_BLOCK = COMPACT_BLOCK_DEF;
constexpr int MAX_MINIMIZE_ITERS = 12;  // generation.py:19

// One face that survived the cull and the Lipschitz prune (k_face_prep), waiting
// for its projected-gradient descent (the k_pgd_* wavefront).
struct FaceWork {
    int32_t row;        // staging row: cand_base[e] + f0 + rank among the chunk's survivors (< 2^31)
    int32_t blk;        // k_face_prep block (env, chunk)
    int32_t face;       // face index | start corner << 30 (0 centroid, 1..3 = a, b, c)
    int32_t env;        // the block's env (saves the descent a dependent block_map lookup)
    double phi[4];      // phi at a, b, c and at the start point
};
static_assert(sizeof(FaceWork) == 48, "FaceWork is three 16-byte words");

// Per-face staging. k_face_prep block b covers faces [f0, f0 + FACE_CHUNK) of one
// env; its survivors own rows cand_base[e] + f0 + [0, chunk_count[b]) in face order.
struct Staging {
    double *point;         // [row,3] grid frame
    double *phi;
    double *grad;          // [row,3] unnormalised
    int32_t *face;         // [row] face index if found, else -1
    int32_t *chunk_count;  // [nblocks] survivors per block
    int32_t *chunk_found;  // [nblocks] found faces per block
    int32_t *chunk_off;    // [nblocks] candidate offset of the block's first found face
    FaceWork *work;        // [capacity] survivors, dense
    double *alpha;         // [row] descent step of a moved face
    uint32_t *acc;         // [capacity] work indices moved by k_pgd_first (| ACC_FINAL)
    int4 *acc_hd;          // [capacity] ... and their work-record headers (row, blk, face, env)
    uint32_t *slow;        // [capacity] work indices still moving after iteration 0
    unsigned *work_count;  // [0] survivors, [1] left to k_pgd_first by stage 0 (listed in slow), [2] accepted, [3] slow
};

// Candidate arrays (row = cand_base[e] + candidate index).
struct Candidates {
    double *point;
    double *normal;
    double *depth;
    int32_t *face;
};

void launch_env_xf(int64_t E, const int32_t *env_sdf, const int32_t *env_mesh, const SdfDesc *sdfs,
                   const double *sdf_pose, const double *mesh_pose, int pose_format, const double *cd, EnvXf *xf,
                   int32_t *env_status, double *env_min_depth, unsigned *work_count, cudaStream_t s,
                   const int32_t *active = nullptr);
void launch_face_prep(int64_t nblocks, const int4 *block_map, const EnvXf *xf, const SdfDesc *sdfs,
                      const MeshDesc *meshes, const int64_t *cand_base, const Staging &st, int max_chunk_verts,
                      unsigned long long *counter, const PlanGrid *uniform, cudaStream_t s,
                      const MeshDesc *umesh = nullptr);
void launch_pgd_wave(int sm_count, const int2 *block_map, const EnvXf *xf, const SdfDesc *sdfs, const MeshDesc *meshes,
                     const Staging &st, unsigned long long *counter, const PlanGrid *uniform, cudaStream_t s,
                     const MeshDesc *umesh = nullptr);
size_t face_prep_smem(int max_chunk_verts);
void launch_compact(int64_t E, const EnvXf *xf, const int64_t *cand_base, const int2 *block_map,
                    const int32_t *chunk_first, const Staging &st, const Candidates &cs, int32_t *n_cand,
                    cudaStream_t s);
void build_cell_windows(const float *values, int nx, int ny, int nz, float *tables, float *tmp, cudaStream_t s);
// brick minima bm [bx by bz], the 8 brick-window tables bw [8][bx by bz], and the grid
// scan (scan[0]: a value is not finite; scan[1]: max |value| as float bits)
void build_brick_windows(const float *values, int nx, int ny, int nz, int bx, int by, int bz, float *bm, float *bw,
                         unsigned *scan, cudaStream_t s);
void launch_face_contacts(const GridView &g, const double *tv, int64_t m, double cd, int max_iters, double tol,
                          double *op, double *ophi, double *og, uint8_t *ofd, cudaStream_t s);
void launch_sdf_sample(const GridView &g, const double *p, int64_t n, double *out, cudaStream_t s);
void launch_sdf_gradient(const GridView &g, const double *p, int64_t n, double *out, cudaStream_t s);

}  // namespace cs
