#pragma once
#include "cs_common.cuh"

namespace cs {

constexpr int FACE_BLOCK = 128;
constexpr int COMPACT_BLOCK = 256;
constexpr int MAX_MINIMIZE_ITERS = 12;  // generation.py:19

// Per-face staging. k_faces block b covers faces [f0, f0 + FACE_BLOCK) of one env
// and writes its found faces, compacted, to rows cand_base[e] + f0 + [0, count).
struct Staging {
    double *point;         // [row,3] grid frame
    double *phi;
    double *grad;          // [row,3] unnormalised
    int32_t *face;         // [row]
    int32_t *chunk_count;  // [nblocks] found faces per k_faces block
    int32_t *chunk_off;    // [nblocks] candidate offset of the block's first found face
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
                   int32_t *env_status, double *env_min_depth, cudaStream_t s);
void launch_faces(int64_t nblocks, const int2 *block_map, const EnvXf *xf, const SdfDesc *sdfs,
                  const MeshDesc *meshes, const int64_t *cand_base, const Staging &st, unsigned long long *counter,
                  const GridT<double> *uniform, cudaStream_t s);
void launch_compact(int64_t E, const EnvXf *xf, const int64_t *cand_base, const int2 *block_map,
                    const int32_t *chunk_first, const Staging &st, const Candidates &cs, int32_t *n_cand,
                    cudaStream_t s);
void launch_face_contacts(const GridView &g, const double *tv, int64_t m, double cd, int max_iters, double tol,
                          double *op, double *ophi, double *og, uint8_t *ofd, cudaStream_t s);
void launch_sdf_sample(const GridView &g, const double *p, int64_t n, double *out, cudaStream_t s);
void launch_sdf_gradient(const GridView &g, const double *p, int64_t n, double *out, cudaStream_t s);

}  // namespace cs
