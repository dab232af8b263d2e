/*
 * contactsim_b200 — C ABI of the B200-native SDF contact generation + contact
 * reduction path (Factory, arXiv 2205.03532; reference package `contactsim`).
 *
 * Plain pointers and sizes only: no torch or CUDA C++ types. `stream` is a
 * cudaStream_t passed as void* (NULL = legacy default stream). Device pointers
 * are marked [dev], host pointers [host]. Every function returns a cs_status;
 * on failure cs_last_error() holds a thread-local message, and the Python shim
 * (paper_2205_03532_b200/_native.py) raises the reference's exception class:
 *
 *   CS_ERR_VALUE     -> ValueError               (e.g. generation.py:64-65)
 *   CS_ERR_NONFINITE -> NonFiniteStateError       (generation.py:66-68, errors.py:19)
 *   CS_ERR_MESH      -> MeshValidationError       (grid.py:169,189-192, errors.py:8)
 *   CS_ERR_HANDLE / CS_ERR_CUDA / CS_ERR_OOM -> RuntimeError
 *   CS_ERR_IO        -> OSError                  (open() in grid.py:154)
 *
 * Numerics: IEEE double arithmetic in the reference's operation order (numba
 * kernels: no FMA contraction), and the reference's BLAS 3-term dot products
 * reproduced with explicit FMAs, so outputs are bit-identical to the reference
 * on the same inputs.
 */
#ifndef CONTACTSIM_B200_H
#define CONTACTSIM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    CS_OK = 0,
    CS_ERR_VALUE = 1,
    CS_ERR_NONFINITE = 2,
    CS_ERR_MESH = 3,
    CS_ERR_HANDLE = 4,
    CS_ERR_CUDA = 5,
    CS_ERR_OOM = 6,
    CS_ERR_IO = 7
} cs_status;

#define CS_ABI_VERSION 1

/* Thread-local message of the last failing call on this thread. */
const char *cs_last_error(void);
int cs_abi_version(void);
/* SM count, L2 bytes and max persisting-L2 bytes of the current device. */
int cs_device_info(int32_t *sm_count, int64_t *l2_bytes, int64_t *persist_l2_max);

/* Roofline denominator measured on this device (no reference counterpart: bench.py
 * support). Random 32-byte-sector gathers from an L2-resident buffer of `bytes`
 * (mode 0: ld.global.cg, L2 only; 1: __ldg, L1 + L2; 2: tld4 on a 2D layered texture,
 * 16 B per fetch) or a streaming read of a buffer above L2 (mode 3: the HBM read peak);
 * `iters` timed launches after two warm ones. *gbs: achieved GB/s. */
int cs_bench_gather(int32_t mode, int64_t bytes, int32_t iters, double *gbs);

/* ------------------------------------------------------------------------
 * Device-resident SDF store.
 * Replaces holding SignedDistanceGrid.values per call (sdf/grid.py:48-68):
 * the grid is uploaded once and shared by every env that names the handle.
 * values: float32, x-fastest, index = ix + nx*(iy + ny*iz) (grid.py:1-6).
 * values_on_device != 0 means `values` is already a device pointer (copied).
 * ---------------------------------------------------------------------- */
int cs_sdf_register(const float *values, int values_on_device, int32_t nx, int32_t ny, int32_t nz,
                    const double origin[3], double voxel, const double aabb_lo[3], const double aabb_hi[3],
                    int32_t *handle);
/* SignedDistanceGrid.load (sdf/grid.py:151-160) straight into the device store:
 * the CSIMSDF1 header ("<8s3i d 3d 6d") is parsed here and the float32 values are
 * streamed from the file to the device through pinned staging buffers (no host
 * array). Errors: CS_ERR_IO (cannot open), CS_ERR_VALUE (bad magic -> the
 * reference's "not an SDF grid file", short file, bad dims). `info` (optional)
 * receives the grid metadata. */
typedef struct {
    int32_t dims[3];
    double origin[3];
    double voxel;
    double aabb_lo[3], aabb_hi[3];
} cs_sdf_file_info;
int cs_sdf_register_file(const char *path, int32_t *handle, cs_sdf_file_info *info);
/* Freeing a grid (or mesh) that live plans sample defers the release to the
 * destruction of the last such plan; the handle is invalid for new plans at once. */
int cs_sdf_free(int32_t handle);
/* [dev] pointer to the stored values (for the per-pair drop-ins below). */
int cs_sdf_values(int32_t handle, const float **values);
/* Pin the grid in L2 for launches on `stream` (cudaAccessPolicyWindow,
 * hitRatio scaled to the persisting-L2 limit). hit_ratio <= 0 clears it. */
int cs_sdf_l2_persist(int32_t handle, void *stream, float hit_ratio);

/* Mesh store (geometry/mesh.py:16-47): float64 vertices, int32 triangles. */
int cs_mesh_register(const double *vertices, int64_t nv, const int32_t *triangles, int64_t nt, int32_t *handle);
int cs_mesh_free(int32_t handle);

/* ------------------------------------------------------------------------
 * Per-pair drop-ins for the reference's numba kernels (same argument lists).
 * ---------------------------------------------------------------------- */

/* contacts/_kernels.py:11-17 face_contacts(values, nx, ny, nz, ox, oy, oz, voxel,
 * tri_verts, contact_distance, max_iters, tol, out_point, out_phi, out_grad, out_found).
 * tri_verts [dev] (m,3,3) f64 grid frame; outputs [dev], caller-allocated.
 * Pruned faces write only out_found = 0, like the reference. */
int cs_face_contacts(const float *values, int64_t nx, int64_t ny, int64_t nz, double ox, double oy, double oz,
                     double voxel, const double *tri_verts, int64_t m, double contact_distance, int32_t max_iters,
                     double tol, double *out_point, double *out_phi, double *out_grad, uint8_t *out_found,
                     void *stream);

/* sdf/_kernels.py:330-346 sample_batch / gradient_batch: points [dev] (n,3) grid frame. */
int cs_sdf_sample(const float *values, int64_t nx, int64_t ny, int64_t nz, double ox, double oy, double oz,
                  double voxel, const double *points, int64_t n, double *out, void *stream);
int cs_sdf_gradient(const float *values, int64_t nx, int64_t ny, int64_t nz, double ox, double oy, double oz,
                    double voxel, const double *points, int64_t n, double *out, void *stream);

/* ------------------------------------------------------------------------
 * Batched collide: the vectorised body of Scene._collect_contacts
 * (dynamics/scene.py:197-227) over E independent envs, one (SDF, mesh) pair each.
 * A plan fixes the env -> (sdf, mesh) assignment and ReductionParams, owns all
 * device buffers, and runs stream-ordered (CUDA-graph capturable).
 * ---------------------------------------------------------------------- */

/* ReductionParams (contacts/types.py:62-78). */
typedef struct cs_reduction_params {
    int32_t max_patches;    /* N, default 128 */
    int32_t per_patch_cap;  /* K, default 6 */
    int32_t batch_size;     /* default 1024 */
    int32_t has_min_depth;  /* 0: min_depth None */
    double normal_cone_cos; /* default cos(20 deg) */
    double min_depth;
} cs_reduction_params;

/* Pose formats for cs_collide. */
enum { CS_POSE7 = 0 /* (px,py,pz,qw,qx,qy,qz) */, CS_POSE12 = 1 /* (R row-major 9, t 3) */ };

/* What a plan runs. */
enum { CS_STAGE_GENERATE = 1, CS_STAGE_REDUCE = 2, CS_STAGE_ALL = 3 };

/* Device views of a plan's buffers (all [dev]). Env e owns rows
 * [cand_base[e], cand_base[e] + capacity_e) of the candidate/member arrays,
 * where capacity_e = triangle count of its mesh (one candidate per face at most). */
typedef struct cs_outputs {
    int64_t n_envs;
    int32_t max_patches, per_patch_cap;
    int64_t total_capacity;
    const int64_t *cand_base;   /* [E] */
    int32_t *env_status;        /* [E] 0 ok, 1 non-finite pose, 2 cd < 0, 3 inactive (cs_collide_active) */
    int32_t *n_cand;            /* [E] candidates (ContactSet length) */
    int32_t *n_patch;           /* [E] */
    int32_t *n_kept;            /* [E] sum of kept contacts over patches */
    float *stats;               /* [E,4] n_cand, n_patch, n_kept, max kept depth (all-gather payload) */
    double *cand_point;         /* [cap,3] world frame (ContactSet.points) */
    double *cand_normal;        /* [cap,3] */
    double *cand_depth;         /* [cap] */
    int32_t *cand_face;         /* [cap] ascending per env */
    double *patch_normal;       /* [E,N,3] representative normal */
    int32_t *patch_nkept;       /* [E,N] */
    int32_t *kept_cand;         /* [E,N,K] candidate index (within env), -1 pad */
    double *kept_point;         /* [E,N,K,3] */
    double *kept_normal;        /* [E,N,K,3] */
    double *kept_depth;         /* [E,N,K] */
    int32_t *kept_face;         /* [E,N,K] mesh face index, -1 pad */
    double *w_sum;              /* [E,N] */
    double *wp_sum;             /* [E,N,3] */
    double *wn_sum;             /* [E,N,3] */
    double *wt_sum;             /* [E,N,3] */
    double *area;               /* [E,N] */
    double *max_depth;          /* [E,N] */
    int32_t *member_offsets;    /* [E,N+1] CSR into members (relative to cand_base[e]) */
    int32_t *members;           /* [cap] candidate indices, patch-major, ascending within a patch */
    uint32_t *face_work;        /* [4] last step's face-descent workload: faces descended, faces whose
                                 * first iteration was not settled by the stage-0 corner test, faces
                                 * moved by the first iteration, faces still moving after it
                                 * (diagnostics) */
} cs_outputs;

typedef struct cs_plan cs_plan;

/* Generate (+ reduce) plan. sdf_handles / mesh_handles [host] (E).
 * With the reduce stage and has_min_depth == 0 the cull is min_depth = -cd per
 * env, as Scene._collect_contacts builds ReductionParams (scene.py:215-225). */
int cs_plan_create(int64_t n_envs, const int32_t *sdf_handles, const int32_t *mesh_handles,
                   const cs_reduction_params *params, int32_t stages, cs_plan **plan);
/* Reduce-only plan over caller-supplied candidate sets with per-env capacity [host] (E). */
int cs_plan_create_reduce(int64_t n_envs, const int64_t *capacity, const cs_reduction_params *params,
                          cs_plan **plan);
int cs_plan_destroy(cs_plan *plan);
int cs_plan_outputs(cs_plan *plan, cs_outputs *out);
/* Device bytes the plan holds (its buffers, including solver rows once allocated);
 * for sizing env counts per GPU. Not in the reference (its arrays are per call). */
int cs_plan_device_bytes(cs_plan *plan, int64_t *bytes);

/* One collide step: sdf_pose/mesh_pose [dev] (E,7) or (E,12) per pose_format,
 * contact_distance [dev] (E). Stream-ordered; no host synchronisation. */
int cs_collide(cs_plan *plan, const double *sdf_pose, const double *mesh_pose, int32_t pose_format,
               const double *contact_distance, void *stream);

/* Phase timing: with slots > 0 every cs_collide records CUDA events on its
 * stream around its phases into a ring of `slots` steps (0 disables).
 * cs_plan_timing_read writes, per recorded step (oldest first, at most
 * max_steps), CS_TIMING_PHASES floats in ms:
 *   [env_xf, face_prep, face_pgd, compact, reduce, finalize(+stats), total]. */
#define CS_TIMING_EVENTS 7
#define CS_TIMING_PHASES 7
int cs_plan_timing(cs_plan *plan, int32_t slots);
int cs_plan_timing_read(cs_plan *plan, float *ms, int32_t max_steps, int32_t *n_steps);

/* Roofline accounting: enable != 0 zeroes the device counters and switches the
 * plan's face kernels to builds that tally every trilinear SDF sample;
 * enable == 0 synchronises, writes CS_SAMPLE_COUNTERS tallies to count
 * ([0] k_face_prep: vertex + centroid samples, [1] k_face_pgd: descent
 * samples) and switches back. */
#define CS_SAMPLE_COUNTERS 2
int cs_plan_count_samples(cs_plan *plan, int32_t enable, uint64_t *count);

/* Reduce step of a reduce-only plan: the caller has written n_cand and the
 * cand_point/cand_normal/cand_depth/cand_face rows of cs_outputs. */
int cs_reduce(cs_plan *plan, void *stream);

/* Host-buffer end-to-end call (the e2e path): copies poses/cd from host,
 * runs cs_collide, copies stats [E,4] back. Host buffers should be pinned. */
int cs_collide_host(cs_plan *plan, const double *sdf_pose_host, const double *mesh_pose_host, int32_t pose_format,
                    const double *contact_distance_host, float *stats_host, void *stream);

/* ------------------------------------------------------------------------
 * Contact solver, the consumer of the reduced contacts:
 * dynamics/solver.py ContactConstraints.build / body_wrenches and
 * dynamics/_kernels.py gauss_seidel_sweeps, bit-identical to the reference.
 * Batched over n_sys independent systems: system s owns rows
 * [row_off[s], row_off[s+1]) (sweep order; row_off [dev] (n_sys+1) int64) and
 * bodies [s*n_bodies, (s+1)*n_bodies) of the state arrays (ref (.,3),
 * w_mat (.,6,6), vel/imp (.,6)); body_a/body_b hold system-local ids
 * (0 <= id < n_bodies <= 2^20: no limit in the reference; systems above 8
 * bodies keep their state in global memory). All arrays [dev], float64 /
 * int64, C order.
 * With n_sys = 1 and row_off = {0, m} these are the reference's per-scene calls.
 * ---------------------------------------------------------------------- */

/* dynamics/solver.py:105-141 (rows' point/normal/depth/restitution/slop -> constraint rows). */
int cs_constraints_build(int64_t n_sys, int32_t n_bodies, const int64_t *row_off, const int64_t *body_a,
                         const int64_t *body_b, const double *point, const double *normal, const double *depth,
                         const double *restitution, const double *slop, const double *ref, const double *w_mat,
                         const double *vel, double h, double bias_factor, double *ra, double *rb, double *tan1,
                         double *tan2, double *kn, double *kt1, double *kt2, double *bias_target,
                         double *restitution_target, void *stream);

/* dynamics/_kernels.py:52-115 gauss_seidel_sweeps(iters, w_mat, vel, imp, body_a, body_b, ra, rb,
 * nrm, tan1, tan2, kn, kt1, kt2, target_vn, mu, lam_n, lam_t1, lam_t2, with_friction):
 * vel, imp, lam_n, lam_t1, lam_t2 updated in place. */
int cs_gauss_seidel_sweeps(int64_t n_sys, int32_t n_bodies, const int64_t *row_off, int64_t iters,
                           const double *w_mat, double *vel, double *imp, const int64_t *body_a,
                           const int64_t *body_b, const double *ra, const double *rb, const double *nrm,
                           const double *tan1, const double *tan2, const double *kn, const double *kt1,
                           const double *kt2, const double *target_vn, const double *mu, double *lam_n,
                           double *lam_t1, double *lam_t2, int32_t with_friction, void *stream);

/* dynamics/solver.py:154-163 body_wrenches: out (n_sys*n_bodies, 6), overwritten. */
int cs_body_wrenches(int64_t n_sys, int32_t n_bodies, const int64_t *row_off, const int64_t *body_a,
                     const int64_t *body_b, const double *ra, const double *rb, const double *nrm,
                     const double *tan1, const double *tan2, const double *lam_n, const double *lam_vel,
                     const double *lam_t1, const double *lam_t2, double h, double *out, void *stream);

/* SolverParams (dynamics/solver.py:24-43) of one substep: h = dt / substeps. */
typedef struct cs_solver_params {
    double h;
    double bias_factor;    /* default 0.2 */
    int32_t pos_iterations;  /* default 16 */
    int32_t vel_iterations;  /* default 1 */
} cs_solver_params;

/* Device views of a plan's solver rows (valid after the first cs_plan_solve).
 * Env e's rows j = 0 .. n_kept[e]-1 are in Scene order (scene.py:228-243: patch
 * slot, then kept contact), body_a = 0 (the SDF body), body_b = 1 (the mesh body).
 * Layout, interleaved by blocks of 32 envs so one env per lane reads a row of 32
 * envs as one line: row (e, j) is element r = ((e/32)*stride + j)*32 + e%32 of every
 * scalar field; 3-vector fields hold 3 planes of `planes` elements (component q
 * of row r at q*planes + r). */
typedef struct cs_solver_rows {
    int64_t stride;
    int64_t planes;
    int64_t *body_a, *body_b;
    double *point, *normal, *depth, *mu, *restitution, *slop;
    double *ra, *rb, *tan1, *tan2, *kn, *kt1, *kt2, *bias_target, *restitution_target;
    double *lam_n, *lam_vel, *lam_t1, *lam_t2;
} cs_solver_rows;

/* The contact solve of one substep on a plan's last cs_collide, one system per env
 * with two bodies (0 = SDF body, 1 = mesh body): builds the rows, runs
 * pos_iterations sweeps with friction toward the bias targets, then
 * vel_iterations sweeps toward the restitution targets (Scene._substep,
 * scene.py:130-145), and writes the body wrenches. State [dev]: ref (E,2,3),
 * w_mat (E,2,6,6), vel (E,2,6) and imp (E,2,6) in/out; mu, restitution, slop
 * (E) per pair (scene.py:206-212,226-227); wrench (E,2,6) out. Stream-ordered. */
int cs_plan_solve(cs_plan *plan, const double *ref, const double *w_mat, double *vel, double *imp, const double *mu,
                  const double *restitution, const double *slop, const cs_solver_params *params, double *wrench,
                  void *stream);
int cs_plan_solver_rows(cs_plan *plan, cs_solver_rows *rows);

/* The contact solve of one substep for multi-pair scenes (cs_collide_active plans):
 * system s = scene s with n_bodies bodies, owning the pair slots (plan envs)
 * [slot_off[s], slot_off[s+1]) (at most max_slots); its rows are the slots' kept
 * contacts slot by slot in Scene order (scene.py:228-243) with body_a =
 * slot_a[e] (the slot's SDF body) and body_b = slot_b[e] (its mesh body), both
 * local to the scene; inactive slots contribute none. State [dev] per body
 * (S*n_bodies): ref (.,3), w_mat (.,6,6), vel/imp (.,6) in/out; mu, restitution,
 * slop [dev] per slot (E); wrench (S*n_bodies, 6) out. slot_off, slot_a, slot_b
 * [dev] int64. Row views: cs_plan_multipair_rows (stride = max_slots*N*K,
 * counts per system in n_rows). */
int cs_multipair_solve(cs_plan *plan, int64_t n_sys, int32_t n_bodies, const int64_t *slot_off,
                       const int64_t *slot_a, const int64_t *slot_b, int32_t max_slots, const double *ref,
                       const double *w_mat, double *vel, double *imp, const double *mu, const double *restitution,
                       const double *slop, const cs_solver_params *params, double *wrench, void *stream);
int cs_plan_multipair_rows(cs_plan *plan, cs_solver_rows *rows, const int32_t **n_rows);

/* ------------------------------------------------------------------------
 * Broadphase and multi-pair scenes, bit-identical to the
 * reference. All arrays [dev].
 * ---------------------------------------------------------------------- */

/* dynamics/body.py:77-83 RigidBody.world_aabb (no margin) for n bodies: mesh AABBs
 * (n,3) + poses (n,7) (px,py,pz,qw,qx,qy,qz) -> world lo/hi (n,3). */
int cs_world_aabb(int64_t n, const double *mesh_lo, const double *mesh_hi, const double *pose7, double *lo,
                  double *hi, void *stream);

/* geometry/broadphase.py:25-68 broadphase_pairs over n_scenes independent scenes:
 * scene s owns bodies [body_off[s], body_off[s+1]) of lo/hi (.,3) and ids (unique
 * within the scene), inflated by margin[s]. Its pairs (id_a < id_b, sorted) go to
 * rows [pair_off[s], pair_off[s] + n_pairs[s]) of pairs (.,2) int64; the capacity
 * of scene s is pair_off[s+1] - pair_off[s]. status[s]: 0 ok, 1 non-finite box (the
 * reference raises ValueError), 2 capacity exceeded, 3 more than 2048 bodies,
 * 4 duplicate ids. Up to 64 bodies the all-pairs test, above it the sweep-and-prune
 * test, as the reference (they differ only on inverted boxes). */
int cs_broadphase(int64_t n_scenes, const int64_t *body_off, const double *lo, const double *hi, const int64_t *ids,
                  const double *margin, const int64_t *pair_off, int64_t *pairs, int32_t *n_pairs, int32_t *status,
                  void *stream);

/* Pair slots -> active mask: active[t] = (slot_pair[t,0], slot_pair[t,1]) is among
 * the broadphase pairs of scene slot_scene[t] (cs_broadphase output). */
int cs_pair_slots_active(int64_t n_slots, const int64_t *slot_scene, const int64_t *slot_pair,
                         const int64_t *pair_off, const int64_t *pairs, const int32_t *n_pairs, int32_t *active,
                         void *stream);

/* cs_collide with an active mask [dev] (E) int32: envs with active[e] == 0 are
 * skipped (env_status 3, no candidates, no patches; their poses are not
 * validated). A plan over every candidate pair slot of a set of multi-body
 * scenes plus this mask from cs_pair_slots_active runs Scene._collect_contacts'
 * pair loop (scene.py:188-227) for the pairs the broadphase reports. */
int cs_collide_active(cs_plan *plan, const double *sdf_pose, const double *mesh_pose, int32_t pose_format,
                      const double *contact_distance, const int32_t *active, void *stream);

/* ------------------------------------------------------------------------
 * SDF generation (sdf/grid.py:163-239): exact unsigned distance to the mesh
 * and ray-parity sign voting on the GPU, bit-identical to the reference.
 * vertices/triangles [host]; values_out [host] (nx*ny*nz).
 * ---------------------------------------------------------------------- */
int cs_sdf_generate(const double *vertices, int64_t nv, const int32_t *triangles, int64_t nt, int32_t nx, int32_t ny,
                    int32_t nz, const double origin[3], double voxel, float *values_out);

#ifdef __cplusplus
}
#endif

#endif /* CONTACTSIM_B200_H */
