#pragma once
// Broadphase: world AABBs of bodies and the overlapping pairs
// of each scene, batched over independent scenes, bit-identical to the reference
//   RigidBody.world_aabb        dynamics/body.py:77-83
//   broadphase_pairs            geometry/broadphase.py:25-68
// plus the pair-slot mask that turns a scene's pair list into the active envs of a
// collide plan built over every candidate pair slot (cs_collide_active).
#include "cs_common.cuh"

namespace cs {

constexpr int BROAD_MAX_BODIES = 2048;  // bodies per scene (one CTA per scene, ranks in shared memory)
constexpr int BROAD_SWEEP_THRESHOLD = 64;  // broadphase.py:12

struct BroadIO {
    const int64_t *body_off;  // [S + 1] scene s owns bodies [body_off[s], body_off[s + 1])
    const double *lo, *hi;    // [B, 3] boxes (before the margin)
    const int64_t *ids;       // [B] body ids, unique within a scene
    const double *margin;     // [S]
    const int64_t *pair_off;  // [S + 1] pair capacity of scene s: [pair_off[s], pair_off[s + 1])
    int64_t *pairs;           // [cap, 2] (id_a, id_b), id_a < id_b, sorted
    int32_t *n_pairs;         // [S]
    int32_t *status;          // [S] 0 ok, 1 non-finite box, 2 capacity exceeded, 3 too many bodies
};
void launch_world_aabb(int64_t n, const double *mesh_lo, const double *mesh_hi, const double *pose7, double *lo,
                       double *hi, cudaStream_t s);
void launch_broadphase(int64_t n_scenes, const BroadIO &io, cudaStream_t s);
void launch_pair_slots(int64_t n_slots, const int64_t *slot_scene, const int64_t *slot_pair,
                       const int64_t *pair_off, const int64_t *pairs, const int32_t *n_pairs, int32_t *active,
                       cudaStream_t s);

}  // namespace cs
