"""Per-pair contact generation, drop-in for contactsim.contacts.generation
(/root/reference/pkg/src/contactsim/contacts/generation.py).

`generate_contacts` keeps the reference's signature, validation and return
type; the work (grid-frame transform, AABB cull, per-face projected-gradient
SDF minimisation, compaction, world-frame epilogue) runs in the sm_100a kernels
k_env_xf / k_faces / k_compact through a one-env plan. `face_contacts` is the
drop-in for the reference's numba kernel (contacts/_kernels.py:11), over CUDA
tensors.
"""

from __future__ import annotations

import logging
from dataclasses import dataclass

import numpy as np

from .. import _native
from ..errors import NonFiniteStateError
from ..geometry.mesh import TriMesh
from ..math3d import Transform
from ..sdf.grid import SignedDistanceGrid
from .types import CollisionPairing, ContactSet

log = logging.getLogger(__name__)

MAX_MINIMIZE_ITERS = 12
CONVERGENCE_TOL_VOXELS = 0.1


@dataclass(frozen=True)
class BodyShape:
    body_id: int
    triangle_count: int
    sdf_enabled: bool


def assign_roles(body_a: BodyShape, body_b: BodyShape) -> CollisionPairing:
    """Which body is sampled as the SDF (generation.py:32-51): the one that opted
    in; if both or neither did, the one with more triangles, ties to the lower id."""
    if body_a.sdf_enabled != body_b.sdf_enabled:
        sdf, mesh = (body_a, body_b) if body_a.sdf_enabled else (body_b, body_a)
    elif body_a.triangle_count != body_b.triangle_count:
        sdf, mesh = (body_a, body_b) if body_a.triangle_count > body_b.triangle_count else (body_b, body_a)
    else:
        sdf, mesh = (body_a, body_b) if body_a.body_id < body_b.body_id else (body_b, body_a)
    return CollisionPairing(sdf.body_id, mesh.body_id, not (body_a.sdf_enabled or body_b.sdf_enabled))


def _gen_plans():
    global _GEN_PLANS
    if _GEN_PLANS is None:
        from ..collide import PlanCache

        _GEN_PLANS = PlanCache(maxsize=8)
    return _GEN_PLANS


_GEN_PLANS = None


def _plan_for(sdf_handle: int, mesh_handle: int):
    """One-env generate plan per (thread, grid, mesh): bounded LRU, dropped when the
    grid or mesh is finalised (collide.PlanCache)."""
    from ..collide import Plan

    return _gen_plans().get((sdf_handle, mesh_handle),
                            lambda: Plan([sdf_handle], [mesh_handle], None, stages=_native.CS_STAGE_GENERATE),
                            (sdf_handle,), (mesh_handle,))


def generate_contacts(pairing: CollisionPairing, grid: SignedDistanceGrid, mesh: TriMesh, sdf_pose: Transform,
                      mesh_pose: Transform, contact_distance: float) -> ContactSet:
    """At most one contact per mesh face whose SDF minimum is within
    contact_distance; depth = -phi, normal = normalised SDF gradient in world."""
    import torch

    from ..collide import register_mesh

    if contact_distance < 0.0:
        raise ValueError("contact_distance must be non-negative")
    for pose in (sdf_pose, mesh_pose):
        if not (np.all(np.isfinite(pose.rotation)) and np.all(np.isfinite(pose.translation))):
            raise NonFiniteStateError("non-finite pose in contact generation")
    plan = _plan_for(grid.device_handle(), register_mesh(mesh))
    poses = torch.from_numpy(np.stack([sdf_pose.pose12(), mesh_pose.pose12()])).cuda()
    cd = torch.tensor([float(contact_distance)], dtype=torch.float64, device="cuda")
    plan.collide(poses[0:1].contiguous(), poses[1:2].contiguous(), cd, _native.CS_POSE12)
    n = int(_native.fetch(plan.n_cand[0:1])[0][0])
    if n == 0:
        return ContactSet.empty(pairing.sdf_body, pairing.mesh_body)
    pt, nr, dp, fc = _native.fetch(plan.cand_point[:n], plan.cand_normal[:n], plan.cand_depth[:n], plan.cand_face[:n])
    return ContactSet(pt, nr, dp, fc.astype(np.int64), pairing.sdf_body, pairing.mesh_body)


def face_contacts(values, nx, ny, nz, ox, oy, oz, voxel, tri_verts, contact_distance, max_iters, tol, out_point,
                  out_phi, out_grad, out_found, stream=None) -> None:
    """The numba kernel's argument list (contacts/_kernels.py:12-17) over CUDA
    tensors: values float32, tri_verts (m,3,3) float64, caller-allocated outputs
    (out_found uint8). Pruned faces only get out_found = 0."""
    m = int(tri_verts.shape[0])
    _native.call("cs_face_contacts", values.data_ptr(), int(nx), int(ny), int(nz), float(ox), float(oy), float(oz),
                 float(voxel), tri_verts.data_ptr(), m, float(contact_distance), int(max_iters), float(tol),
                 out_point.data_ptr(), out_phi.data_ptr(), out_grad.data_ptr(), out_found.data_ptr(),
                 _native.stream_handle(stream))
