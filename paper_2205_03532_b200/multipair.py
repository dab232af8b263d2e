"""Multi-pair scenes on the device.

The batched form of Scene._collect_contacts (contactsim/dynamics/scene.py:170-227)
for many independent multi-body scenes: world AABBs (RigidBody.world_aabb,
dynamics/body.py:77-83), the broadphase (geometry/broadphase.py:25), the pair
filter (exclusions, two fixed bodies: scene.py:189-196), role assignment
(assign_roles, contacts/generation.py:32-51) and, for every pair the broadphase
reports, generate_contacts + reduce_contacts with the pair's own contact distance
(2 voxel of its SDF body's grid, scene.py:206). Everything after construction
runs on the GPU without host round trips:

    cs_world_aabb -> cs_broadphase -> cs_pair_slots_active -> cs_collide_active

A plan is built once over every candidate pair slot (pairs that pass the filter);
each step activates the slots whose pair the broadphase reports, in the
reference's pair order (sorted by body id).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native
from .collide import Plan, ReducedContacts
from .contacts.generation import BodyShape, assign_roles
from .contacts.types import ReductionParams
from .geometry.broadphase import MAX_BODIES


@dataclass
class SceneBody:
    """One body of a scene: its id (unique in the scene), registered mesh handle,
    optional registered SDF handle (+ the grid's voxel size), the mesh AABB, the
    triangle count and sdf_enabled flag that assign_roles reads, and whether it is
    fixed (static or chain-driven: pairs of two fixed bodies are skipped)."""

    body_id: int
    mesh_handle: int
    mesh_aabb: tuple
    triangle_count: int
    sdf_handle: int | None = None
    voxel: float | None = None
    sdf_enabled: bool = False
    fixed: bool = False
    friction: float = 0.5      # RigidBody defaults (dynamics/body.py:27-28)
    restitution: float = 0.0


class MultiPairScenes:
    def __init__(self, scenes: list[list[SceneBody]], params: ReductionParams | None = None,
                 exclusions: list[set] | None = None, contact_distance: float | None = None):
        import torch

        self.scenes = scenes
        S = len(scenes)
        body_off = np.zeros(S + 1, np.int64)
        for s, bodies in enumerate(scenes):
            if len(bodies) > MAX_BODIES:
                raise ValueError(f"scene {s}: at most {MAX_BODIES} bodies")
            ids = [b.body_id for b in bodies]
            if len(set(ids)) != len(ids):
                raise ValueError(f"scene {s}: body ids must be unique")
            body_off[s + 1] = body_off[s] + len(bodies)
        self.body_off = body_off
        flat = [b for bodies in scenes for b in bodies]
        self.n_bodies = len(flat)
        # broadphase margin per scene (scene.py:181-185)
        margins = []
        for bodies in scenes:
            mv = max((b.voxel for b in bodies if b.sdf_handle is not None and b.voxel), default=0.0)
            margins.append(contact_distance or 2.0 * mv or 1e-3)
        # candidate pair slots, in the reference's pair order
        slot_scene, slot_pair, sdf_idx, mesh_idx, sdf_h, mesh_h, cd = [], [], [], [], [], [], []
        slot_a, slot_b, slot_mu, slot_e, slot_voxel = [], [], [], [], []
        for s, bodies in enumerate(scenes):
            by_id = {b.body_id: (k, b) for k, b in enumerate(bodies)}
            order = sorted(by_id)
            excl = exclusions[s] if exclusions else set()
            for x in range(len(order)):
                for y in range(x + 1, len(order)):
                    ia, ib = order[x], order[y]
                    (ka, a), (kb, b) = by_id[ia], by_id[ib]
                    if frozenset((ia, ib)) in excl or (a.fixed and b.fixed):
                        continue
                    pr = assign_roles(BodyShape(ia, a.triangle_count, a.sdf_enabled),
                                      BodyShape(ib, b.triangle_count, b.sdf_enabled))
                    ks, sb = by_id[pr.sdf_body]
                    km, mb = by_id[pr.mesh_body]
                    if sb.sdf_handle is None:
                        raise ValueError(f"scene {s}: body {sb.body_id} is the SDF body of pair ({ia}, {ib}) "
                                         "but has no registered grid")
                    slot_scene.append(s)
                    slot_pair.append((ia, ib))
                    sdf_idx.append(body_off[s] + ks)
                    mesh_idx.append(body_off[s] + km)
                    sdf_h.append(sb.sdf_handle)
                    mesh_h.append(mb.mesh_handle)
                    cd.append(contact_distance or 2.0 * sb.voxel)
                    # solver rows of this pair (scene.py:224-243): body_a = SDF body
                    slot_a.append(ks)
                    slot_b.append(km)
                    slot_mu.append(float(np.sqrt(sb.friction * mb.friction)))
                    slot_e.append(max(sb.restitution, mb.restitution))
                    slot_voxel.append(sb.voxel)
        self.n_slots = len(slot_scene)
        if self.n_slots == 0:
            raise ValueError("no candidate pairs")
        self.slot_scene = np.array(slot_scene, np.int64)
        self.slot_pair = np.array(slot_pair, np.int64).reshape(-1, 2)
        self.slot_sdf_body = np.array([flat[i].body_id for i in sdf_idx], np.int64)
        self.slot_mesh_body = np.array([flat[i].body_id for i in mesh_idx], np.int64)
        self.plan = Plan(sdf_h, mesh_h, params or ReductionParams())
        dev = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to(dt).cuda()  # noqa: E731
        self.d_body_off = dev(body_off, torch.int64)
        self.d_ids = dev(np.array([b.body_id for b in flat], np.int64), torch.int64)
        self.d_mesh_lo = dev(np.array([np.asarray(b.mesh_aabb[0], np.float64) for b in flat]), torch.float64)
        self.d_mesh_hi = dev(np.array([np.asarray(b.mesh_aabb[1], np.float64) for b in flat]), torch.float64)
        self.d_margin = dev(np.array(margins, np.float64), torch.float64)
        n = np.diff(body_off)
        self.pair_off_h = np.concatenate([[0], np.cumsum(n * (n - 1) // 2)]).astype(np.int64)
        self.d_pair_off = dev(self.pair_off_h, torch.int64)
        self.pairs = torch.zeros((max(int(self.pair_off_h[-1]), 1), 2), dtype=torch.int64, device="cuda")
        self.n_pairs = torch.zeros(S, dtype=torch.int32, device="cuda")
        self.bp_status = torch.zeros(S, dtype=torch.int32, device="cuda")
        self.d_slot_scene = dev(self.slot_scene, torch.int64)
        self.d_slot_pair = dev(self.slot_pair, torch.int64)
        self.d_sdf_idx = dev(np.array(sdf_idx, np.int64), torch.int64)
        self.d_mesh_idx = dev(np.array(mesh_idx, np.int64), torch.int64)
        self.d_cd = dev(np.array(cd, np.float64), torch.float64)
        self.active = torch.zeros(self.n_slots, dtype=torch.int32, device="cuda")
        # solver: scenes' slots are contiguous, in pair order
        slot_off = np.searchsorted(self.slot_scene, np.arange(S + 1)).astype(np.int64)
        self.max_slots = int(np.diff(slot_off).max())
        self.max_bodies = int(np.diff(body_off).max())
        self.d_slot_off = dev(slot_off, torch.int64)
        self.d_slot_a = dev(np.array(slot_a, np.int64), torch.int64)
        self.d_slot_b = dev(np.array(slot_b, np.int64), torch.int64)
        self.d_slot_mu = dev(np.array(slot_mu, np.float64), torch.float64)
        self.d_slot_e = dev(np.array(slot_e, np.float64), torch.float64)
        self.slot_voxel = np.array(slot_voxel, np.float64)
        self.world_lo = torch.zeros((self.n_bodies, 3), dtype=torch.float64, device="cuda")
        self.world_hi = torch.zeros_like(self.world_lo)

    def step(self, poses7, stream=None, check: bool = True) -> ReducedContacts:
        """One contact step for every scene: poses7 (B,7) float64 per body, scenes'
        bodies concatenated in order. Slot t of the result holds pair
        slot_pair[t] of scene slot_scene[t] (SDF body slot_sdf_body[t]); inactive
        slots (active[t] == 0) have no candidates."""
        import torch

        p = poses7 if isinstance(poses7, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(poses7))
        p = p.to(device="cuda", dtype=torch.float64).contiguous().reshape(self.n_bodies, 7)
        sp = p.index_select(0, self.d_sdf_idx).contiguous()
        mp = p.index_select(0, self.d_mesh_idx).contiguous()
        _native.hand_to_stream(stream, p, sp, mp)  # staged on the current stream, read on `stream`
        st = _native.stream_handle(stream)
        _native.call("cs_world_aabb", self.n_bodies, self.d_mesh_lo.data_ptr(), self.d_mesh_hi.data_ptr(),
                     p.data_ptr(), self.world_lo.data_ptr(), self.world_hi.data_ptr(), st)
        _native.call("cs_broadphase", len(self.scenes), self.d_body_off.data_ptr(), self.world_lo.data_ptr(),
                     self.world_hi.data_ptr(), self.d_ids.data_ptr(), self.d_margin.data_ptr(),
                     self.d_pair_off.data_ptr(), self.pairs.data_ptr(), self.n_pairs.data_ptr(),
                     self.bp_status.data_ptr(), st)
        _native.call("cs_pair_slots_active", self.n_slots, self.d_slot_scene.data_ptr(), self.d_slot_pair.data_ptr(),
                     self.d_pair_off.data_ptr(), self.pairs.data_ptr(), self.n_pairs.data_ptr(),
                     self.active.data_ptr(), st)
        _native.call("cs_collide_active", self.plan.ptr, sp.data_ptr(), mp.data_ptr(), _native.CS_POSE7,
                     self.d_cd.data_ptr(), self.active.data_ptr(), st)
        res = ReducedContacts(self.plan, stream=stream)
        if check:
            _native.sync_stream(stream)
            bs = self.bp_status.cpu().numpy()
            if (bs == 1).any():
                raise ValueError("non-finite AABB in broadphase input")
            res.check()
        return res

    def solve(self, state, params=None, wrench=None, stream=None):
        """The contact solve of one substep (Scene._substep, scene.py:130-160) for
        every scene on the last step's reduced contacts: system s = scene s, its
        rows the active pairs' kept contacts in pair order with body_a the pair's
        SDF body, mu = sqrt(f_a f_b), e = max(e_a, e_b), slop = penetration_slop or
        0.5 voxel of the pair's grid (scene.py:207-212,226-227).
        state: dynamics.BatchedSolverState(n_scenes, max bodies per scene), bodies
        in scene order (vel, impulse updated in place). Returns wrenches (S, nb, 6)."""
        import torch

        from .dynamics.solver import SolverParams

        params = params or SolverParams()
        S, nb = len(self.scenes), state.vel.shape[1]
        if state.vel.shape[0] != S or nb < self.max_bodies:
            raise ValueError("state must hold (n_scenes, >= bodies per scene) systems")
        from .dynamics.solver import check_solver_bodies

        check_solver_bodies(nb)
        slop = np.full(self.n_slots, params.penetration_slop) if params.penetration_slop is not None \
            else 0.5 * self.slot_voxel
        d_slop = torch.from_numpy(slop.astype(np.float64)).cuda()
        if wrench is None:
            wrench = torch.empty((S, nb, 6), dtype=torch.float64, device="cuda")
        cp = params.to_c()
        _native.hand_to_stream(stream, d_slop, wrench)
        _native.call("cs_multipair_solve", self.plan.ptr, S, nb, self.d_slot_off.data_ptr(), self.d_slot_a.data_ptr(),
                     self.d_slot_b.data_ptr(), self.max_slots, state.ref.data_ptr(), state.w_mat.data_ptr(),
                     state.vel.data_ptr(), state.impulse.data_ptr(), self.d_slot_mu.data_ptr(),
                     self.d_slot_e.data_ptr(), d_slop.data_ptr(), ctypes.byref(cp), wrench.data_ptr(),
                     _native.stream_handle(stream))
        return wrench

    def scene_pairs(self, s: int) -> list[tuple[int, int]]:
        """Scene s's broadphase pairs of the last step (sorted (id_a, id_b))."""
        k = int(self.n_pairs[s].item())
        a = int(self.pair_off_h[s])
        return [tuple(int(x) for x in r) for r in self.pairs[a:a + k].cpu().numpy()]
