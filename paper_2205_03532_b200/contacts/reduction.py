"""Per-pair contact reduction, drop-in for contactsim.contacts.reduction
(/root/reference/pkg/src/contactsim/contacts/reduction.py).

`reduce_contacts` runs Algorithm 1 (batched assign / seed / bin / add-patch with
merge and eviction, then kept-contact selection and aggregates) in the sm_100a
kernels k_reduce / k_finalize through a one-env reduce plan and returns the
reference's list[ContactPatch]. The verification helpers
(equivalent_system_check, CSV dumps) are host utilities, as in the reference.
"""

from __future__ import annotations

import numpy as np

from .types import ContactPatch, ContactSet, ReductionParams

MERGE_COS = float(np.cos(np.radians(5.0)))

_RED_PLANS = None


def _plan_for(capacity: int, params: ReductionParams):
    """One-env reduce plan per (thread, capacity class, params): bounded LRU
    (collide.PlanCache), so concurrent callers never share buffers."""
    global _RED_PLANS
    from ..collide import Plan, PlanCache
    from .. import _native

    if _RED_PLANS is None:
        _RED_PLANS = PlanCache(maxsize=8)
    cap = 1 << max(10, int(capacity - 1).bit_length())
    key = (cap, params.max_patches, params.per_patch_cap, params.normal_cone_cos, params.min_depth, params.batch_size)
    return _RED_PLANS.get(key, lambda: Plan(None, None, params, stages=_native.CS_STAGE_REDUCE, capacity=[cap]))


def reduce_contacts(candidates: ContactSet, params: ReductionParams | None = None) -> list[ContactPatch]:
    import torch

    from ..collide import ReducedContacts

    params = params or ReductionParams()
    n = len(candidates)
    if n == 0:
        return []
    plan = _plan_for(n, params)
    plan.cand_point[:n].copy_(torch.from_numpy(np.ascontiguousarray(candidates.points)))
    plan.cand_normal[:n].copy_(torch.from_numpy(np.ascontiguousarray(candidates.normals)))
    plan.cand_depth[:n].copy_(torch.from_numpy(np.ascontiguousarray(candidates.depths)))
    plan.cand_face[:n].copy_(torch.from_numpy(np.arange(n, dtype=np.int32)))
    plan.n_cand.fill_(n)
    plan.reduce()
    return ReducedContacts(plan).patches(0, face_indices=candidates.face_indices)


# ---------------------------------------------------------------------------
# Verification utilities (host side, reduction.py:239-354)
# ---------------------------------------------------------------------------


def patches_from_contacts(candidates: ContactSet) -> list[ContactPatch]:
    """Identity reduction: one single-contact patch per candidate."""
    out = []
    for i in range(len(candidates)):
        p, nrm = candidates.points[i], candidates.normals[i]
        d = float(candidates.depths[i])
        w = max(d, 0.0)
        out.append(ContactPatch(nrm.copy(), p[None].copy(), nrm[None].copy(), candidates.depths[i:i + 1].copy(),
                                candidates.face_indices[i:i + 1].copy(), np.array([i], dtype=np.int64), w, w * p,
                                w * nrm, w * np.cross(p, nrm), 0.0, d))
    return out


def _rebalanced_weights(patch: ContactPatch, ref: np.ndarray) -> np.ndarray:
    from scipy.optimize import nnls

    k = len(patch)
    if k == 0 or patch.weight_sum <= 0.0:
        return np.zeros(k)
    arms = patch.points - ref
    scale = max(np.linalg.norm(arms, axis=1).max(), 1e-9)
    a = np.vstack([patch.normals.T, np.cross(arms, patch.normals).T / scale])
    b = np.concatenate([patch.weighted_normal_sum,
                        (patch.weighted_torque_sum - np.cross(ref, patch.weighted_normal_sum)) / scale])
    return nnls(a, b)[0]


def equivalent_system_check(candidates: ContactSet, patches: list[ContactPatch], reference_point):
    """Relative net-force / net-torque error of the reduced system against the
    full candidate set, each candidate weighted by its clamped depth and patch
    weights rebalanced by NNLS (reduction.py:270-321)."""
    ref = np.asarray(reference_point, dtype=np.float64)
    w = np.maximum(candidates.depths, 0.0)
    force_full = (candidates.normals * w[:, None]).sum(axis=0)
    w_total = w.sum()
    f_scale = np.linalg.norm(force_full)
    degenerate = f_scale < 1e-12 * max(w_total, 1.0)
    if degenerate and w_total > 0.0:
        ref = (candidates.points * w[:, None]).sum(axis=0) / w_total
    torque_full = (np.cross(candidates.points - ref, candidates.normals) * w[:, None]).sum(axis=0)
    force_red = np.zeros(3)
    torque_red = np.zeros(3)
    for patch in patches:
        lam = _rebalanced_weights(patch, ref)
        force_red += lam @ patch.normals
        torque_red += lam @ np.cross(patch.points - ref, patch.normals)
    f_err = np.linalg.norm(force_red - force_full)
    if not degenerate:
        f_err /= f_scale
    t_scale = np.linalg.norm(torque_full)
    t_err = np.linalg.norm(torque_red - torque_full)
    if t_scale > 1e-12 * max(w_total, 1.0):
        t_err /= t_scale
    return float(f_err), float(t_err)


POINTCLOUD_HEADER = "x,y,z,nx,ny,nz,depth,patch_id"


def _row(p, n, d, pid) -> str:
    return ",".join(f"{v:.10g}" for v in (*p, *n, d)) + f",{pid}"


def candidates_csv(candidates: ContactSet, patches: list[ContactPatch]) -> str:
    label = np.full(len(candidates), -1, dtype=np.int64)
    for pid, patch in enumerate(patches):
        label[patch.member_indices] = pid
    rows = [POINTCLOUD_HEADER] + [_row(candidates.points[i], candidates.normals[i], candidates.depths[i], label[i])
                                  for i in range(len(candidates))]
    return "\n".join(rows) + "\n"


def patches_csv(patches: list[ContactPatch]) -> str:
    rows = [POINTCLOUD_HEADER] + [_row(pt.points[i], pt.normals[i], pt.depths[i], pid)
                                  for pid, pt in enumerate(patches) for i in range(len(pt))]
    return "\n".join(rows) + "\n"
