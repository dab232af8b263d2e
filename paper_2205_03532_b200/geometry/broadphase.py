"""Broadphase pair finding over margin-inflated AABBs, on the GPU.

Mirrors contactsim/geometry/broadphase.py (SWEEP_THRESHOLD, aabb_of_points,
aabb_overlap, broadphase_pairs: same names, arguments, errors and results) and adds
the batched forms the multi-pair scenes use (`world_aabbs`, `broadphase_batched`).
The pair tests run in cs_broadphase (csrc/cs_broadphase.cu): all three axes both
ways up to SWEEP_THRESHOLD bodies, the reference's sweep-and-prune tests above it
(the two agree on valid boxes and differ on inverted ones; both are reproduced),
pairs sorted by (id_a, id_b).
"""

from __future__ import annotations

import numpy as np

from .. import _native

SWEEP_THRESHOLD = 64
MAX_BODIES = 2048  # per scene (cs_broadphase)

Aabb = tuple[np.ndarray, np.ndarray]


def aabb_of_points(points: np.ndarray) -> Aabb:
    return points.min(axis=0), points.max(axis=0)


def aabb_overlap(lo_a, hi_a, lo_b, hi_b) -> bool:
    return bool(np.all(lo_a <= hi_b) and np.all(lo_b <= hi_a))


def _dev(a, dtype):
    import torch

    if isinstance(a, torch.Tensor):
        return a.to(device="cuda", dtype=dtype).contiguous()
    return torch.from_numpy(np.array(a, dtype=np.float64 if dtype == torch.float64 else np.int64, order="C")).cuda()


def world_aabbs(mesh_lo, mesh_hi, pose7):
    """RigidBody.world_aabb (dynamics/body.py:77-83, no margin) for n bodies at once:
    mesh AABBs (n,3) and poses (n,7) -> device tensors lo, hi (n,3)."""
    import torch

    ml, mh, p = (_dev(x, torch.float64).reshape(-1, c) for x, c in ((mesh_lo, 3), (mesh_hi, 3), (pose7, 7)))
    lo, hi = torch.empty_like(ml), torch.empty_like(ml)
    _native.call("cs_world_aabb", len(ml), ml.data_ptr(), mh.data_ptr(), p.data_ptr(), lo.data_ptr(), hi.data_ptr(),
                 _native.stream_handle())
    return lo, hi


def broadphase_batched(lo, hi, body_off, margin, ids=None, pair_capacity=None):
    """Broadphase of many scenes in one launch. Scene s owns bodies
    [body_off[s], body_off[s+1]) of lo/hi (B,3) (device or host) with unique ids
    (default: the index within the scene). Returns device tensors
    (pair_off (S+1), pairs (cap,2) int64, n_pairs (S,) int32, status (S,) int32)."""
    import torch

    off = np.asarray(body_off, np.int64)
    S = len(off) - 1
    n = np.diff(off)
    cap = n * (n - 1) // 2 if pair_capacity is None else np.broadcast_to(np.asarray(pair_capacity, np.int64), (S,))
    pair_off = np.concatenate([[0], np.cumsum(cap)]).astype(np.int64)
    if ids is None:
        ids = np.concatenate([np.arange(k) for k in n]) if S else np.zeros(0, np.int64)
    d_lo, d_hi = _dev(lo, torch.float64).reshape(-1, 3), _dev(hi, torch.float64).reshape(-1, 3)
    d_ids = _dev(ids, torch.int64)
    d_off, d_poff = _dev(off, torch.int64), _dev(pair_off, torch.int64)
    d_m = _dev(np.broadcast_to(np.asarray(margin, np.float64), (S,)), torch.float64)
    pairs = torch.zeros((max(int(pair_off[-1]), 1), 2), dtype=torch.int64, device="cuda")
    n_pairs = torch.zeros(max(S, 1), dtype=torch.int32, device="cuda")
    status = torch.zeros(max(S, 1), dtype=torch.int32, device="cuda")
    _native.call("cs_broadphase", S, d_off.data_ptr(), d_lo.data_ptr(), d_hi.data_ptr(), d_ids.data_ptr(),
                 d_m.data_ptr(), d_poff.data_ptr(), pairs.data_ptr(), n_pairs.data_ptr(), status.data_ptr(),
                 _native.stream_handle())
    return d_poff, pairs, n_pairs[:S], status[:S]


def broadphase_pairs(bodies: list[tuple[Aabb, int]], margin: float = 0.0) -> list[tuple[int, int]]:
    """geometry/broadphase.py:25-44: every unordered id pair whose inflated boxes
    overlap, reported once, sorted by (id_a, id_b)."""
    n = len(bodies)
    if n < 2:
        return []
    lo = np.array([np.asarray(aabb[0], dtype=float) for aabb, _ in bodies])
    hi = np.array([np.asarray(aabb[1], dtype=float) for aabb, _ in bodies])
    if not (np.all(np.isfinite(lo - margin)) and np.all(np.isfinite(hi + margin))):
        raise ValueError("non-finite AABB in broadphase input")
    ids = np.array([body_id for _, body_id in bodies], dtype=np.int64)
    if len(np.unique(ids)) != n:
        raise ValueError("broadphase body ids must be unique")
    if n > MAX_BODIES:
        raise ValueError(f"broadphase supports at most {MAX_BODIES} bodies per scene")
    _, pairs, n_pairs, status = broadphase_batched(lo, hi, [0, n], margin, ids)
    st = int(status[0].item())
    if st == 1:
        raise ValueError("non-finite AABB in broadphase input")
    if st != 0:
        raise RuntimeError(f"cs_broadphase status {st}")
    k = int(n_pairs[0].item())
    return [tuple(int(x) for x in p) for p in pairs[:k].cpu().numpy()]
