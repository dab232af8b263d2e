"""Generate tests/golden/broadphase.npz by running the REFERENCE broadphase.

Run here (the build container), never on the GPU box:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_broadphase_golden.py

SURVEY §8(f) row 2. Records, on seeded inputs:
* broadphase_pairs(bodies, margin) (geometry/broadphase.py:25-44) for scenes below
  and above SWEEP_THRESHOLD (all-pairs and sweep-and-prune paths), with permuted
  body ids, touching boxes (== bounds) and margins;
* world AABBs as RigidBody.world_aabb computes them (dynamics/body.py:77-83):
  mesh AABB corners through Transform.from_pose(...).apply (math3d.py:164-169).
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from contactsim.geometry.broadphase import broadphase_pairs  # noqa: E402
from contactsim.math3d import Transform  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    rng = np.random.default_rng(21)
    out = {}
    names = []
    for si, (n, spread, margin) in enumerate([(2, 0.01, 0.0), (4, 0.02, 1e-3), (17, 0.05, 2e-3), (63, 0.1, 1e-3),
                                              (64, 0.1, 0.0), (65, 0.1, 5e-4), (150, 0.2, 1e-3), (300, 0.3, 2e-3)]):
        c = rng.uniform(-spread, spread, (n, 3))
        ext = rng.uniform(0.002, 0.03, (n, 3))
        lo, hi = c - ext, c + ext
        if n >= 4:  # exactly touching / inverted boxes (lo of one := hi of another)
            lo[1, 0] = hi[0, 0]
            lo[2] = hi[3]
        if n >= 10:  # ties in lo.x (the sweep's stable order) and a box inverted in y only
            lo[5, 0] = lo[6, 0] = lo[7, 0]
            lo[8, 1], hi[8, 1] = hi[8, 1], lo[8, 1]
        ids = rng.permutation(np.arange(n) * 3 + 7)
        bodies = [((lo[i], hi[i]), int(ids[i])) for i in range(n)]
        pairs = broadphase_pairs(bodies, margin)
        name = f"s{si}"
        out[f"{name}_lo"], out[f"{name}_hi"], out[f"{name}_ids"] = lo, hi, ids.astype(np.int64)
        out[f"{name}_margin"] = np.float64(margin)
        out[f"{name}_pairs"] = np.array(pairs, np.int64).reshape(-1, 2)
        names.append(name)
    out["scenes"] = np.array(names)
    # world AABBs (RigidBody.world_aabb without the margin argument)
    m = 40
    mlo = rng.uniform(-0.02, 0.0, (m, 3))
    mhi = mlo + rng.uniform(0.001, 0.04, (m, 3))
    pose = np.zeros((m, 7))
    pose[:, :3] = rng.uniform(-0.1, 0.1, (m, 3))
    q = rng.standard_normal((m, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    pose[:, 3:] = q
    pose[0, 3:] = (1.0, 0.0, 0.0, 0.0)
    wlo, whi = np.zeros((m, 3)), np.zeros((m, 3))
    for i in range(m):
        lo, hi = mlo[i], mhi[i]
        corners = np.array([[x, y, z] for x in (lo[0], hi[0]) for y in (lo[1], hi[1]) for z in (lo[2], hi[2])])
        w = Transform.from_pose(pose[i, :3], pose[i, 3:]).apply(corners)
        wlo[i], whi[i] = w.min(axis=0), w.max(axis=0)
    out.update(aabb_mesh_lo=mlo, aabb_mesh_hi=mhi, aabb_pose=pose, aabb_world_lo=wlo, aabb_world_hi=whi)
    np.savez_compressed(os.path.join(HERE, "broadphase.npz"), **out)
    print("wrote broadphase.npz:", ", ".join(f"{n}({len(out[n + '_ids'])} bodies, {len(out[n + '_pairs'])} pairs)"
                                             for n in names))


if __name__ == "__main__":
    main()
