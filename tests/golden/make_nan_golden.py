"""Golden reduction cases with NaN inputs, by running the REFERENCE.

Run here (the build container), never on the GPU box:

    python tests/golden/make_nan_golden.py

reduce_contacts (pkg/src/contactsim/contacts/reduction.py:45-236) takes any
ContactSet; NaN coordinates, normals or depths follow numpy's rules through it:
argmax returns the first NaN, comparisons with NaN are False (so `cross <= 0` keeps
a point on the hull chain, reduction.py:215), lexsort orders NaN after every number
(reduction.py:211), sums propagate NaN. These cases put NaN in points (one or two
coordinates: the projections u and/or v), in normals and in depths, alone and
together, with and without min_depth, at several batch sizes, and are written to
red_nan.npz in red_synth.npz's layout.

Generation on a grid holding NaN nodes: the r64 bolt grid (grid_bolt_r64.npz) with
40 nodes near the surface set to NaN (their flat indices are stored as g_bad), three
of gen_r64's envs through generate_contacts + reduce_contacts as Scene calls them
(ReductionParams(min_depth=-cd)); NaN samples never make a contact (phi <= cd is
False) but NaN gradients give NaN normals, which reach the reduction.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from contactsim.contacts.generation import generate_contacts  # noqa: E402
from contactsim.contacts.reduction import reduce_contacts  # noqa: E402
from contactsim.contacts.types import CollisionPairing, ContactSet, ReductionParams  # noqa: E402
from contactsim.geometry.mesh import TriMesh  # noqa: E402
from contactsim.math3d import Transform  # noqa: E402
from contactsim.sdf.grid import SignedDistanceGrid  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from make_golden import flatten, pack_contactset, pack_patches  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def cloud(rng, n, spread=0.05):
    """A patch-like contact cloud: points on a small disc, normals near +z, mixed depths."""
    P = rng.normal(size=(n, 3)) * np.array([1e-3, 1e-3, 1e-5])
    N = np.tile([0.0, 0.0, 1.0], (n, 1)) + spread * rng.normal(size=(n, 3))
    N /= np.linalg.norm(N, axis=1)[:, None]
    D = rng.uniform(-1e-4, 5e-4, n)
    return P, N, D


def main() -> None:
    rng = np.random.default_rng(532)
    out, cases = {}, []
    # (n, where the NaNs go, params)
    specs = [
        (200, {"pt_u": [5, 77, 150]}, ReductionParams()),
        (200, {"pt_v": [3, 4, 199]}, ReductionParams()),
        (150, {"pt_xyz": [0, 60]}, ReductionParams(per_patch_cap=8)),
        (120, {"pt_u": [10], "pt_v": [11, 12]}, ReductionParams(batch_size=7)),
        (300, {"nrm": [2, 90]}, ReductionParams()),
        (300, {"nrm": [0]}, ReductionParams(batch_size=64)),
        (200, {"dep": [7, 8, 100]}, ReductionParams()),
        (200, {"dep": [0]}, ReductionParams(min_depth=-5e-5)),
        (250, {"pt_u": [1, 2, 3], "dep": [40], "nrm": [41]}, ReductionParams(max_patches=4, batch_size=50)),
        (90, {"pt_u": list(range(0, 90, 3))}, ReductionParams(per_patch_cap=4)),
        (60, {"pt_xyz": list(range(10))}, ReductionParams()),
    ]
    for ci, (n, nans, rp) in enumerate(specs):
        P, N, D = cloud(rng, n)
        if ci % 2:  # a second, tilted cluster: more than one patch
            P2, N2, D2 = cloud(rng, n // 3)
            N2 = N2 @ np.array([[1.0, 0, 0], [0, 0, -1.0], [0, 1.0, 0]])
            P, N, D = np.vstack([P, P2 + 3e-3]), np.vstack([N, N2]), np.concatenate([D, D2])
            n = len(D)
        for i in nans.get("pt_u", []):
            P[i, 0] = np.nan  # t1 has an x component for normals near +z: u is NaN
        for i in nans.get("pt_v", []):
            P[i, 1] = np.nan
        for i in nans.get("pt_xyz", []):
            P[i] = np.nan
        for i in nans.get("nrm", []):
            N[i] = np.nan
        for i in nans.get("dep", []):
            D[i] = np.nan
        cs = ContactSet(P, N, D, np.arange(n) * 3 + 1, 0, 1)
        patches = reduce_contacts(cs, rp)
        pre = f"c{ci}_"
        md = np.nan if rp.min_depth is None else rp.min_depth
        out[pre + "params"] = np.array([rp.max_patches, rp.per_patch_cap, rp.normal_cone_cos, md, rp.batch_size])
        flatten(pre + "cs_", pack_contactset(cs), out)
        flatten(pre + "pt_", pack_patches(patches, rp.per_patch_cap), out)
        cases.append(ci)
        print(f"nan case {ci}: n={n} {sorted(nans)} -> {len(patches)} patches")
    out["cases"] = np.array(cases)

    g = np.load(os.path.join(OUT, "grid_bolt_r64.npz"))
    m = np.load(os.path.join(OUT, "meshes.npz"))
    gen = np.load(os.path.join(OUT, "gen_r64.npz"))
    vals = g["values"].astype(np.float32).copy()
    near = np.nonzero(np.abs(vals) < 2.0 * float(g["voxel"]))[0]
    bad = np.sort(rng.choice(near, 40, replace=False))
    vals[bad] = np.nan
    grid = SignedDistanceGrid(g["origin"], float(g["voxel"]), g["dims"], vals, (g["aabb_lo"], g["aabb_hi"]))
    nut = TriMesh(m["nut_v"], m["nut_t"])
    cd = float(gen["cd"])
    envs = [int(e) for e in gen["envs"][:3]]
    out["g_bad"] = bad
    out["g_envs"] = np.array(envs)
    out["g_cd"] = np.array(cd)
    for e in envs:
        sp, mp = gen[f"e{e}_sdf_pose"], gen[f"e{e}_mesh_pose"]
        cs = generate_contacts(CollisionPairing(0, 1), grid, nut, Transform.from_pose(sp[:3], sp[3:]),
                               Transform.from_pose(mp[:3], mp[3:]), cd)
        patches = reduce_contacts(cs, ReductionParams(min_depth=-cd))
        pre = f"ge{e}_"
        out[pre + "sdf_pose"] = sp
        out[pre + "mesh_pose"] = mp
        flatten(pre + "cs_", pack_contactset(cs), out)
        flatten(pre + "pt_", pack_patches(patches, 6), out)
        print(f"nan grid env {e}: {len(cs)} candidates ({int(np.isnan(cs.normals).any(axis=1).sum())} NaN normals) "
              f"-> {len(patches)} patches")
    np.savez_compressed(os.path.join(OUT, "red_nan.npz"), **out)


if __name__ == "__main__":
    main()
