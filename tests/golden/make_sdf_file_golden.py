"""Golden files for the SDF on-disk format, written by the
REFERENCE itself: SignedDistanceGrid.save (/root/reference/pkg/src/contactsim/sdf/grid.py:138-149)
of the r64 peg grid, and the reference's TriMesh.content_digest of the golden meshes
(the cached_sdf key, grid.py:259). Run once in the build container:

    python tests/golden/make_sdf_file_golden.py
"""

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from contactsim.geometry.mesh import TriMesh  # noqa: E402
from contactsim.sdf.grid import SignedDistanceGrid  # noqa: E402

g = np.load(os.path.join(HERE, "grid_peg_r64.npz"))
grid = SignedDistanceGrid(g["origin"], float(g["voxel"]), tuple(int(d) for d in g["dims"]), g["values"],
                          (g["aabb_lo"], g["aabb_hi"]))
grid.save(os.path.join(HERE, "ref_peg_r64.sdf"))
m = np.load(os.path.join(HERE, "meshes.npz"))
digests = {k: TriMesh(m[f"{k}_v"], m[f"{k}_t"]).content_digest() for k in ("nut", "bolt", "peg", "hole")}
with open(os.path.join(HERE, "sdf_file.json"), "w") as fh:
    json.dump({"file": "ref_peg_r64.sdf", "mesh_digests": digests}, fh, indent=1)
print(digests)
