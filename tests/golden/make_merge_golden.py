"""Golden cases for the merge branch of the reference's _add_patch, by running the REFERENCE.

Run here (the build container), never on the GPU box:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_merge_golden.py

_add_patch (pkg/src/contactsim/contacts/reduction.py:91-106) merges a new patch into
an existing one when the nearest builder is `similar` (cos >= cone) and either
cos >= cos 5 deg or the builder list is at its cap. Under consistent arithmetic a seed
is never similar: _assign_to_existing would have absorbed it. The reference's
arithmetic is not consistent: the assignment cosines come from a BLAS gemm
(`normals[batch] @ reps.T`, reduction.py:82) and the _add_patch cosines from a gemv
(`reps @ patch.normal`, reduction.py:94), which round differently in the last ulp
for about a third of the inputs. A candidate whose gemm cosine is 1 ulp below the
cone and whose gemv cosine reaches it is therefore left unassigned, seeds a patch,
and that patch merges. These cases put such a candidate in a second batch:

  batch 1: a seed with normal b (builder A) and one with a far normal (builder B)
  batch 2: the boundary candidate x (gemm(x, b) < cone <= gemv(b, x)) and a copy of b

The cone is set to the gemv cosine itself. Variants: cone above cos 5 deg (the merge
by similarity) and below it with max_patches = 2 (the merge at the cap); the merged
patch deeper than A (A adopts the new normal) or shallower. Every case is checked
here to really take the merge branch (instrumented _add_patch) and written to
red_merge.npz in red_synth.npz's layout.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from contactsim.contacts import reduction as ref_red  # noqa: E402
from contactsim.contacts.reduction import MERGE_COS, reduce_contacts  # noqa: E402
from contactsim.contacts.types import ContactSet, ReductionParams  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from make_golden import flatten, pack_contactset, pack_patches  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def unit(v):
    return v / np.linalg.norm(v)


def boundary_pair(rng, angle_deg):
    """(b, x, cone): unit normals about angle_deg apart whose gemm cosine (as in the
    assignment of a 2-candidate batch against 2 builders) is strictly below the gemv
    cosine (as in _add_patch with 2 builders); cone = the gemv cosine."""
    far = np.array([0.0, 0.0, -1.0])
    for _ in range(100000):
        b = unit(np.array([0.3, -0.2, 1.0]) + 0.2 * rng.normal(size=3))
        axis = unit(np.cross(b, rng.normal(size=3)))
        t = np.radians(angle_deg) * (0.8 + 0.4 * rng.random())
        x = unit(b * np.cos(t) + axis * np.sin(t))
        reps = np.array([b, far])
        gemm = (np.array([x, b]) @ reps.T)[0, 0]  # reduction.py:82, batch of 2, 2 builders
        gemv = (reps @ x)[0]                       # reduction.py:94, 2 builders
        if gemm < gemv:
            return b, x, float(gemv)
    raise RuntimeError("no boundary pair found")


class MergeCounter:
    """Wraps _add_patch and classifies each call by the reference's own branch test."""

    def __init__(self):
        self.calls = self.merges = 0

    def __enter__(self):
        self.orig = ref_red._add_patch

        def wrapped(patch, builders, candidates, params):
            self.calls += 1
            if builders:
                cos = np.array([b.normal for b in builders]) @ patch.normal
                best = int(np.argmax(cos))
                if cos[best] >= params.normal_cone_cos and (cos[best] >= MERGE_COS or
                                                            len(builders) >= params.max_patches):
                    self.merges += 1
            return self.orig(patch, builders, candidates, params)

        ref_red._add_patch = wrapped
        return self

    def __exit__(self, *a):
        ref_red._add_patch = self.orig


def main() -> None:
    rng = np.random.default_rng(2205)
    out, cases = {}, []
    far = np.array([0.0, 0.0, -1.0])
    specs = [  # (angle deg, max_patches, x deeper than A, extra candidates)
        (2.0, 128, False, 0),
        (2.0, 128, True, 0),
        (3.5, 128, True, 40),
        (12.0, 2, False, 0),
        (12.0, 2, True, 0),
        (25.0, 2, True, 30),
    ]
    for ci, (ang, N, deeper, extra) in enumerate(specs):
        b, x, cone = boundary_pair(rng, ang)
        pts = [rng.normal(size=3) * 1e-3 for _ in range(4)]
        nrm = [b, far, x, b]
        dep = [2e-4, 1e-4, 3e-4 if deeper else 5e-5, 1.5e-4]
        for _ in range(extra):  # more candidates after the boundary pair: more batches on the merged state
            pts.append(rng.normal(size=3) * 1e-3)
            nrm.append(unit(b + 0.05 * rng.normal(size=3)) if rng.random() < 0.7 else unit(rng.normal(size=3)))
            dep.append(rng.normal() * 2e-4)
        n = len(dep)
        cs = ContactSet(np.array(pts), np.array(nrm), np.array(dep), np.arange(n) * 5 + 2, 0, 1)
        rp = ReductionParams(max_patches=N, normal_cone_cos=cone, batch_size=2)
        with MergeCounter() as mc:
            patches = reduce_contacts(cs, rp)
        assert mc.merges >= 1, f"case {ci}: the merge branch was not taken ({mc.calls} _add_patch calls)"
        pre = f"c{ci}_"
        out[pre + "params"] = np.array([rp.max_patches, rp.per_patch_cap, rp.normal_cone_cos, np.nan, rp.batch_size])
        out[pre + "merges"] = np.array(mc.merges)
        flatten(pre + "cs_", pack_contactset(cs), out)
        flatten(pre + "pt_", pack_patches(patches, rp.per_patch_cap), out)
        cases.append(ci)
        print(f"merge case {ci}: n={n} cone={cone!r} N={N} -> {len(patches)} patches, "
              f"{mc.merges} merges in {mc.calls} _add_patch calls")
    out["cases"] = np.array(cases)
    np.savez_compressed(os.path.join(OUT, "red_merge.npz"), **out)


if __name__ == "__main__":
    main()
