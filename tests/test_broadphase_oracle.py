"""Broadphase oracle (oracle/cs_oracle_broadphase.c) pinned against the reference's
own outputs (tests/golden/broadphase.npz, tests/golden/make_broadphase_golden.py):
broadphase_pairs (geometry/broadphase.py:25-44, all-pairs and sweep-and-prune paths)
and the world AABBs of RigidBody.world_aabb (dynamics/body.py:77-83)."""

import numpy as np
import pytest

from conftest import golden
from oracle import oracle as O

G = golden("broadphase.npz")


@pytest.mark.parametrize("name", [str(s) for s in G["scenes"]])
def test_broadphase_oracle_matches_reference(name):
    got = O.broadphase_pairs(G[f"{name}_lo"], G[f"{name}_hi"], G[f"{name}_ids"], float(G[f"{name}_margin"]))
    assert np.array_equal(got, G[f"{name}_pairs"])


def test_world_aabb_oracle_matches_reference():
    lo, hi = O.world_aabb(G["aabb_mesh_lo"], G["aabb_mesh_hi"], G["aabb_pose"])
    assert lo.tobytes() == G["aabb_world_lo"].tobytes() and hi.tobytes() == G["aabb_world_hi"].tobytes()


def test_broadphase_oracle_rejects_non_finite():
    lo = np.zeros((3, 3)); hi = np.ones((3, 3)); lo[1, 2] = np.nan
    with pytest.raises(ValueError):
        O.broadphase_pairs(lo, hi, [0, 1, 2], 0.0)
