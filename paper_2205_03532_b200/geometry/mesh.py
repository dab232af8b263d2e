"""Triangle meshes as the contact path consumes them.

Same data contract as contactsim.geometry.mesh.TriMesh
(/root/reference/pkg/src/contactsim/geometry/mesh.py:16-111): float64 vertices
(n, 3), int32 triangles (m, 3), immutable after construction, validated on
entry with MeshValidationError. Only what the hot path and SDF generation use is
provided (OBJ import/export is out of scope).
"""

from __future__ import annotations

import hashlib

import numpy as np

from ..errors import MeshValidationError


class TriMesh:
    __slots__ = ("vertices", "triangles", "face_normals", "_watertight", "_aabb", "_device_handle", "__weakref__")

    def __init__(self, vertices, triangles):
        v = np.ascontiguousarray(np.asarray(vertices, dtype=np.float64).reshape(-1, 3))
        t = np.ascontiguousarray(np.asarray(triangles, dtype=np.int32).reshape(-1, 3))
        if not np.isfinite(v).all():
            raise MeshValidationError("non-finite vertex coordinate")
        if t.size:
            if t.min() < 0 or t.max() >= len(v):
                raise MeshValidationError(f"triangle index out of range (have {len(v)} vertices)")
            if ((t[:, 0] == t[:, 1]) | (t[:, 1] == t[:, 2]) | (t[:, 0] == t[:, 2])).any():
                raise MeshValidationError("triangle with repeated vertex indices")
        corners = v[t]
        n = np.cross(corners[:, 1] - corners[:, 0], corners[:, 2] - corners[:, 0])
        length = np.linalg.norm(n, axis=1)
        if (length <= 0.0).any():
            raise MeshValidationError(f"zero-area face at triangle {int(np.argmin(length))}")
        self.vertices = v
        self.triangles = t
        self.face_normals = n / length[:, None]
        for a in (self.vertices, self.triangles, self.face_normals):
            a.flags.writeable = False
        self._watertight = None
        self._aabb = None
        self._device_handle = None  # set by collide.register_mesh

    def __len__(self) -> int:
        return len(self.triangles)

    @property
    def num_vertices(self) -> int:
        return len(self.vertices)

    def aabb(self) -> tuple[np.ndarray, np.ndarray]:
        if self._aabb is None:
            self._aabb = (self.vertices.min(axis=0), self.vertices.max(axis=0))
        return self._aabb

    def triangle_corners(self) -> np.ndarray:
        return self.vertices[self.triangles]

    def is_watertight(self) -> bool:
        """Closed, consistently wound 2-manifold: every directed edge once, with its reverse present."""
        if self._watertight is None:
            if len(self.triangles) == 0:
                self._watertight = False
            else:
                t = self.triangles.astype(np.int64)
                src = t.reshape(-1)
                dst = t[:, [1, 2, 0]].reshape(-1)
                nv = len(self.vertices)
                fwd = src * nv + dst
                rev = dst * nv + src
                self._watertight = bool(len(np.unique(fwd)) == len(fwd) and np.isin(fwd, rev).all())
        return self._watertight

    def require_watertight(self, what: str) -> None:
        if not self.is_watertight():
            raise MeshValidationError(f"{what} requires a watertight mesh")

    def content_digest(self) -> str:
        """sha256 over vertex then triangle bytes, 24 hex chars (the SDF cache key)."""
        h = hashlib.sha256()
        h.update(self.vertices.tobytes())
        h.update(self.triangles.tobytes())
        return h.hexdigest()[:24]
