"""Rigid-transform helpers used at the API boundary.

Conventions follow contactsim.math3d (/root/reference/pkg/src/contactsim/math3d.py):
quaternions are scalar-first (w, x, y, z) and not renormalised by
`Transform.from_pose`; `Transform.apply` maps points as p R^T + t. The contact
kernels redo the pose arithmetic on the device (quat -> matrix, inverse,
compose, apply) in the reference's rounding order, so these host helpers only
carry data to the C ABI and build fixtures.
"""

from __future__ import annotations

import numpy as np

IDENTITY_QUAT = np.array([1.0, 0.0, 0.0, 0.0])


def quat_to_matrix(q) -> np.ndarray:
    """Rotation matrix of a unit quaternion (math3d.py:45-53 rounding order)."""
    w, x, y, z = (float(c) for c in q)
    xx, yy, zz = x * x, y * y, z * z
    return np.array([
        [1 - 2 * (yy + zz), 2 * (x * y - w * z), 2 * (x * z + w * y)],
        [2 * (x * y + w * z), 1 - 2 * (xx + zz), 2 * (y * z - w * x)],
        [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (xx + yy)],
    ])


def quat_multiply(a, b) -> np.ndarray:
    """Hamilton product a * b."""
    aw, av = float(a[0]), np.asarray(a[1:], dtype=float)
    bw, bv = float(b[0]), np.asarray(b[1:], dtype=float)
    w = aw * bw - av[0] * bv[0] - av[1] * bv[1] - av[2] * bv[2]
    x = aw * bv[0] + av[0] * bw + av[1] * bv[2] - av[2] * bv[1]
    y = aw * bv[1] - av[0] * bv[2] + av[1] * bw + av[2] * bv[0]
    z = aw * bv[2] + av[0] * bv[1] - av[1] * bv[0] + av[2] * bw
    return np.array([w, x, y, z])


def quat_from_axis_angle(axis, angle: float) -> np.ndarray:
    """Unit quaternion rotating by `angle` about `axis` (identity for a zero axis)."""
    v = np.asarray(axis, dtype=float)
    n = np.linalg.norm(v)
    if n == 0.0:
        return IDENTITY_QUAT.copy()
    h = 0.5 * angle
    return np.concatenate([[np.cos(h)], np.sin(h) * v / n])


def matrix_to_quat(m) -> np.ndarray:
    """Shepperd's method (robust on all rotations), normalised."""
    m = np.asarray(m, dtype=float)
    tr = m[0, 0] + m[1, 1] + m[2, 2]
    if tr > 0.0:
        s = 2.0 * np.sqrt(tr + 1.0)
        q = [0.25 * s, (m[2, 1] - m[1, 2]) / s, (m[0, 2] - m[2, 0]) / s, (m[1, 0] - m[0, 1]) / s]
    elif m[0, 0] > m[1, 1] and m[0, 0] > m[2, 2]:
        s = 2.0 * np.sqrt(1.0 + m[0, 0] - m[1, 1] - m[2, 2])
        q = [(m[2, 1] - m[1, 2]) / s, 0.25 * s, (m[0, 1] + m[1, 0]) / s, (m[0, 2] + m[2, 0]) / s]
    elif m[1, 1] > m[2, 2]:
        s = 2.0 * np.sqrt(1.0 + m[1, 1] - m[0, 0] - m[2, 2])
        q = [(m[0, 2] - m[2, 0]) / s, (m[0, 1] + m[1, 0]) / s, 0.25 * s, (m[1, 2] + m[2, 1]) / s]
    else:
        s = 2.0 * np.sqrt(1.0 + m[2, 2] - m[0, 0] - m[1, 1])
        q = [(m[1, 0] - m[0, 1]) / s, (m[0, 2] + m[2, 0]) / s, (m[1, 2] + m[2, 1]) / s, 0.25 * s]
    q = np.array(q)
    return q / np.linalg.norm(q)


class Transform:
    """Rotation matrix + translation; `apply` maps body-frame points to world."""

    __slots__ = ("rotation", "translation")

    def __init__(self, rotation=None, translation=None):
        self.rotation = np.eye(3) if rotation is None else np.asarray(rotation, dtype=float)
        self.translation = np.zeros(3) if translation is None else np.asarray(translation, dtype=float)

    @classmethod
    def from_pose(cls, position, quaternion) -> "Transform":
        return cls(quat_to_matrix(np.asarray(quaternion, dtype=float)), position)

    def apply(self, points) -> np.ndarray:
        return np.asarray(points, dtype=float) @ self.rotation.T + self.translation

    def apply_vector(self, vectors) -> np.ndarray:
        return np.asarray(vectors, dtype=float) @ self.rotation.T

    def inverse(self) -> "Transform":
        rt = self.rotation.T
        return Transform(rt, -rt @ self.translation)

    def compose(self, other: "Transform") -> "Transform":
        return Transform(self.rotation @ other.rotation, self.rotation @ other.translation + self.translation)

    def pose12(self) -> np.ndarray:
        """(R row-major, t): the CS_POSE12 row the C ABI consumes."""
        return np.concatenate([np.ascontiguousarray(self.rotation, dtype=np.float64).reshape(9),
                               np.asarray(self.translation, dtype=np.float64).reshape(3)])
