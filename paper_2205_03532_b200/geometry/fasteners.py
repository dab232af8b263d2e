"""Procedural benchmark assets: ISO metric nut/bolt threads, pegs/holes, boxes.

These are fixtures for the benchmark scenes, not part of the
hot path. They rebuild the reference's lathe meshes
(/root/reference/pkg/src/contactsim/geometry/threads.py:139-223,
shapes.py:45-130) vertex-for-vertex and triangle-for-triangle — the ring/band
ordering is produced with vectorised index arithmetic here — so that
tests/test_fixtures.py can compare them with the golden meshes byte for byte.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .mesh import TriMesh

# ISO 724 coarse pitches, nominal diameters, ISO 965 nut/bolt and ISO 286 peg/hole
# diametral clearances (threads.py:30-56).
ISO_COARSE_PITCH = {"M4": 0.0007, "M8": 0.00125, "M12": 0.00175, "M16": 0.0020, "M20": 0.0025}
ISO_NOMINAL_DIAMETER = {"M4": 0.004, "M8": 0.008, "M12": 0.012, "M16": 0.016, "M20": 0.020}
ISO_NUT_BOLT_CLEARANCE = {
    "M4": (0.416e-3, 0.736e-3), "M8": (0.848e-3, 1.325e-3), "M12": (1.26e-3, 1.86e-3),
    "M16": (1.472e-3, 2.127e-3), "M20": (1.879e-3, 2.664e-3),
}
ISO_PEG_HOLE_CLEARANCE = {
    0.004: (0.104e-3, 0.112e-3), 0.008: (0.105e-3, 0.114e-3),
    0.012: (0.206e-3, 0.217e-3), 0.016: (0.506e-3, 0.517e-3),
}
HEX_WIDTH_FACTOR = 1.5
HEAD_HEIGHT_FACTOR = 0.65
DEFAULT_NUT_TURNS = 5
ROWS_PER_TURN_MIN = 16


@dataclass(frozen=True)
class ThreadSpec:
    nominal_diameter: float
    pitch: float
    clearance: float = 0.0
    turns: int = DEFAULT_NUT_TURNS
    segments_per_turn: int = 64
    kind: str = "bolt"

    def __post_init__(self):
        checks = [(self.pitch > 0.0, "pitch must be positive"), (self.clearance >= 0.0, "clearance must be non-negative"),
                  (self.turns >= 1, "turns must be at least 1"),
                  (self.segments_per_turn >= 16, "segments_per_turn must be at least 16"),
                  (self.kind in ("nut", "bolt"), f"unknown thread kind {self.kind!r}")]
        for ok, msg in checks:
            if not ok:
                raise ValueError(msg)

    @classmethod
    def standard(cls, size: str, kind: str, fit: str = "tight", turns=None, segments_per_turn: int = 64):
        if size not in ISO_COARSE_PITCH:
            raise ValueError(f"unknown metric size {size!r}")
        lo, hi = ISO_NUT_BOLT_CLEARANCE[size]
        return cls(ISO_NOMINAL_DIAMETER[size], ISO_COARSE_PITCH[size],
                   {"tight": lo, "loose": hi}[fit] if kind == "nut" else 0.0,
                   DEFAULT_NUT_TURNS if turns is None else turns, segments_per_turn, kind)

    @property
    def major_radius(self) -> float:
        return self.nominal_diameter / 2.0

    @property
    def thread_depth(self) -> float:
        return 5.0 / 8.0 * (np.sqrt(3.0) / 2.0) * self.pitch

    @property
    def minor_radius(self) -> float:
        return self.major_radius - self.thread_depth


# ------------------------------------------------------------------ angular sampling

def thetas_with_corners(segments: int, sides=None) -> np.ndarray:
    base = np.linspace(0.0, 2.0 * np.pi, segments, endpoint=False)
    if sides is None:
        return base
    half = np.pi / sides
    merged = np.unique(np.round(np.concatenate([base, half + np.arange(sides) * 2.0 * half]), 12))
    return merged[merged < 2.0 * np.pi - 1e-12]


def polygon_radius(thetas, width_across_flats: float, sides: int) -> np.ndarray:
    half = np.pi / sides
    return (width_across_flats / 2.0) / np.cos(np.mod(thetas + half, 2.0 * half) - half)


def thread_profile_radius(thetas, z: float, diameter: float, pitch: float, radial_offset: float = 0.0):
    """ISO basic profile radius at height z (right-handed helix phase u = z - p θ / 2π)."""
    p = pitch
    r_major = diameter / 2.0
    r_minor = r_major - 5.0 / 8.0 * (np.sqrt(3.0) / 2.0 * p)
    u = np.mod(z - p * thetas / (2.0 * np.pi), p)
    a = np.minimum(u, p - u)
    flank = r_major - (a - p / 16.0) * np.sqrt(3.0)
    return np.where(a <= p / 16.0, r_major, np.where(a >= 3.0 * p / 8.0, r_minor, flank)) + radial_offset


# ------------------------------------------------------------------ lathe meshing

def _rings(thetas, rows) -> np.ndarray:
    c, s = np.cos(thetas), np.sin(thetas)
    out = []
    for z, radii in rows:
        r = np.asarray(radii, dtype=float)
        out.append(np.column_stack([r * c, r * s, np.full_like(thetas, z)]))
    return np.vstack(out)


def _bands(first_ring: int, n_rings: int, m: int, flip: bool) -> np.ndarray:
    """Two triangles per quad between consecutive rings, j-major, wrapped in theta."""
    if n_rings < 2:
        return np.zeros((0, 3), np.int64)
    i = np.arange(n_rings - 1)[:, None]
    j = np.arange(m)[None, :]
    a0 = first_ring * m + i * m + j
    a1 = first_ring * m + i * m + (j + 1) % m
    b0, b1 = a0 + m, a1 + m
    if flip:
        t = np.stack([np.stack([a0, b1, a1], -1), np.stack([a0, b0, b1], -1)], axis=2)
    else:
        t = np.stack([np.stack([a0, a1, b1], -1), np.stack([a0, b1, b0], -1)], axis=2)
    return t.reshape(-1, 3)


def revolve_solid(thetas, rows) -> TriMesh:
    """Heightfield r(θ, z) closed with fan caps (shapes.py:45-66 layout)."""
    m, nr = len(thetas), len(rows)
    verts = np.vstack([_rings(thetas, rows), [[0.0, 0.0, rows[0][0]]], [[0.0, 0.0, rows[-1][0]]]])
    bottom, top = nr * m, nr * m + 1
    j = np.arange(m)
    k = (j + 1) % m
    last = (nr - 1) * m
    caps = np.stack([np.stack([np.full(m, bottom), k, j], -1),
                     np.stack([np.full(m, top), last + j, last + k], -1)], axis=1).reshape(-1, 3)
    return TriMesh(verts, np.vstack([_bands(0, nr, m, False), caps]).astype(np.int32))


def annular_solid(thetas, inner_rows, outer_rows) -> TriMesh:
    """Solid between an inner and an outer heightfield (shapes.py:69-103 layout)."""
    if not (np.isclose(inner_rows[0][0], outer_rows[0][0]) and np.isclose(inner_rows[-1][0], outer_rows[-1][0])):
        raise ValueError("inner and outer stations must agree at bottom and top z")
    m, ni, no = len(thetas), len(inner_rows), len(outer_rows)
    verts = np.vstack([_rings(thetas, inner_rows), _rings(thetas, outer_rows)])
    j = np.arange(m)
    k = (j + 1) % m
    ib, ob, it, ot = 0, ni * m, (ni - 1) * m, (ni + no - 1) * m
    caps = np.stack([np.stack([ib + j, ob + k, ob + j], -1), np.stack([ib + j, ib + k, ob + k], -1),
                     np.stack([it + j, ot + j, ot + k], -1), np.stack([it + j, ot + k, it + k], -1)],
                    axis=1).reshape(-1, 3)
    tris = np.vstack([_bands(0, ni, m, True), _bands(ni, no, m, False), caps])
    return TriMesh(verts, tris.astype(np.int32))


# ------------------------------------------------------------------ assets

def _thread_rows(spec: ThreadSpec, thetas, z0: float, z1: float, offset: float):
    per_turn = max(ROWS_PER_TURN_MIN, spec.segments_per_turn // 4)
    n = int(round((z1 - z0) / spec.pitch * per_turn))
    return [(float(z), thread_profile_radius(thetas, float(z), spec.nominal_diameter, spec.pitch, offset))
            for z in np.linspace(z0, z1, n + 1)]


def bolt_thread_base_z(spec: ThreadSpec) -> float:
    """Thread start height, snapped up to a whole number of pitches (threads.py:157-161)."""
    return np.ceil((HEAD_HEIGHT_FACTOR + 0.5) * spec.nominal_diameter / spec.pitch) * spec.pitch


def generate_iso_thread(spec: ThreadSpec) -> TriMesh:
    """Watertight bolt (hex head + shank + thread) or nut (hex body, threaded bore)."""
    d = spec.nominal_diameter
    thetas = thetas_with_corners(spec.segments_per_turn, sides=6)
    hex_r = polygon_radius(thetas, HEX_WIDTH_FACTOR * d, 6)
    if spec.kind == "bolt":
        z0 = bolt_thread_base_z(spec)
        shank = np.full(len(thetas), spec.major_radius)
        head = HEAD_HEIGHT_FACTOR * d
        rows = [(0.0, hex_r), (head, hex_r), (head, shank), (z0, shank)]
        rows += _thread_rows(spec, thetas, z0, z0 + spec.turns * spec.pitch, 0.0)[1:]
        return revolve_solid(thetas, rows)
    height = spec.turns * spec.pitch
    inner = _thread_rows(spec, thetas, 0.0, height, spec.clearance / 2.0)
    return annular_solid(thetas, inner, [(0.0, hex_r), (height, hex_r)])


def generate_peg_hole(diameter: float, clearance: float, length: float, segments: int = 32, hole_depth=None):
    """Round peg (z in [0, length]) and a square block with a matching through-hole."""
    if clearance < 0.0:
        raise ValueError("clearance must be non-negative")
    if diameter <= 0.0 or length <= 0.0:
        raise ValueError("diameter and length must be positive")
    depth = hole_depth if hole_depth is not None else 2.0 * length / 3.0
    thetas = thetas_with_corners(segments, sides=4)
    ring_pitch = np.pi * diameter / segments
    n_peg = max(2, int(round(length / ring_pitch)))
    peg = revolve_solid(thetas, [(float(z), np.full(len(thetas), diameter / 2.0))
                                 for z in np.linspace(0.0, length, n_peg + 1)])
    n_hole = max(2, int(round(depth / ring_pitch)))
    hole_r = np.full(len(thetas), (diameter + clearance) / 2.0)
    block_r = polygon_radius(thetas, 3.0 * diameter, 4)
    block = annular_solid(thetas, [(float(z), hole_r) for z in np.linspace(0.0, depth, n_hole + 1)],
                          [(0.0, block_r), (depth, block_r)])
    return peg, block


def make_box(extents, subdivisions: int = 1, center=(0.0, 0.0, 0.0)) -> TriMesh:
    """Axis-aligned box, each face split into subdivisions² quads, outward winding
    (shapes.py:130-164: vertices are numbered in first-use order)."""
    e = np.asarray(extents, dtype=float)
    n = max(1, int(subdivisions))
    index: dict = {}
    verts = []
    tris = []

    def vid(p) -> int:
        key = (int(p[0]), int(p[1]), int(p[2]))
        got = index.get(key)
        if got is None:
            got = index[key] = len(verts)
            verts.append(np.array(key, dtype=float) / n * e - e / 2.0 + center)
        return got

    faces = [((0, 0, 0), (0, 1, 0), (1, 0, 0)), ((0, 0, n), (1, 0, 0), (0, 1, 0)),
             ((0, 0, 0), (1, 0, 0), (0, 0, 1)), ((0, n, 0), (0, 0, 1), (1, 0, 0)),
             ((0, 0, 0), (0, 0, 1), (0, 1, 0)), ((n, 0, 0), (0, 1, 0), (0, 0, 1))]
    for o, du, dv in faces:
        o, du, dv = np.array(o), np.array(du), np.array(dv)
        for a in range(n):
            for b in range(n):
                q = [vid(o + a * du + b * dv), vid(o + (a + 1) * du + b * dv),
                     vid(o + (a + 1) * du + (b + 1) * dv), vid(o + a * du + (b + 1) * dv)]
                tris += [(q[0], q[1], q[2]), (q[0], q[2], q[3])]
    return TriMesh(np.array(verts), np.array(tris, dtype=np.int32))
