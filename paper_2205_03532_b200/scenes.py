"""Benchmark workloads of BASELINE.json.

Config 2, the headline: E M16 nut-on-bolt envs. Bolt = SDF body
(SdfResolutionSpec(256, 4) -> 207 x 238 x 256 grid), nut = mesh (80 segments per
turn -> 8 652 vertices / 17 304 triangles), bolt at the identity, nut poses
drawn from the seeded, helix-consistent distribution below.
"""

from __future__ import annotations

import numpy as np

from .geometry.fasteners import ThreadSpec, bolt_thread_base_z, generate_iso_thread
from .math3d import quat_from_axis_angle, quat_multiply

IDENTITY_POSE7 = np.array([0.0, 0.0, 0.0, 1.0, 0.0, 0.0, 0.0])


def nut_poses(n: int, seed: int, pitch: float, z0: float) -> np.ndarray:
    """(n, 7) nut poses, per env in draw order: yaw ~ U[0, 2π), axis ~ N(0, I), tilt ~ U[0, 0.01],
    k ~ {0, 1, 2}, dz ~ U[-6e-4, -2e-4], dx, dy ~ U[-1e-4, 1e-4];
    R = R(axis, tilt) R_z(yaw), t = (dx, dy, z0 + pitch (k + yaw / 2π) + dz)."""
    rng = np.random.default_rng(seed)
    out = np.zeros((n, 7))
    zaxis = np.array([0.0, 0.0, 1.0])
    for e in range(n):
        yaw = rng.uniform(0.0, 2.0 * np.pi)
        axis = rng.normal(size=3)
        tilt = rng.uniform(0.0, 0.01)
        k = int(rng.integers(0, 3))
        dz = rng.uniform(-6e-4, -2e-4)
        dx = rng.uniform(-1e-4, 1e-4)
        dy = rng.uniform(-1e-4, 1e-4)
        out[e, 3:] = quat_multiply(quat_from_axis_angle(axis, tilt), quat_from_axis_angle(zaxis, yaw))
        out[e, :3] = (dx, dy, z0 + pitch * (k + yaw / (2.0 * np.pi)) + dz)
    return out


def m16_specs(segments_per_turn: int = 80):
    return (ThreadSpec.standard("M16", "nut", "tight", segments_per_turn=segments_per_turn),
            ThreadSpec.standard("M16", "bolt", "tight", segments_per_turn=segments_per_turn))


def m16_meshes(segments_per_turn: int = 80):
    nut_spec, bolt_spec = m16_specs(segments_per_turn)
    return generate_iso_thread(nut_spec), generate_iso_thread(bolt_spec), bolt_spec


def m16_workload(n_envs: int, seed: int = 0, resolution: int = 256, segments_per_turn: int = 80, grid=None):
    """Assets + poses of config 2. The bolt grid is generated on the GPU unless given."""
    from .sdf.grid import SdfResolutionSpec, generate_sdf

    nut, bolt, bolt_spec = m16_meshes(segments_per_turn)
    if grid is None:
        grid = generate_sdf(bolt, SdfResolutionSpec(resolution, 4))
    poses = nut_poses(n_envs, seed, bolt_spec.pitch, float(bolt_thread_base_z(bolt_spec)))
    sdf_poses = np.tile(IDENTITY_POSE7, (n_envs, 1))
    cd = np.full(n_envs, 2.0 * grid.voxel_size)  # Scene default contact distance (scene.py:206)
    return {"nut": nut, "bolt": bolt, "grid": grid, "sdf_pose": sdf_poses, "mesh_pose": poses, "cd": cd}


def shard_range(n_envs: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous env block [lo, hi) owned by `rank`."""
    base, extra = divmod(n_envs, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)
