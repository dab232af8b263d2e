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


# ---------------------------------------------------------------- config 3

SUITE_PEGS = (0.004, 0.008, 0.012, 0.016)
SUITE_THREADS = ("M4", "M8", "M12", "M16", "M20")


def _peg_poses(rng, n: int, clearance: float, depth: float) -> np.ndarray:
    """Peg (SDF body, its frame: z in [0, length]) partially inserted into the
    hole block (mesh body at the identity, hole along z in [0, depth]): insertion
    U[0.1, 0.9] depth, lateral offset U[-1.5, 1.5] half-clearances (some
    penetrating the wall), tilt U[0, 0.01] rad about a random axis."""
    out = np.zeros((n, 7))
    for e in range(n):
        axis = rng.normal(size=3)
        tilt = rng.uniform(0.0, 0.01)
        ins = rng.uniform(0.1, 0.9) * depth
        c = 0.75 * clearance
        out[e, 3:] = quat_from_axis_angle(axis, tilt)
        out[e, :3] = (rng.uniform(-c, c), rng.uniform(-c, c), depth - ins)
    return out


def suite_workload(n_envs: int, seed: int = 0, resolution: int = 256, segments_per_turn: int = 64):
    """Config 3: pegs 4/8/12/16 mm in ISO 286 holes (tight fit) and
    M4..M20 nuts on bolts, env i using asset i mod 9. Roles as assign_roles picks
    them (contacts/generation.py:32-51: larger triangle count -> SDF). Returns the
    assets (each with its grid generated on the GPU) and per-env asset index,
    poses and contact distances."""
    from .contacts.generation import BodyShape, assign_roles
    from .geometry.fasteners import ISO_PEG_HOLE_CLEARANCE, generate_peg_hole
    from .sdf.grid import SdfResolutionSpec, generate_sdf

    rng = np.random.default_rng(seed)
    assets = []
    for d in SUITE_PEGS:
        clearance = ISO_PEG_HOLE_CLEARANCE[d][0]
        peg, block = generate_peg_hole(d, clearance, 5.0 * d)
        assets.append({"name": f"peg{int(d * 1000)}", "a": peg, "b": block, "kind": "peg", "clearance": clearance,
                       "depth": 2.0 * 5.0 * d / 3.0})
    for size in SUITE_THREADS:
        nut_spec = ThreadSpec.standard(size, "nut", "tight", segments_per_turn=segments_per_turn)
        bolt_spec = ThreadSpec.standard(size, "bolt", "tight", segments_per_turn=segments_per_turn)
        assets.append({"name": size, "a": generate_iso_thread(bolt_spec), "b": generate_iso_thread(nut_spec),
                       "kind": "thread", "pitch": bolt_spec.pitch, "z0": float(bolt_thread_base_z(bolt_spec))})
    for a in assets:
        pr = assign_roles(BodyShape(0, len(a["a"].triangles), False), BodyShape(1, len(a["b"].triangles), False))
        a["sdf"], a["mesh"] = (a["a"], a["b"]) if pr.sdf_body == 0 else (a["b"], a["a"])
        a["sdf_is_a"] = pr.sdf_body == 0
        a["grid"] = generate_sdf(a["sdf"], SdfResolutionSpec(resolution, 4))
    asset = np.arange(n_envs) % len(assets)
    sdf_pose = np.tile(IDENTITY_POSE7, (n_envs, 1))
    mesh_pose = np.tile(IDENTITY_POSE7, (n_envs, 1))
    for k, a in enumerate(assets):
        idx = np.nonzero(asset == k)[0]
        if a["kind"] == "peg":
            p = _peg_poses(rng, len(idx), a["clearance"], a["depth"])
        else:
            p = nut_poses(len(idx), int(rng.integers(1 << 30)), a["pitch"], a["z0"])
            scale = a["pitch"] / 0.002  # nut_poses' offsets are for the M16 pitch
            p[:, 0:2] *= scale
            p[:, 2] = a["z0"] + (p[:, 2] - a["z0"]) * scale
        # the moving part (peg / nut) carries the pose; the other stays at the identity
        moving_is_a = a["kind"] == "peg"
        if moving_is_a == a["sdf_is_a"]:
            sdf_pose[idx] = p
        else:
            mesh_pose[idx] = p
    cd = np.array([2.0 * assets[k]["grid"].voxel_size for k in asset])  # scene.py:206
    return {"assets": assets, "asset": asset, "sdf_pose": sdf_pose, "mesh_pose": mesh_pose, "cd": cd}
