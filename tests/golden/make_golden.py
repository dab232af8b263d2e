"""Generate the golden fixtures under tests/golden/ by running the REFERENCE.

Run here (the build container), never on the GPU box:

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

It imports the reference package `contactsim` (read-only, /root/reference/pkg/src)
and records its outputs for the hot path on seeded inputs:

* meshes.npz        M16 nut/bolt (80 seg/turn) and a 4 mm peg/hole, exactly as
                    `generate_iso_thread` / `generate_peg_hole` build them
                    (pkg/src/contactsim/geometry/threads.py:139,193).
* grid_bolt_r64.npz the bolt SDF at SdfResolutionSpec(64, 4) (grid.py:163).
* grids.json        dims/origin/voxel/aabb + sha256 of the float32 values for the
                    bolt at res 64/128/256 and the peg at res 64 (pins GPU SDF generation).
* poses.npz         the SURVEY §8(d) seeded pose distribution, seed 0, 64 envs.
* gen_r{64,256}.npz per env: generate_contacts() output (generation.py:54) and the
                    sha256 of its internal tri_verts; reduce_contacts() patches
                    (reduction.py:45) with the Scene's parameters (scene.py:206-226).
* red_synth.npz     reduce_contacts() on synthetic candidate sets with non-default
                    ReductionParams (eviction, small batches, caps, cones, min_depth).
* sdf_query.npz     SignedDistanceGrid.sample / gradient (grid.py:78,93) at random points.
* kat.npz           SPEC known-answer cases (sphere-plane, coplanar, +/-Z).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from contactsim.contacts import generation as ref_gen  # noqa: E402
from contactsim.contacts.generation import assign_roles, BodyShape, generate_contacts  # noqa: E402
from contactsim.contacts.reduction import reduce_contacts  # noqa: E402
from contactsim.contacts.types import ContactSet, ReductionParams  # noqa: E402
from contactsim.geometry.shapes import make_box, make_icosphere  # noqa: E402
from contactsim.geometry.threads import (  # noqa: E402
    ThreadSpec,
    bolt_thread_base_z,
    generate_iso_thread,
    generate_peg_hole,
)
from contactsim.math3d import Transform, quat_from_axis_angle, quat_multiply  # noqa: E402
from contactsim.sdf.grid import SdfResolutionSpec, SignedDistanceGrid, generate_sdf  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def grid_meta(g: SignedDistanceGrid) -> dict:
    return {
        "dims": list(g.dims),
        "origin": [float(x) for x in g.origin],
        "voxel": float(g.voxel_size),
        "aabb_lo": [float(x) for x in g.mesh_aabb[0]],
        "aabb_hi": [float(x) for x in g.mesh_aabb[1]],
        "sha256": sha(g.values),
    }


def nut_poses(n: int, seed: int, pitch: float, z0: float) -> np.ndarray:
    """yaw, axis, tilt, k, dz, dx, dy drawn per env in this order."""
    rng = np.random.default_rng(seed)
    out = np.zeros((n, 7))
    for e in range(n):
        yaw = rng.uniform(0.0, 2.0 * np.pi)
        axis = rng.normal(size=3)
        tilt = rng.uniform(0.0, 0.01)
        k = int(rng.integers(0, 3))
        dz = rng.uniform(-6e-4, -2e-4)
        dx = rng.uniform(-1e-4, 1e-4)
        dy = rng.uniform(-1e-4, 1e-4)
        q = quat_multiply(quat_from_axis_angle(axis, tilt), quat_from_axis_angle(np.array([0.0, 0.0, 1.0]), yaw))
        out[e, :3] = (dx, dy, z0 + pitch * (k + yaw / (2.0 * np.pi)) + dz)
        out[e, 3:] = q
    return out


def pack_contactset(cs: ContactSet) -> dict:
    return {
        "points": cs.points,
        "normals": cs.normals,
        "depths": cs.depths,
        "faces": cs.face_indices,
    }


def pack_patches(patches, cap: int) -> dict:
    P = len(patches)
    rep = np.zeros((P, 3))
    nkept = np.zeros(P, np.int64)
    kept_members = np.full((P, max(cap, 1)), -1, np.int64)  # candidate indices of kept contacts
    kept_points = np.zeros((P, max(cap, 1), 3))
    kept_normals = np.zeros((P, max(cap, 1), 3))
    kept_depths = np.zeros((P, max(cap, 1)))
    kept_faces = np.full((P, max(cap, 1)), -1, np.int64)
    moff = [0]
    members = []
    wsum = np.zeros(P)
    wp = np.zeros((P, 3))
    wn = np.zeros((P, 3))
    wt = np.zeros((P, 3))
    area = np.zeros(P)
    maxd = np.zeros(P)
    for i, p in enumerate(patches):
        rep[i] = p.representative_normal
        k = len(p)
        nkept[i] = k
        kept_points[i, :k] = p.points
        kept_normals[i, :k] = p.normals
        kept_depths[i, :k] = p.depths
        kept_faces[i, :k] = p.face_indices
        members.extend(p.member_indices.tolist())
        moff.append(len(members))
        wsum[i] = p.weight_sum
        wp[i] = p.weighted_point_sum
        wn[i] = p.weighted_normal_sum
        wt[i] = p.weighted_torque_sum
        area[i] = p.area_metric
        maxd[i] = p.max_depth
    return {
        "rep": rep, "nkept": nkept, "kept_points": kept_points, "kept_normals": kept_normals,
        "kept_depths": kept_depths, "kept_faces": kept_faces,
        "member_offsets": np.array(moff, np.int64), "members": np.array(members, np.int64),
        "wsum": wsum, "wp": wp, "wn": wn, "wt": wt, "area": area, "maxd": maxd,
    }


def flatten(prefix: str, d: dict, out: dict) -> None:
    for k, v in d.items():
        out[f"{prefix}{k}"] = np.asarray(v)


def capture_tri_verts(grid, mesh, sdf_pose, mesh_pose):
    """sha256 of the tri_verts array the reference hands to face_contacts."""
    to_grid = sdf_pose.inverse().compose(mesh_pose)
    verts_grid = to_grid.apply(mesh.vertices)
    tri_verts = np.ascontiguousarray(verts_grid[mesh.triangles])
    return sha(tri_verts), to_grid


def main() -> None:
    t0 = time.time()
    nut_spec = ThreadSpec.standard("M16", "nut", "tight", segments_per_turn=80)
    bolt_spec = ThreadSpec.standard("M16", "bolt", "tight", segments_per_turn=80)
    nut = generate_iso_thread(nut_spec)
    bolt = generate_iso_thread(bolt_spec)
    peg, hole = generate_peg_hole(0.004, 0.104e-3, 0.03)
    np.savez_compressed(
        os.path.join(OUT, "meshes.npz"),
        nut_v=nut.vertices, nut_t=nut.triangles, bolt_v=bolt.vertices, bolt_t=bolt.triangles,
        peg_v=peg.vertices, peg_t=peg.triangles, hole_v=hole.vertices, hole_t=hole.triangles,
    )
    print("meshes", nut.vertices.shape, bolt.vertices.shape, peg.vertices.shape, hole.vertices.shape)

    grids = {}
    meta = {}
    for res in (64, 128, 256):
        t = time.time()
        g = generate_sdf(bolt, SdfResolutionSpec(res, 4))
        grids[res] = g
        meta[f"bolt_r{res}"] = grid_meta(g)
        print("bolt grid", res, g.dims, f"{time.time() - t:.1f}s")
    gp = generate_sdf(peg, SdfResolutionSpec(64, 4))
    meta["peg_r64"] = grid_meta(gp)
    g64 = grids[64]
    np.savez_compressed(
        os.path.join(OUT, "grid_bolt_r64.npz"),
        values=g64.values, dims=np.array(g64.dims), origin=g64.origin, voxel=np.array(g64.voxel_size),
        aabb_lo=g64.mesh_aabb[0], aabb_hi=g64.mesh_aabb[1],
    )
    np.savez_compressed(
        os.path.join(OUT, "grid_peg_r64.npz"),
        values=gp.values, dims=np.array(gp.dims), origin=gp.origin, voxel=np.array(gp.voxel_size),
        aabb_lo=gp.mesh_aabb[0], aabb_hi=gp.mesh_aabb[1],
    )

    pitch = bolt_spec.pitch
    z0 = float(bolt_thread_base_z(bolt_spec))
    poses = nut_poses(64, 0, pitch, z0)
    np.savez_compressed(os.path.join(OUT, "poses.npz"), nut_pose=poses, pitch=pitch, z0=z0)

    # sdf is the bolt (more triangles, both opted in) -> SCENE rule (generation.py:32-51)
    pairing = assign_roles(BodyShape(0, len(bolt), True), BodyShape(1, len(nut), True))
    assert pairing.sdf_body == 0 and pairing.mesh_body == 1, pairing

    # a non-identity SDF pose for a couple of envs exercises the world-frame epilogue
    sdf_q = quat_from_axis_angle(np.array([0.3, -0.5, 0.8]), 0.7)
    sdf_p = np.array([0.01, -0.02, 0.005])

    for res, envs in ((64, range(6)), (256, range(3))):
        g = grids[res]
        cd = 2.0 * g.voxel_size
        rp = ReductionParams(min_depth=-cd)
        out = {"cd": np.array(cd), "envs": np.array(list(envs))}
        for e in envs:
            moved_sdf = (e % 3 == 2)
            if moved_sdf:
                spose7 = np.concatenate([sdf_p, sdf_q])
                mpose_local = Transform.from_pose(poses[e, :3], poses[e, 3:])
                sp = Transform.from_pose(spose7[:3], spose7[3:])
                # nut placed relative to the moved bolt: world = sp ∘ local; the
                # reference consumes (position, wxyz) so store the composed pose.
                comp = sp.compose(mpose_local)
                from contactsim.math3d import matrix_to_quat
                mpose7 = np.concatenate([comp.translation, matrix_to_quat(comp.rotation)])
            else:
                spose7 = np.array([0, 0, 0, 1.0, 0, 0, 0])
                mpose7 = poses[e]
            sdf_pose = Transform.from_pose(spose7[:3], spose7[3:])
            mesh_pose = Transform.from_pose(mpose7[:3], mpose7[3:])
            tv_sha, _ = capture_tri_verts(g, nut, sdf_pose, mesh_pose)
            t = time.time()
            cs = generate_contacts(pairing, g, nut, sdf_pose, mesh_pose, cd)
            t1 = time.time()
            patches = reduce_contacts(cs, rp)
            t2 = time.time()
            print(f"res {res} env {e}: {len(cs)} cands -> {len(patches)} patches, "
                  f"{sum(len(p) for p in patches)} kept  gen {t1 - t:.3f}s red {t2 - t1:.3f}s")
            pre = f"e{e}_"
            out[pre + "sdf_pose"] = spose7
            out[pre + "mesh_pose"] = mpose7
            out[pre + "tri_verts_sha"] = np.array(tv_sha)
            flatten(pre + "cs_", pack_contactset(cs), out)
            flatten(pre + "pt_", pack_patches(patches, rp.per_patch_cap), out)
        np.savez_compressed(os.path.join(OUT, f"gen_r{res}.npz"), **out)

    # ------------------------------------------------------------------ synthetic reduction cases
    rng = np.random.default_rng(1234)
    synth = {}
    cases = []
    # (n, params, normal-spread, point-dup fraction)
    specs = [
        (300, dict(), 1.0, 0.0),
        (3000, dict(), 0.4, 0.3),
        (2500, dict(max_patches=4), 1.0, 0.2),          # eviction + fold
        (1200, dict(max_patches=2, per_patch_cap=3), 1.0, 0.0),
        (800, dict(max_patches=1), 1.0, 0.0),
        (900, dict(batch_size=7), 0.6, 0.2),
        (700, dict(batch_size=1, max_patches=6), 1.0, 0.1),
        (1500, dict(per_patch_cap=1), 0.5, 0.5),
        (1500, dict(per_patch_cap=9, normal_cone_cos=float(np.cos(np.radians(40)))), 0.8, 0.4),
        (1000, dict(normal_cone_cos=float(np.cos(np.radians(3)))), 0.1, 0.0),
        (2000, dict(min_depth=-1e-4), 0.5, 0.3),
        (5, dict(), 1.0, 0.0),
        (1, dict(), 1.0, 0.0),
        (2, dict(batch_size=1), 1.0, 0.0),
        (4000, dict(max_patches=3, batch_size=512), 1.0, 0.3),
        (600, dict(normal_cone_cos=-1.0), 1.0, 0.0),
        (600, dict(normal_cone_cos=1.0), 0.05, 0.0),
    ]
    for ci, (n, kw, spread, dup) in enumerate(specs):
        pts = rng.normal(size=(n, 3)) * 1e-3
        # planar-ish clusters so hulls are non-trivial, with exact duplicate points
        if dup > 0 and n > 4:
            ndup = int(dup * n)
            src = rng.integers(0, n, size=ndup)
            dst = rng.integers(0, n, size=ndup)
            pts[dst] = pts[src]
        base = np.array([0.0, 0.0, 1.0])
        nrm = base + spread * rng.normal(size=(n, 3))
        nrm /= np.linalg.norm(nrm, axis=1)[:, None]
        depths = rng.normal(size=n) * 2e-4
        # exact depth ties between duplicates, like shared mesh vertices
        if n > 10:
            tie = rng.integers(0, n, size=n // 5)
            depths[tie] = depths[tie[0]]
        faces = np.arange(n) * 3 + 1
        cs = ContactSet(pts, nrm, depths, faces, 0, 1)
        rp = ReductionParams(**kw)
        patches = reduce_contacts(cs, rp)
        pre = f"c{ci}_"
        synth[pre + "params"] = np.array([rp.max_patches, rp.per_patch_cap, rp.normal_cone_cos,
                                          np.nan if rp.min_depth is None else rp.min_depth, rp.batch_size])
        flatten(pre + "cs_", pack_contactset(cs), synth)
        flatten(pre + "pt_", pack_patches(patches, rp.per_patch_cap), synth)
        cases.append(ci)
        print(f"synth {ci}: n={n} {kw} -> {len(patches)} patches")
    synth["cases"] = np.array(cases)
    np.savez_compressed(os.path.join(OUT, "red_synth.npz"), **synth)

    # ------------------------------------------------------------------ SDF point queries
    q = {}
    lo = g64.origin - 3 * g64.voxel_size
    hi = g64.origin + (np.array(g64.dims) + 2) * g64.voxel_size
    P = lo + rng.random((4000, 3)) * (hi - lo)
    P[:64] = g64.node_points()[rng.integers(0, len(g64.values), 64)]  # exact nodes
    q["points"] = P
    q["sample"] = g64.sample(P)
    q["gradient"] = g64.gradient(P, normalize=False)
    q["gradient_n"] = g64.gradient(P)
    pose = Transform.from_pose(np.array([0.001, 0.002, -0.003]), quat_from_axis_angle(np.array([1.0, 2.0, 3.0]), 0.4))
    q["pose7"] = np.concatenate([pose.translation, quat_from_axis_angle(np.array([1.0, 2.0, 3.0]), 0.4)])
    q["sample_posed"] = g64.sample(P, pose)
    q["gradient_posed"] = g64.gradient(P, pose)
    np.savez_compressed(os.path.join(OUT, "sdf_query.npz"), **q)

    # ------------------------------------------------------------------ SPEC known answers
    kat = {}
    sphere = make_icosphere(0.01, subdivisions=3)
    gs = generate_sdf(sphere, SdfResolutionSpec(48, 4))
    plane = make_box((0.05, 0.05, 0.004), subdivisions=12)
    kat["sphere_values"] = gs.values
    kat["sphere_dims"] = np.array(gs.dims)
    kat["sphere_origin"] = gs.origin
    kat["sphere_voxel"] = np.array(gs.voxel_size)
    kat["sphere_aabb_lo"] = gs.mesh_aabb[0]
    kat["sphere_aabb_hi"] = gs.mesh_aabb[1]
    kat["plane_v"] = plane.vertices
    kat["plane_t"] = plane.triangles
    pairing_sp = assign_roles(BodyShape(0, len(sphere), True), BodyShape(1, len(plane), False))
    for j, d in enumerate([0.1e-3, 0.5e-3, 1.0e-3, -2e-3]):
        # plane top face at z = 0.002 in its frame; place it so it overlaps the sphere by d
        mp = np.array([0.0, 0.0, -0.01 - 0.002 + d, 1.0, 0.0, 0.0, 0.0])
        sp = np.array([0.0, 0.0, 0.0, 1.0, 0.0, 0.0, 0.0])
        cd = 2.0 * gs.voxel_size
        cs = generate_contacts(pairing_sp, gs, plane, Transform.from_pose(sp[:3], sp[3:]),
                               Transform.from_pose(mp[:3], mp[3:]), cd)
        patches = reduce_contacts(cs, ReductionParams(min_depth=-cd))
        kat[f"sp{j}_mesh_pose"] = mp
        kat[f"sp{j}_cd"] = np.array(cd)
        flatten(f"sp{j}_cs_", pack_contactset(cs), kat)
        flatten(f"sp{j}_pt_", pack_patches(patches, 6), kat)
        print(f"sphere-plane d={d}: {len(cs)} candidates, {len(patches)} patches")
    np.savez_compressed(os.path.join(OUT, "kat.npz"), **kat)

    with open(os.path.join(OUT, "grids.json"), "w") as fh:
        json.dump(meta, fh, indent=1)
    print(f"done in {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
