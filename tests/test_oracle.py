"""Pin the oracle (oracle/cs_oracle.c) bit-for-bit against the reference's own
outputs (tests/golden, produced by tests/golden/make_golden.py). CPU only."""

import hashlib

import numpy as np
import pytest

from conftest import CS_KEYS, PATCH_KEYS, assert_same
from oracle import oracle as O


def test_sdf_queries_match_reference(grid64_npz, sdf_query):
    g = O.Grid.from_npz(grid64_npz)
    assert np.array_equal(O.sample(g, sdf_query["points"]), sdf_query["sample"])
    assert np.array_equal(O.gradient(g, sdf_query["points"]), sdf_query["gradient"])


def test_node_samples_are_stored_values(grid64_npz):
    g = O.Grid.from_npz(grid64_npz)
    nx, ny, nz = g.dims
    rng = np.random.default_rng(3)
    idx = rng.integers(0, [nx, ny, nz], size=(500, 3))
    pts = g.origin + idx * g.voxel
    flat = idx[:, 0] + nx * (idx[:, 1] + ny * idx[:, 2])
    # (p - o) / voxel lands within an ulp of the node index, so the lerp weights are ~1e-16
    np.testing.assert_allclose(O.sample(g, pts), g.values[flat].astype(np.float64), rtol=0, atol=1e-12)


def test_tri_verts_match_reference(meshes, gen64):
    for e in gen64["envs"]:
        tv = O.tri_verts(gen64[f"e{e}_sdf_pose"], gen64[f"e{e}_mesh_pose"], meshes["nut_v"], meshes["nut_t"])
        assert hashlib.sha256(tv.tobytes()).hexdigest() == str(gen64[f"e{e}_tri_verts_sha"])


@pytest.mark.parametrize("e", range(6))
def test_generate_contacts_r64(e, meshes, grid64_npz, gen64):
    g = O.Grid.from_npz(grid64_npz)
    cs = O.generate_contacts(g, meshes["nut_v"], meshes["nut_t"], gen64[f"e{e}_sdf_pose"], gen64[f"e{e}_mesh_pose"],
                             float(gen64["cd"]))
    assert_same(cs, gen64, f"e{e}_cs_", CS_KEYS, f"env {e} ")


@pytest.mark.parametrize("e", range(6))
def test_reduce_contacts_r64(e, gen64):
    pre = f"e{e}_"
    r = O.reduce_contacts(gen64[pre + "cs_points"], gen64[pre + "cs_normals"], gen64[pre + "cs_depths"],
                          gen64[pre + "cs_faces"], min_depth=-float(gen64["cd"]))
    assert_same(r, gen64, pre + "pt_", PATCH_KEYS, f"env {e} ")


def test_reduce_contacts_synthetic(synth):
    for c in synth["cases"]:
        pre = f"c{c}_"
        N, K, cone, md, bs = synth[pre + "params"]
        r = O.reduce_contacts(synth[pre + "cs_points"], synth[pre + "cs_normals"], synth[pre + "cs_depths"],
                              synth[pre + "cs_faces"], max_patches=int(N), per_patch_cap=int(K), normal_cone_cos=cone,
                              min_depth=None if np.isnan(md) else md, batch_size=int(bs))
        assert_same(r, synth, pre + "pt_", PATCH_KEYS, f"case {c} ")


def test_reduce_contacts_merge_branch(merge):
    """The merge branch of _add_patch (reduction.py:99-105): the reference took it in every case."""
    for c in merge["cases"]:
        assert int(merge[f"c{c}_merges"]) >= 1
        pre = f"c{c}_"
        N, K, cone, md, bs = merge[pre + "params"]
        r = O.reduce_contacts(merge[pre + "cs_points"], merge[pre + "cs_normals"], merge[pre + "cs_depths"],
                              merge[pre + "cs_faces"], max_patches=int(N), per_patch_cap=int(K), normal_cone_cos=cone,
                              min_depth=None if np.isnan(md) else md, batch_size=int(bs))
        assert_same(r, merge, pre + "pt_", PATCH_KEYS, f"case {c} ")


def test_reduce_contacts_nan_inputs(nan_cases):
    """NaN coordinates, normals and depths follow numpy's rules (NaN last in lexsort,
    `cross <= 0` false on NaN, first-NaN argmax, NaN sums) as the reference ran them."""
    for c in nan_cases["cases"]:
        pre = f"c{c}_"
        N, K, cone, md, bs = nan_cases[pre + "params"]
        r = O.reduce_contacts(nan_cases[pre + "cs_points"], nan_cases[pre + "cs_normals"], nan_cases[pre + "cs_depths"],
                              nan_cases[pre + "cs_faces"], max_patches=int(N), per_patch_cap=int(K),
                              normal_cone_cos=cone, min_depth=None if np.isnan(md) else md, batch_size=int(bs))
        assert_same(r, nan_cases, pre + "pt_", PATCH_KEYS, f"case {c} ")


def test_generate_reduce_on_nan_grid(nan_cases, meshes, grid64_npz):
    """A grid with NaN nodes: NaN samples make no contact, NaN gradients make NaN normals
    that seed patches up to the cap (eviction), as the reference ran it."""
    g = O.Grid.from_npz(grid64_npz)
    vals = g.values.copy()
    vals[nan_cases["g_bad"]] = np.nan
    g.values = vals
    cd = float(nan_cases["g_cd"])
    for e in nan_cases["g_envs"]:
        pre = f"ge{e}_"
        cs = O.generate_contacts(g, meshes["nut_v"], meshes["nut_t"], nan_cases[pre + "sdf_pose"],
                                 nan_cases[pre + "mesh_pose"], cd)
        assert_same(cs, nan_cases, pre + "cs_", CS_KEYS, f"env {e} ")
        r = O.reduce_contacts(cs["points"], cs["normals"], cs["depths"], cs["faces"], min_depth=-cd)
        assert_same(r, nan_cases, pre + "pt_", PATCH_KEYS, f"env {e} ")


def test_sphere_plane_known_answers(kat):
    g = O.Grid(kat["sphere_values"], kat["sphere_dims"], kat["sphere_origin"], float(kat["sphere_voxel"]),
               kat["sphere_aabb_lo"], kat["sphere_aabb_hi"])
    for j in range(4):
        cs = O.generate_contacts(g, kat["plane_v"], kat["plane_t"], [0, 0, 0, 1.0, 0, 0, 0], kat[f"sp{j}_mesh_pose"],
                                 float(kat[f"sp{j}_cd"]))
        assert_same(cs, kat, f"sp{j}_cs_", CS_KEYS, f"sphere-plane {j} ")
        r = O.reduce_contacts(cs["points"], cs["normals"], cs["depths"], cs["faces"], min_depth=-float(kat[f"sp{j}_cd"]))
        assert_same(r, kat, f"sp{j}_pt_", PATCH_KEYS, f"sphere-plane {j} ")
    # SPEC: separated pair -> no contacts; overlapping -> depth within 2 voxels of the overlap
    assert len(kat["sp3_cs_depths"]) == 0
    vox = float(kat["sphere_voxel"])
    for j, d in enumerate([0.1e-3, 0.5e-3, 1.0e-3]):
        assert abs(kat[f"sp{j}_cs_depths"].max() - d) <= 2 * vox


def test_face_contacts_dropin_is_generate_kernel(meshes, grid64_npz, gen64):
    """og_face_contacts fed the reference's tri_verts reproduces generate_contacts' found set."""
    g = O.Grid.from_npz(grid64_npz)
    tv = O.tri_verts(gen64["e0_sdf_pose"], gen64["e0_mesh_pose"], meshes["nut_v"], meshes["nut_t"])
    _, phi, _, found = O.face_contacts(g, tv, float(gen64["cd"]))
    faces = np.nonzero(found)[0]
    # culled faces are never found: every golden face is in the kernel's found set
    assert set(gen64["e0_cs_faces"].tolist()) <= set(faces.tolist())
    assert np.array_equal(-phi[gen64["e0_cs_faces"]], gen64["e0_cs_depths"])


def test_batched_collide_stats(meshes, grid64_npz, gen64):
    g = O.Grid.from_npz(grid64_npz)
    envs = [0, 1, 3, 4]
    s7 = np.stack([gen64[f"e{e}_sdf_pose"] for e in envs])
    m7 = np.stack([gen64[f"e{e}_mesh_pose"] for e in envs])
    st = O.collide_batched(g, meshes["nut_v"], meshes["nut_t"], s7, m7, float(gen64["cd"]))
    for row, e in zip(st, envs):
        assert row[0] == len(gen64[f"e{e}_cs_depths"])
        assert row[1] == len(gen64[f"e{e}_pt_nkept"])
        assert row[2] == gen64[f"e{e}_pt_nkept"].sum()


def test_env_digest_matches_oracle_word_stream(meshes, grid64_npz, gen64):
    """tests/conftest.py:digest_env (applied to the GPU outputs by the full-size parity
    tests) and the oracle's og_collide_digest hash the same word stream."""
    from conftest import digest_env

    og = O.Grid.from_npz(grid64_npz)
    cd = float(gen64["cd"])
    envs = list(gen64["envs"])
    sp = np.stack([gen64[f"e{e}_sdf_pose"] for e in envs])
    mp = np.stack([gen64[f"e{e}_mesh_pose"] for e in envs])
    ref = O.collide_digest(og, meshes["nut_v"], meshes["nut_t"], sp, mp, cd)
    for i in range(len(envs)):
        g = O.generate_contacts(og, meshes["nut_v"], meshes["nut_t"], sp[i], mp[i], cd)
        r = O.reduce_contacts(g["points"], g["normals"], g["depths"], g["faces"], min_depth=-cd)
        d = digest_env(g["points"], g["normals"], g["depths"], g["faces"], r["rep"], r["nkept"], r["kept"],
                       r["member_offsets"], r["members"], r["wsum"], r["wp"], r["wn"], r["wt"], r["area"], r["maxd"])
        assert d == int(ref[i]), i
