"""GPU parity: the sm_100a path (through libcontactsim_b200.so) against the
reference's golden outputs and the pinned oracle. Bit-exact, no exclusions:
the kernels reproduce the reference's IEEE operation order and its BLAS FMA
patterns."""

import hashlib
import json
import os

import numpy as np
import pytest

from conftest import CS_KEYS, GOLDEN, PATCH_KEYS, assert_same, env_digests, pack_patch_list

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def P():
    import paper_2205_03532_b200 as P
    from paper_2205_03532_b200 import _native

    _native.lib()  # fails loudly without the library / a GPU
    return P


@pytest.fixture(scope="module")
def grid64(P, grid64_npz):
    d = grid64_npz
    return P.SignedDistanceGrid(d["origin"], float(d["voxel"]), d["dims"], d["values"], (d["aabb_lo"], d["aabb_hi"]))


@pytest.fixture(scope="module")
def nut(P, meshes):
    return P.TriMesh(meshes["nut_v"], meshes["nut_t"])


@pytest.fixture(scope="module")
def bolt(P, meshes):
    return P.TriMesh(meshes["bolt_v"], meshes["bolt_t"])


def _tf(P, pose7):
    return P.Transform.from_pose(pose7[:3], pose7[3:])


def test_library_loaded(P):
    from paper_2205_03532_b200 import _native

    assert _native.lib().cs_abi_version() == 1


def test_sdf_sample_gradient(P, grid64, sdf_query):
    q = sdf_query
    assert np.array_equal(grid64.sample(q["points"]), q["sample"])
    assert np.array_equal(grid64.gradient(q["points"], normalize=False), q["gradient"])
    assert np.array_equal(grid64.gradient(q["points"]), q["gradient_n"])
    pose = _tf(P, q["pose7"])
    np.testing.assert_array_equal(grid64.sample(q["points"], pose), q["sample_posed"])
    np.testing.assert_array_equal(grid64.gradient(q["points"], pose), q["gradient_posed"])


def test_face_contacts_dropin_bitexact(P, grid64, grid64_npz, meshes, gen64):
    """Stage 1a: cs_face_contacts fed the reference's tri_verts == numba kernel output."""
    from oracle import oracle as O

    g = O.Grid.from_npz(grid64_npz)
    for e in gen64["envs"]:
        tv = O.tri_verts(gen64[f"e{e}_sdf_pose"], gen64[f"e{e}_mesh_pose"], meshes["nut_v"], meshes["nut_t"])
        assert hashlib.sha256(tv.tobytes()).hexdigest() == str(gen64[f"e{e}_tri_verts_sha"])
        cd = float(gen64["cd"])
        op, ophi, ogr, ofd = O.face_contacts(g, tv, cd)
        m = len(tv)
        d_tv = torch.from_numpy(tv).cuda()
        outs = [torch.zeros((m, 3), dtype=torch.float64, device="cuda"), torch.zeros(m, dtype=torch.float64, device="cuda"),
                torch.zeros((m, 3), dtype=torch.float64, device="cuda"), torch.full((m,), 7, dtype=torch.uint8, device="cuda")]
        vals = torch.from_numpy(grid64_npz["values"]).cuda()
        nx, ny, nz = g.dims
        P.contacts.face_contacts(vals, nx, ny, nz, *g.origin, g.voxel, d_tv, cd, 12, 0.1 * g.voxel, *outs)
        gp, gphi, ggr, gfd = (t.cpu().numpy() for t in outs)
        assert np.array_equal(gfd, ofd), f"env {e}: found flags differ"
        # both sides zero-initialise, and pruned faces leave point/phi/grad untouched
        assert np.array_equal(gp, op) and np.array_equal(gphi, ophi) and np.array_equal(ggr, ogr)


@pytest.mark.parametrize("e", range(6))
def test_generate_contacts_r64(P, grid64, nut, gen64, e):
    pairing = P.CollisionPairing(0, 1)
    cs = P.generate_contacts(pairing, grid64, nut, _tf(P, gen64[f"e{e}_sdf_pose"]), _tf(P, gen64[f"e{e}_mesh_pose"]),
                             float(gen64["cd"]))
    got = {"points": cs.points, "normals": cs.normals, "depths": cs.depths, "faces": cs.face_indices}
    assert_same(got, gen64, f"e{e}_cs_", CS_KEYS, f"env {e} ")


@pytest.mark.parametrize("e", range(6))
def test_reduce_contacts_r64(P, gen64, e):
    pre = f"e{e}_"
    cs = P.ContactSet(gen64[pre + "cs_points"], gen64[pre + "cs_normals"], gen64[pre + "cs_depths"],
                      gen64[pre + "cs_faces"], 0, 1)
    patches = P.reduce_contacts(cs, P.ReductionParams(min_depth=-float(gen64["cd"])))
    assert_same(pack_patch_list(patches, 6), gen64, pre + "pt_", PATCH_KEYS, f"env {e} ")


def test_reduce_contacts_synthetic(P, synth):
    """Eviction + fold, batch sizes 1 / 7 / 512, caps 1..9, cones, min_depth."""
    for c in synth["cases"]:
        pre = f"c{c}_"
        N, K, cone, md, bs = synth[pre + "params"]
        cs = P.ContactSet(synth[pre + "cs_points"], synth[pre + "cs_normals"], synth[pre + "cs_depths"],
                          synth[pre + "cs_faces"], 0, 1)
        rp = P.ReductionParams(int(N), int(K), float(cone), None if np.isnan(md) else float(md), int(bs))
        patches = P.reduce_contacts(cs, rp)
        assert_same(pack_patch_list(patches, int(K)), synth, pre + "pt_", PATCH_KEYS, f"case {c} ")


def test_reduce_contacts_merge_branch(P, merge):
    """The merge branch of _add_patch (reduction.py:99-105): gemm/gemv cosines one ulp apart at the cone."""
    for c in merge["cases"]:
        pre = f"c{c}_"
        N, K, cone, md, bs = merge[pre + "params"]
        cs = P.ContactSet(merge[pre + "cs_points"], merge[pre + "cs_normals"], merge[pre + "cs_depths"],
                          merge[pre + "cs_faces"], 0, 1)
        rp = P.ReductionParams(int(N), int(K), float(cone), None if np.isnan(md) else float(md), int(bs))
        patches = P.reduce_contacts(cs, rp)
        assert_same(pack_patch_list(patches, int(K)), merge, pre + "pt_", PATCH_KEYS, f"case {c} ")


def test_reduce_contacts_nan_inputs(P, nan_cases):
    """NaN points, normals and depths: numpy's NaN rules, as the reference ran them."""
    for c in nan_cases["cases"]:
        pre = f"c{c}_"
        N, K, cone, md, bs = nan_cases[pre + "params"]
        cs = P.ContactSet(nan_cases[pre + "cs_points"], nan_cases[pre + "cs_normals"], nan_cases[pre + "cs_depths"],
                          nan_cases[pre + "cs_faces"], 0, 1)
        rp = P.ReductionParams(int(N), int(K), float(cone), None if np.isnan(md) else float(md), int(bs))
        patches = P.reduce_contacts(cs, rp)
        assert_same(pack_patch_list(patches, int(K)), nan_cases, pre + "pt_", PATCH_KEYS, f"case {c} ")


def test_collide_on_nan_grid(P, nan_cases, grid64_npz, nut):
    """A grid holding NaN nodes (no face bound for it; NaN normals reach the reduction
    and seed patches up to the cap): batched collide against the reference's outputs."""
    d = grid64_npz
    vals = d["values"].astype(np.float32).copy()
    vals[nan_cases["g_bad"]] = np.nan
    grid = P.SignedDistanceGrid(d["origin"], float(d["voxel"]), d["dims"], vals, (d["aabb_lo"], d["aabb_hi"]))
    envs = list(nan_cases["g_envs"])
    E = len(envs)
    cd = float(nan_cases["g_cd"])
    sp = np.stack([nan_cases[f"ge{e}_sdf_pose"] for e in envs])
    mp = np.stack([nan_cases[f"ge{e}_mesh_pose"] for e in envs])
    res = P.collide([P.register_sdf(grid)] * E, [P.register_mesh(nut)] * E, sp, mp, np.full(E, cd))
    for i, e in enumerate(envs):
        cs = res.contact_set(i)
        got = {"points": cs.points, "normals": cs.normals, "depths": cs.depths, "faces": cs.face_indices}
        assert_same(got, nan_cases, f"ge{e}_cs_", CS_KEYS, f"env {e} ")
        assert_same(pack_patch_list(res.patches(i), 6), nan_cases, f"ge{e}_pt_", PATCH_KEYS, f"env {e} ")


def test_batched_collide_r64(P, grid64, nut, gen64):
    """All six golden envs (two with a moved SDF pose) in one collide call."""
    envs = list(gen64["envs"])
    E = len(envs)
    h_sdf = [P.register_sdf(grid64)] * E
    h_mesh = [P.register_mesh(nut)] * E
    sp = np.stack([gen64[f"e{e}_sdf_pose"] for e in envs])
    mp = np.stack([gen64[f"e{e}_mesh_pose"] for e in envs])
    res = P.collide(h_sdf, h_mesh, sp, mp, np.full(E, float(gen64["cd"])))
    for i, e in enumerate(envs):
        cs = res.contact_set(i)
        got = {"points": cs.points, "normals": cs.normals, "depths": cs.depths, "faces": cs.face_indices}
        assert_same(got, gen64, f"e{e}_cs_", CS_KEYS, f"env {e} ")
        assert_same(pack_patch_list(res.patches(i), 6), gen64, f"e{e}_pt_", PATCH_KEYS, f"env {e} ")


def test_sphere_plane_known_answers(P, kat):
    g = P.SignedDistanceGrid(kat["sphere_origin"], float(kat["sphere_voxel"]), kat["sphere_dims"], kat["sphere_values"],
                             (kat["sphere_aabb_lo"], kat["sphere_aabb_hi"]))
    plane = P.TriMesh(kat["plane_v"], kat["plane_t"])
    for j in range(4):
        cd = float(kat[f"sp{j}_cd"])
        cs = P.generate_contacts(P.CollisionPairing(0, 1), g, plane, P.Transform(), _tf(P, kat[f"sp{j}_mesh_pose"]), cd)
        got = {"points": cs.points, "normals": cs.normals, "depths": cs.depths, "faces": cs.face_indices}
        assert_same(got, kat, f"sp{j}_cs_", CS_KEYS, f"sphere-plane {j} ")
        patches = P.reduce_contacts(cs, P.ReductionParams(min_depth=-cd))
        assert_same(pack_patch_list(patches, 6), kat, f"sp{j}_pt_", PATCH_KEYS, f"sphere-plane {j} ")


def test_gpu_sdf_generation_matches_reference(P, bolt, meshes):
    """cs_sdf_generate reproduces the reference's generate_sdf grids bit for bit."""
    meta = json.load(open(os.path.join(GOLDEN, "grids.json")))
    for res in (64, 128, 256):
        g = P.generate_sdf(bolt, P.SdfResolutionSpec(res, 4))
        m = meta[f"bolt_r{res}"]
        assert list(g.dims) == m["dims"]
        assert g.voxel_size == m["voxel"] and list(g.origin) == m["origin"]
        assert hashlib.sha256(g.values.tobytes()).hexdigest() == m["sha256"], f"res {res} grid differs"
    peg = P.TriMesh(meshes["peg_v"], meshes["peg_t"])
    gp = P.generate_sdf(peg, P.SdfResolutionSpec(64, 4))
    assert hashlib.sha256(gp.values.tobytes()).hexdigest() == meta["peg_r64"]["sha256"]


def test_batched_collide_r256_vs_golden(P, bolt, nut, gen256):
    g = P.generate_sdf(bolt, P.SdfResolutionSpec(256, 4))
    envs = list(gen256["envs"])
    E = len(envs)
    sp = np.stack([gen256[f"e{e}_sdf_pose"] for e in envs])
    mp = np.stack([gen256[f"e{e}_mesh_pose"] for e in envs])
    res = P.collide([P.register_sdf(g)] * E, [P.register_mesh(nut)] * E, sp, mp, np.full(E, float(gen256["cd"])))
    for i, e in enumerate(envs):
        cs = res.contact_set(i)
        got = {"points": cs.points, "normals": cs.normals, "depths": cs.depths, "faces": cs.face_indices}
        assert_same(got, gen256, f"e{e}_cs_", CS_KEYS, f"env {e} ")
        assert_same(pack_patch_list(res.patches(i), 6), gen256, f"e{e}_pt_", PATCH_KEYS, f"env {e} ")


def test_full_size_1024_envs_vs_oracle(P):
    """Config 2 at full size: every output field of all 1024 envs against the oracle
    (per-env digests), a sample of envs field by field, determinism across runs, and
    Algorithm-1 invariants."""
    from oracle import oracle as O
    from paper_2205_03532_b200.scenes import m16_workload

    E = 1024
    w = m16_workload(E, seed=0)
    grid, nut = w["grid"], w["nut"]
    res = P.collide([P.register_sdf(grid)] * E, [P.register_mesh(nut)] * E, w["sdf_pose"], w["mesh_pose"], w["cd"])
    stats = res.stats.cpu().numpy()
    n_cand = res.n_cand.cpu().numpy()
    n_patch = res.n_patch.cpu().numpy()
    og = O.Grid(grid.values, grid.dims, grid.origin, grid.voxel_size, *grid.mesh_aabb)
    ost = O.collide_batched(og, nut.vertices, nut.triangles, w["sdf_pose"], w["mesh_pose"], w["cd"])
    assert np.array_equal(n_cand, ost[:, 0].astype(np.int64))
    assert np.array_equal(n_patch, ost[:, 1].astype(np.int64))
    assert np.array_equal(stats[:, 2], ost[:, 2].astype(np.float32))
    assert np.array_equal(stats[:, 3], ost[:, 3].astype(np.float32))
    # EVERY output field of EVERY env, bit for bit: per-env digests of the candidates,
    # patch normals, kept candidates, members, aggregates, areas and max depths
    dig = env_digests(res.plan)
    odig = O.collide_digest(og, nut.vertices, nut.triangles, w["sdf_pose"], w["mesh_pose"], w["cd"])
    bad = np.nonzero(dig != odig)[0]
    assert len(bad) == 0, f"{len(bad)} of {E} envs differ, first {bad[:8].tolist()}"
    rng = np.random.default_rng(7)
    for e in rng.choice(E, size=4, replace=False):
        cs = res.contact_set(int(e))
        ref = O.generate_contacts(og, nut.vertices, nut.triangles, w["sdf_pose"][e], w["mesh_pose"][e], float(w["cd"][e]))
        assert np.array_equal(cs.points, ref["points"]) and np.array_equal(cs.normals, ref["normals"])
        assert np.array_equal(cs.depths, ref["depths"]) and np.array_equal(cs.face_indices, ref["faces"])
        r = O.reduce_contacts(ref["points"], ref["normals"], ref["depths"], ref["faces"], min_depth=-float(w["cd"][e]))
        got = pack_patch_list(res.patches(int(e)), 6)
        for k in ("rep", "nkept", "members", "kept_faces", "wsum", "wp", "wn", "wt", "area", "maxd"):
            assert np.array_equal(np.asarray(got[k]), np.asarray(r[k])), (int(e), k)
        # invariants: patches <= N, kept <= K, members partition the candidates,
        # the deepest candidate of every patch is kept
        assert len(got["nkept"]) <= 128 and (got["nkept"] <= 6).all()
        assert np.array_equal(np.sort(got["members"]), np.arange(len(cs)))
    # descent workload counters: survivors >= faces left to k_pgd_first by the stage-0
    # corner test >= faces moved by iteration 0 >= faces still moving after it; the corner
    # test settles most faces on this workload (78% of them stay at their start corner)
    fw = res.plan.face_work.cpu().numpy().astype(np.int64)
    assert fw[0] >= fw[1] >= fw[2] >= fw[3] >= 0 and fw[1] < 0.5 * fw[0], fw.tolist()
    # bitwise determinism across launches
    snap = {k: getattr(res, k).clone() for k in ("cand_point", "patch_normal", "kept_point", "w_sum", "area")}
    res2 = P.collide([P.register_sdf(grid)] * E, [P.register_mesh(nut)] * E, w["sdf_pose"], w["mesh_pose"], w["cd"])
    for k, v in snap.items():  # bit patterns (stale padding may hold NaNs)
        assert torch.equal(getattr(res2, k).view(torch.int64), v.view(torch.int64)), k


def test_errors_map_to_reference_classes(P, grid64, nut):
    from paper_2205_03532_b200.errors import NonFiniteStateError

    pairing = P.CollisionPairing(0, 1)
    ok = P.Transform()
    with pytest.raises(ValueError):
        P.generate_contacts(pairing, grid64, nut, ok, ok, -1.0)
    bad = P.Transform(translation=[np.nan, 0.0, 0.0])
    with pytest.raises(NonFiniteStateError):
        P.generate_contacts(pairing, grid64, nut, ok, bad, 1e-3)
    sp = np.tile([0, 0, 0, 1.0, 0, 0, 0], (2, 1))
    mp = sp.copy()
    mp[1, 0] = np.inf
    with pytest.raises(NonFiniteStateError):
        P.collide([P.register_sdf(grid64)] * 2, [P.register_mesh(nut)] * 2, sp, mp, np.full(2, 1e-3))
    with pytest.raises(ValueError):
        P.ReductionParams(max_patches=0)
    with pytest.raises(ValueError):
        P.collide([P.register_sdf(grid64)] * 2, [P.register_mesh(nut)] * 2, sp, sp, np.array([1e-3, -1.0]))


def test_empty_and_separated(P, grid64, nut):
    assert P.reduce_contacts(P.ContactSet.empty()) == []
    far = P.Transform(translation=[1.0, 0.0, 0.0])
    cs = P.generate_contacts(P.CollisionPairing(0, 1), grid64, nut, P.Transform(), far, 1e-3)
    assert len(cs) == 0
    res = P.collide([P.register_sdf(grid64)], [P.register_mesh(nut)], [[0, 0, 0, 1.0, 0, 0, 0]],
                    [[1.0, 0, 0, 1.0, 0, 0, 0]], [1e-3])
    assert int(res.n_cand[0]) == 0 and int(res.n_patch[0]) == 0 and res.patches(0) == []


def test_mixed_assets_per_env(P, grid64, nut, meshes):
    """Configs 3/4 shape: envs with different SDF grids and meshes in one collide
    call (M16 bolt grid + nut, peg grid + hole; moved SDF poses; a separated env),
    each env against the oracle field by field."""
    from oracle import oracle as O

    g = np.load(os.path.join(GOLDEN, "grid_peg_r64.npz"))
    peg_grid = P.SignedDistanceGrid(g["origin"], float(g["voxel"]), g["dims"], g["values"], (g["aabb_lo"], g["aabb_hi"]))
    hole = P.TriMesh(meshes["hole_v"], meshes["hole_t"])
    gen = np.load(os.path.join(GOLDEN, "gen_r64.npz"))
    ident = np.array([0, 0, 0, 1.0, 0, 0, 0])
    rng = np.random.default_rng(3)
    envs = []  # (sdf grid, oracle grid, mesh, sdf pose, mesh pose, cd)
    og_bolt = O.Grid.from_npz(np.load(os.path.join(GOLDEN, "grid_bolt_r64.npz")))
    og_peg = O.Grid.from_npz(g)
    for i in range(8):
        if i % 2 == 0:
            e = int(gen["envs"][(i // 2) % len(gen["envs"])])
            envs.append((grid64, og_bolt, nut, meshes["nut_v"], meshes["nut_t"], gen[f"e{e}_sdf_pose"],
                         gen[f"e{e}_mesh_pose"], 2.0 * grid64.voxel_size))
        else:
            dz = 0.05 if i == 7 else rng.uniform(0.0, 0.01)  # env 7: peg far above the hole
            sp = np.array([rng.uniform(-3e-4, 3e-4), rng.uniform(-3e-4, 3e-4), dz, 1.0, 0, 0, 0])
            envs.append((peg_grid, og_peg, hole, meshes["hole_v"], meshes["hole_t"], sp, ident,
                         2.0 * peg_grid.voxel_size))
    res = P.collide([P.register_sdf(x[0]) for x in envs], [P.register_mesh(x[2]) for x in envs],
                    np.stack([x[5] for x in envs]), np.stack([x[6] for x in envs]), np.array([x[7] for x in envs]))
    for i, (_, og, _, v, t, sp, mp, cd) in enumerate(envs):
        ref = O.generate_contacts(og, v, t, sp, mp, cd)
        cs = res.contact_set(i)
        assert np.array_equal(cs.points, ref["points"]) and np.array_equal(cs.normals, ref["normals"]), i
        assert np.array_equal(cs.depths, ref["depths"]) and np.array_equal(cs.face_indices, ref["faces"]), i
        assert (len(cs) > 0) == (i != 7), i
        r = O.reduce_contacts(ref["points"], ref["normals"], ref["depths"], ref["faces"], min_depth=-cd)
        got = pack_patch_list(res.patches(i), 6)
        for k in ("rep", "nkept", "members", "kept_faces", "wsum", "wp", "wn", "wt", "area", "maxd"):
            assert np.array_equal(np.asarray(got[k]), np.asarray(r[k])), (i, k)


def test_reduce_deep_hull_stacks(P):
    """Patches whose hull chains outgrow the kernel's shared-memory stack (points
    on convex curves: every point stays on the chain), plus a touching/non-touching
    mix, against the oracle."""
    from oracle import oracle as O

    rng = np.random.default_rng(11)
    for n, cap in ((300, 6), (1500, 6), (700, 3)):
        s = np.sort(rng.uniform(-1.0, 1.0, n))
        pts = np.stack([s * 1e-2, (s * s) * 1e-2, np.zeros(n)], axis=1)  # a parabola: all on the lower chain
        pts[::7, 2] += 1e-9  # a few off-plane points
        nrm = np.tile([0.0, 0.0, 1.0], (n, 1))
        dep = rng.uniform(-1e-4, 2e-4, n)
        faces = np.arange(n, dtype=np.int64)
        cs = P.ContactSet(pts, nrm, dep, faces, 0, 1)
        rp = P.ReductionParams(per_patch_cap=cap, min_depth=-1e-4)
        got = pack_patch_list(P.reduce_contacts(cs, rp), cap)
        r = O.reduce_contacts(pts, nrm, dep, faces, per_patch_cap=cap, min_depth=-1e-4)
        for k in ("rep", "nkept", "members", "kept_faces", "wsum", "wp", "wn", "wt", "area", "maxd"):
            assert np.array_equal(np.asarray(got[k]), np.asarray(r[k])), (n, k)


def test_config3_suite_4096_envs_vs_oracle(P):
    """Config 3 at full size: 4096 envs over pegs 4/8/12/16 mm in
    tight holes and M4..M20 nuts on bolts (9 assets, res-256 grids), one collide
    call with per-env handles; every output field of all 4096 envs against the oracle
    (per-env digests), two envs per asset field by field."""
    from oracle import oracle as O
    from paper_2205_03532_b200.scenes import suite_workload

    E = 4096
    w = suite_workload(E, seed=1)
    A, asset = w["assets"], w["asset"]
    hs = [P.register_sdf(a["grid"]) for a in A]
    hm = [P.register_mesh(a["mesh"]) for a in A]
    res = P.collide([hs[k] for k in asset], [hm[k] for k in asset], w["sdf_pose"], w["mesh_pose"], w["cd"])
    n_cand = res.n_cand.cpu().numpy()
    n_patch = res.n_patch.cpu().numpy()
    stats = res.stats.cpu().numpy()
    dig = env_digests(res.plan)
    rng = np.random.default_rng(5)
    for k, a in enumerate(A):
        idx = np.nonzero(asset == k)[0]
        g = a["grid"]
        og = O.Grid(g.values, g.dims, g.origin, g.voxel_size, *g.mesh_aabb)
        m = a["mesh"]
        ost = O.collide_batched(og, m.vertices, m.triangles, w["sdf_pose"][idx], w["mesh_pose"][idx], w["cd"][idx])
        assert np.array_equal(n_cand[idx], ost[:, 0].astype(np.int64)), a["name"]
        assert np.array_equal(n_patch[idx], ost[:, 1].astype(np.int64)), a["name"]
        assert np.array_equal(stats[idx, 2], ost[:, 2].astype(np.float32)), a["name"]
        assert np.array_equal(stats[idx, 3], ost[:, 3].astype(np.float32)), a["name"]
        assert (n_cand[idx] > 0).mean() > 0.5, a["name"]  # the poses engage the parts
        # every output field of every env of the asset, bit for bit (per-env digests)
        odig = O.collide_digest(og, m.vertices, m.triangles, w["sdf_pose"][idx], w["mesh_pose"][idx], w["cd"][idx])
        bad = np.nonzero(dig[idx] != odig)[0]
        assert len(bad) == 0, f"{a['name']}: {len(bad)} of {len(idx)} envs differ, first {idx[bad[:8]].tolist()}"
        for e in rng.choice(idx, size=2, replace=False):
            e = int(e)
            ref = O.generate_contacts(og, m.vertices, m.triangles, w["sdf_pose"][e], w["mesh_pose"][e],
                                      float(w["cd"][e]))
            cs = res.contact_set(e)
            assert np.array_equal(cs.points, ref["points"]) and np.array_equal(cs.normals, ref["normals"]), e
            assert np.array_equal(cs.depths, ref["depths"]) and np.array_equal(cs.face_indices, ref["faces"]), e
            r = O.reduce_contacts(ref["points"], ref["normals"], ref["depths"], ref["faces"],
                                  min_depth=-float(w["cd"][e]))
            got = pack_patch_list(res.patches(e), 6)
            for key in ("rep", "nkept", "members", "kept_faces", "wsum", "wp", "wn", "wt", "area", "maxd"):
                assert np.array_equal(np.asarray(got[key]), np.asarray(r[key])), (e, key)


def test_config5_res512_vs_oracle(P):
    """Config 5's largest grid: the M16 bolt at res 512 (~400 MB,
    above L2), generated on the GPU, 8 envs against the oracle field by field."""
    from oracle import oracle as O
    from paper_2205_03532_b200.scenes import m16_meshes, m16_workload
    from paper_2205_03532_b200.sdf.grid import SdfResolutionSpec, generate_sdf

    nut, bolt, _ = m16_meshes()
    grid = generate_sdf(bolt, SdfResolutionSpec(512, 4))
    assert max(grid.dims) == 512 and grid.values.nbytes > 300e6
    E = 8
    w = m16_workload(E, seed=4, grid=grid)
    res = P.collide([P.register_sdf(grid)] * E, [P.register_mesh(nut)] * E, w["sdf_pose"], w["mesh_pose"], w["cd"])
    og = O.Grid(grid.values, grid.dims, grid.origin, grid.voxel_size, *grid.mesh_aabb)
    assert (res.n_cand.cpu().numpy() > 0).sum() >= E // 2  # the poses engage the threads
    for e in range(E):
        cd = float(w["cd"][e])
        ref = O.generate_contacts(og, nut.vertices, nut.triangles, w["sdf_pose"][e], w["mesh_pose"][e], cd)
        cs = res.contact_set(e)
        assert np.array_equal(cs.points, ref["points"]) and np.array_equal(cs.normals, ref["normals"]), e
        assert np.array_equal(cs.depths, ref["depths"]) and np.array_equal(cs.face_indices, ref["faces"]), e
        r = O.reduce_contacts(ref["points"], ref["normals"], ref["depths"], ref["faces"], min_depth=-cd)
        got = pack_patch_list(res.patches(e), 6)
        for key in ("rep", "nkept", "members", "kept_faces", "wsum", "area", "maxd"):
            assert np.array_equal(np.asarray(got[key]), np.asarray(r[key])), (e, key)


def test_collide_cuda_graph_replay(P, grid64, nut, gen64):
    """A collide step captured in a CUDA graph replays bit-identically to eager
    launches, including after new poses are copied into the captured inputs."""
    envs = list(gen64["envs"])
    E = len(envs)
    plan = P.Plan([P.register_sdf(grid64)] * E, [P.register_mesh(nut)] * E, P.ReductionParams())
    sp0 = np.stack([gen64[f"e{e}_sdf_pose"] for e in envs])
    mp0 = np.stack([gen64[f"e{e}_mesh_pose"] for e in envs])
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float64)).cuda()  # noqa: E731
    sp, mp, cd = d(sp0), d(mp0), d(np.full(E, float(gen64["cd"])))
    keys = ("n_cand", "cand_point", "cand_face", "n_patch", "patch_normal", "kept_point", "w_sum", "area")

    def snap():
        # bit patterns: the padding past n_patch is never written and may hold stale NaNs
        # (torch.equal calls NaN != NaN), so floats compare as integers
        torch.cuda.synchronize()
        out = {}
        for k in keys:
            v = getattr(plan, k).clone()
            out[k] = v.view(torch.int64) if v.dtype == torch.float64 else v
        return out

    plan.collide(sp, mp, cd)
    eager = snap()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        plan.collide(sp, mp, cd, stream=s)
    g.replay()
    got = snap()
    for k in keys:
        assert torch.equal(got[k], eager[k]), (k, torch.nonzero(got[k] != eager[k])[:6].tolist())
    # new poses into the captured input buffers
    mp1 = mp0[::-1].copy()
    mp.copy_(d(mp1))
    g.replay()
    got = snap()
    plan.collide(sp, mp, cd)
    eager = snap()
    for k in keys:
        assert torch.equal(got[k], eager[k]), k


def test_plan_memory_released_without_gc(P, grid64, nut):
    """Dropping a Plan frees its device buffers at once (views keep a small handle,
    not the Plan, so there is no reference cycle); a held view keeps them alive."""
    E = 256
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info()[0]
    plan = P.Plan([P.register_sdf(grid64)] * E, [P.register_mesh(nut)] * E, P.ReductionParams())
    used = free0 - torch.cuda.mem_get_info()[0]
    assert used > 100e6
    view = plan.n_cand
    del plan
    assert free0 - torch.cuda.mem_get_info()[0] > 0.9 * used  # still owned through the view
    del view
    assert free0 - torch.cuda.mem_get_info()[0] < 0.1 * used


def test_plan_device_bytes(P, grid64, nut):
    """Plan.device_bytes (cs_plan_device_bytes) accounts for what the plan allocates,
    linear in the env count, and the descent staging shares the reduction's per-row
    arena (at most 200 B of the two per face row, not their 312 B sum)."""
    hs, hm = P.register_sdf(grid64), P.register_mesh(nut)
    F = len(nut.triangles)
    sizes = []
    for E in (256, 512):
        torch.cuda.synchronize()
        free0 = torch.cuda.mem_get_info()[0]
        plan = P.Plan([hs] * E, [hm] * E, P.ReductionParams())
        used = free0 - torch.cuda.mem_get_info()[0]
        b = plan.device_bytes
        assert 0.9 * used <= b <= used + (64 << 20), (b, used)  # cudaMalloc granularity on top
        sizes.append(b)
        del plan
    per_env = (sizes[1] - sizes[0]) / 256
    assert abs(sizes[1] - 2 * sizes[0]) < 0.02 * sizes[1]
    # candidates 60 B + members 4 B + arena <= 200 B per row, plus per-env/patch outputs
    assert per_env < F * 270 + 200_000, per_env


def test_asset_free_deferred_while_plans_use_it(P, grid64, gen64, meshes):
    """cs_sdf_free / cs_mesh_free on an asset a live plan samples defer the release to
    the last such plan's destruction (no use-after-free); a freed handle cannot start
    a new plan."""
    import ctypes

    from paper_2205_03532_b200 import _native

    lib = _native.lib()
    v, t = np.ascontiguousarray(meshes["nut_v"], np.float64), np.ascontiguousarray(meshes["nut_t"], np.int32)
    hm = ctypes.c_int32(-1)
    _native.check(lib.cs_mesh_register(v.ctypes.data, len(v), t.ctypes.data, len(t), ctypes.byref(hm)))
    hs = P.register_sdf(grid64)
    envs = list(gen64["envs"])[:2]
    sp = torch.from_numpy(np.stack([gen64[f"e{e}_sdf_pose"] for e in envs])).cuda()
    mp = torch.from_numpy(np.stack([gen64[f"e{e}_mesh_pose"] for e in envs])).cuda()
    cd = torch.full((2,), float(gen64["cd"]), dtype=torch.float64, device="cuda")
    plan = P.Plan([hs, hs], [hm.value, hm.value], P.ReductionParams())
    plan.collide(sp, mp, cd)
    before = plan.cand_face.clone()
    _native.check(lib.cs_mesh_free(hm.value))  # deferred: the plan still samples it
    plan.collide(sp, mp, cd)
    torch.cuda.synchronize()
    assert torch.equal(plan.cand_face, before)
    assert lib.cs_mesh_free(hm.value) == _native.CS_ERR_HANDLE  # already freed by the caller
    with pytest.raises(RuntimeError):
        P.Plan([hs], [hm.value], P.ReductionParams())
    del plan  # releases the mesh now
    assert lib.cs_mesh_free(hm.value) == _native.CS_ERR_HANDLE


_GRIDS = {}  # GPU-generated grids shared by the tests below


@pytest.mark.parametrize("seed", [11, 12])
def test_random_frames_vs_oracle(P, seed):
    """Fresh pose seeds at res 256 with the SDF body itself moved and rotated per env
    (the nut follows it rigidly, so the pair stays engaged): every env's stats
    against the oracle and four envs field by field."""
    from oracle import oracle as O
    from paper_2205_03532_b200.math3d import quat_multiply, quat_to_matrix
    from paper_2205_03532_b200.scenes import m16_meshes, m16_workload
    from paper_2205_03532_b200.sdf.grid import SdfResolutionSpec, generate_sdf

    nut, bolt, _ = m16_meshes()
    if 256 not in _GRIDS:
        _GRIDS[256] = generate_sdf(bolt, SdfResolutionSpec(256, 4))
    grid = _GRIDS[256]
    E = 128
    w = m16_workload(E, seed=seed, grid=grid)
    rng = np.random.default_rng(seed)
    sp = np.zeros((E, 7))
    mp = np.zeros((E, 7))
    for e in range(E):
        q = rng.standard_normal(4)
        q /= np.linalg.norm(q)
        t = rng.uniform(-0.05, 0.05, 3)
        sp[e, :3], sp[e, 3:] = t, q
        # nut pose relative to the bolt as drawn, composed with the bolt's world pose
        mp[e, :3] = t + quat_to_matrix(q) @ w["mesh_pose"][e, :3]
        mp[e, 3:] = quat_multiply(q, w["mesh_pose"][e, 3:])
    res = P.collide([P.register_sdf(grid)] * E, [P.register_mesh(nut)] * E, sp, mp, w["cd"])
    og = O.Grid(grid.values, grid.dims, grid.origin, grid.voxel_size, *grid.mesh_aabb)
    ost = O.collide_batched(og, nut.vertices, nut.triangles, sp, mp, w["cd"])
    assert np.array_equal(res.n_cand.cpu().numpy(), ost[:, 0].astype(np.int64))
    assert np.array_equal(res.n_patch.cpu().numpy(), ost[:, 1].astype(np.int64))
    st = res.stats.cpu().numpy()
    assert np.array_equal(st[:, 2], ost[:, 2].astype(np.float32)) and np.array_equal(st[:, 3], ost[:, 3].astype(np.float32))
    assert (ost[:, 0] > 0).mean() > 0.9
    for e in rng.choice(E, size=4, replace=False):
        e = int(e)
        cd = float(w["cd"][e])
        ref = O.generate_contacts(og, nut.vertices, nut.triangles, sp[e], mp[e], cd)
        cs = res.contact_set(e)
        assert np.array_equal(cs.points, ref["points"]) and np.array_equal(cs.normals, ref["normals"]), e
        assert np.array_equal(cs.depths, ref["depths"]) and np.array_equal(cs.face_indices, ref["faces"]), e
        r = O.reduce_contacts(ref["points"], ref["normals"], ref["depths"], ref["faces"], min_depth=-cd)
        got = pack_patch_list(res.patches(e), 6)
        for key in ("rep", "nkept", "members", "kept_faces", "wsum", "wp", "wn", "wt", "area", "maxd"):
            assert np.array_equal(np.asarray(got[key]), np.asarray(r[key])), (e, key)
