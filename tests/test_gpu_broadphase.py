"""GPU parity of the broadphase and multi-pair scenes (SURVEY §8(f) row 2,
csrc/cs_broadphase.cu through libcontactsim_b200.so): world AABBs and pair lists
bit-exact against the reference's goldens (tests/golden/broadphase.npz), and the
device pipeline world AABB -> broadphase -> pair slots -> collide against the
oracle per active pair (Scene._collect_contacts semantics, scene.py:170-227)."""

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

G = golden("broadphase.npz")
SCENES = [str(s) for s in G["scenes"]]


@pytest.fixture(scope="module")
def P():
    import paper_2205_03532_b200 as P
    from paper_2205_03532_b200 import _native

    _native.lib()
    return P


def test_world_aabbs_match_reference(P):
    from paper_2205_03532_b200.geometry import world_aabbs

    lo, hi = world_aabbs(G["aabb_mesh_lo"], G["aabb_mesh_hi"], G["aabb_pose"])
    assert lo.cpu().numpy().tobytes() == G["aabb_world_lo"].tobytes()
    assert hi.cpu().numpy().tobytes() == G["aabb_world_hi"].tobytes()


@pytest.mark.parametrize("name", SCENES)
def test_broadphase_pairs_dropin(P, name):
    from paper_2205_03532_b200.geometry import broadphase_pairs

    lo, hi, ids = G[f"{name}_lo"], G[f"{name}_hi"], G[f"{name}_ids"]
    bodies = [((lo[i], hi[i]), int(ids[i])) for i in range(len(ids))]
    got = broadphase_pairs(bodies, float(G[f"{name}_margin"]))
    assert got == [tuple(int(x) for x in p) for p in G[f"{name}_pairs"]]


def test_broadphase_batched_all_scenes_one_launch(P):
    from paper_2205_03532_b200.geometry import broadphase_batched

    lo = np.concatenate([G[f"{n}_lo"] for n in SCENES])
    hi = np.concatenate([G[f"{n}_hi"] for n in SCENES])
    ids = np.concatenate([G[f"{n}_ids"] for n in SCENES])
    off = np.concatenate([[0], np.cumsum([len(G[f"{n}_ids"]) for n in SCENES])])
    margin = np.array([float(G[f"{n}_margin"]) for n in SCENES])
    poff, pairs, n_pairs, status = broadphase_batched(lo, hi, off, margin, ids)
    assert not status.any()
    poff, pairs, n_pairs = poff.cpu().numpy(), pairs.cpu().numpy(), n_pairs.cpu().numpy()
    for s, n in enumerate(SCENES):
        assert np.array_equal(pairs[poff[s]:poff[s] + n_pairs[s]], G[f"{n}_pairs"]), n


def test_broadphase_errors(P):
    from paper_2205_03532_b200.geometry import broadphase_pairs

    with pytest.raises(ValueError):
        broadphase_pairs([((np.zeros(3), np.ones(3)), 0), ((np.full(3, np.nan), np.ones(3)), 1)])
    with pytest.raises(ValueError):
        broadphase_pairs([((np.zeros(3), np.ones(3)), 0), ((np.zeros(3), np.ones(3)), 0)])
    assert broadphase_pairs([((np.zeros(3), np.ones(3)), 0)]) == []


def test_multipair_scenes_match_oracle(P, grid64_npz, meshes):
    """Config-4-style scenes: a static bolt SDF, a dynamic nut mesh and
    two chain-driven finger pads with their own res-64 SDFs, several scenes per
    launch, some pads away from the nut (inactive pairs)."""
    from oracle import oracle as O
    from paper_2205_03532_b200.geometry import make_box
    from paper_2205_03532_b200.multipair import MultiPairScenes, SceneBody

    gen64 = golden("gen_r64.npz")
    d = grid64_npz
    bolt_grid = P.SignedDistanceGrid(d["origin"], float(d["voxel"]), d["dims"], d["values"],
                                     (d["aabb_lo"], d["aabb_hi"]))
    bolt = P.TriMesh(meshes["bolt_v"], meshes["bolt_t"])
    nut = P.TriMesh(meshes["nut_v"], meshes["nut_t"])
    pad = make_box((0.004, 0.016, 0.008), subdivisions=8)
    pad_grid = P.generate_sdf(pad, P.SdfResolutionSpec(64, 4))
    hb, hn, hp = P.register_sdf(bolt_grid), P.register_mesh(nut), P.register_sdf(pad_grid)
    hbm, hpm = P.register_mesh(bolt), P.register_mesh(pad)

    def scene():
        return [SceneBody(0, hbm, bolt.aabb(), len(bolt.triangles), hb, bolt_grid.voxel_size, True, True),
                SceneBody(1, hn, nut.aabb(), len(nut.triangles), None, None, False, False),
                SceneBody(2, hpm, pad.aabb(), len(pad.triangles), hp, pad_grid.voxel_size, True, True),
                SceneBody(3, hpm, pad.aabb(), len(pad.triangles), hp, pad_grid.voxel_size, True, True)]

    envs = list(gen64["envs"])
    S = len(envs)
    mps = MultiPairScenes([scene() for _ in range(S)])
    # slots per scene: (0,1) bolt-nut, (1,2) pad-nut, (1,3) pad-nut; fixed-fixed pairs skipped
    assert mps.n_slots == 3 * S
    poses = np.zeros((S, 4, 7))
    for i, e in enumerate(envs):
        poses[i, 0] = gen64[f"e{e}_sdf_pose"]
        mp = gen64[f"e{e}_mesh_pose"]
        poses[i, 1] = mp
        R = O.quat_to_matrix(mp[3:])
        for b, sgn in ((2, 1.0), (3, -1.0)):
            away = 0.05 if (i % 3 == 2 and b == 3) else 0.0  # some pads off the nut
            poses[i, b, :3] = mp[:3] + R @ np.array([sgn * (0.014 - 0.00005) + sgn * away, 0.0, 0.0])
            poses[i, b, 3:] = mp[3:]
    res = mps.step(poses.reshape(-1, 7))
    active = mps.active.cpu().numpy()
    grids = {0: O.Grid.from_npz(d), 2: O.Grid(pad_grid.values, pad_grid.dims, pad_grid.origin,
                                               pad_grid.voxel_size, *pad_grid.mesh_aabb)}
    grids[3] = grids[2]
    verts = {1: (nut.vertices, nut.triangles)}
    margin = 2.0 * max(bolt_grid.voxel_size, pad_grid.voxel_size)
    n_active = 0
    for i in range(S):
        mlo = np.array([bolt.aabb()[0], nut.aabb()[0], pad.aabb()[0], pad.aabb()[0]])
        mhi = np.array([bolt.aabb()[1], nut.aabb()[1], pad.aabb()[1], pad.aabb()[1]])
        wlo, whi = O.world_aabb(mlo, mhi, poses[i])
        ref_pairs = [tuple(int(x) for x in p) for p in O.broadphase_pairs(wlo, whi, [0, 1, 2, 3], margin)]
        assert mps.scene_pairs(i) == ref_pairs, i
        for t in np.nonzero(mps.slot_scene == i)[0]:
            pair = tuple(int(x) for x in mps.slot_pair[t])
            assert bool(active[t]) == (pair in ref_pairs), (i, pair)
            cs = res.contact_set(int(t))
            if not active[t]:
                assert len(cs) == 0 and int(res.n_patch[t]) == 0
                continue
            n_active += 1
            sb, mb = int(mps.slot_sdf_body[t]), int(mps.slot_mesh_body[t])
            cd = 2.0 * (bolt_grid.voxel_size if sb == 0 else pad_grid.voxel_size)
            ref = O.generate_contacts(grids[sb], *verts[mb], poses[i, sb], poses[i, mb], cd)
            assert np.array_equal(cs.points, ref["points"]) and np.array_equal(cs.face_indices, ref["faces"])
            red = O.reduce_contacts(ref["points"], ref["normals"], ref["depths"], ref["faces"], min_depth=-cd)
            pt = res.patches(int(t))
            assert len(pt) == len(red["nkept"])
            for q, p in enumerate(pt):
                assert np.array_equal(p.face_indices, red["kept_faces"][q, :len(p)])
    assert n_active > S  # bolt-nut in every scene plus touching pads

    # the substep's contact solve over each whole scene (4 bodies; rows of its active
    # pairs in pair order, body_a = the pair's SDF body), against the oracle
    from paper_2205_03532_b200.dynamics import BatchedSolverState, SolverParams

    rng = np.random.default_rng(9)
    ref_pt = np.zeros((S, 4, 3)); W = np.zeros((S, 4, 6, 6)); vel = np.zeros((S, 4, 6))
    ref_pt[:, 1] = poses[:, 1, :3]
    W[:, 1, :3, :3] = np.eye(3) / 0.03
    W[:, 1, 3:, 3:] = np.diag(1.0 / np.array([2.4e-6, 2.4e-6, 3.9e-6]))
    vel[:, 1] = rng.standard_normal((S, 6)) * 0.05
    vel[:, 1, 2] -= 0.3
    st = BatchedSolverState.from_numpy(ref_pt, W, vel)
    prm = SolverParams(pos_iterations=8, vel_iterations=2)
    wrench = mps.solve(st, prm).cpu().numpy()
    gv = st.vel.cpu().numpy()
    h = prm.dt / prm.substeps
    for i in range(S):
        pts, nrm, dep, ba, bb, mu, rs, sl = [], [], [], [], [], [], [], []
        for t in np.nonzero(mps.slot_scene == i)[0]:
            if not active[t]:
                continue
            sb, mb = int(mps.slot_sdf_body[t]), int(mps.slot_mesh_body[t])
            for p in res.patches(int(t)):
                pts.append(p.points); nrm.append(p.normals); dep.append(p.depths)
                k = len(p.depths)
                ba += [sb] * k; bb += [mb] * k
                mu += [0.5] * k; rs += [0.0] * k
                sl += [0.5 * (bolt_grid.voxel_size if sb == 0 else pad_grid.voxel_size)] * k
        m = len(ba)
        pts, nrm, dep = np.concatenate(pts), np.concatenate(nrm), np.concatenate(dep)
        a, b = np.array(ba, np.int64), np.array(bb, np.int64)
        con = O.constraints_build(a, b, pts, nrm, dep, np.array(rs), np.array(sl), ref_pt[i], W[i], vel[i], h,
                                  prm.bias_factor)
        v, imp = np.array(vel[i]), np.zeros((4, 6))
        ln, l1, l2, lv = (np.zeros(m) for _ in range(4))
        geo = (a, b, con["ra"], con["rb"], nrm, con["tan1"], con["tan2"], con["kn"], con["kt1"], con["kt2"])
        O.gauss_seidel_sweeps(prm.pos_iterations, W[i], v, imp, *geo, con["bias_target"], np.array(mu), ln, l1, l2,
                              True)
        O.gauss_seidel_sweeps(prm.vel_iterations, W[i], v, imp, *geo, con["restitution_target"], np.array(mu), lv,
                              l1, l2, False)
        wr = O.body_wrenches(4, a, b, con["ra"], con["rb"], nrm, con["tan1"], con["tan2"], ln, lv, l1, l2, h)
        assert np.array_equal(gv[i], v), i
        assert np.array_equal(wrench[i], wr), i

    # the same solve on the scene state padded to 10 bodies (bodies 4..9 idle): the
    # packed sweeps' global-memory state path (systems above 8 bodies) gives the same bits
    idle = rng.standard_normal((S, 6, 6))
    st10 = BatchedSolverState.from_numpy(np.concatenate([ref_pt, np.zeros((S, 6, 3))], 1),
                                         np.concatenate([W, np.zeros((S, 6, 6, 6))], 1),
                                         np.concatenate([vel, idle], 1))
    wrench10 = mps.solve(st10, prm).cpu().numpy()
    gv10 = st10.vel.cpu().numpy()
    assert np.array_equal(gv10[:, :4], gv) and np.array_equal(gv10[:, 4:], idle)
    assert np.array_equal(wrench10[:, :4], wrench) and not wrench10[:, 4:].any()


def test_broadphase_max_scene_and_status_codes(P):
    """The per-scene cap (2048 bodies, sweep semantics, inverted boxes included)
    against the oracle, and the batched status codes for the scenes it refuses."""
    from oracle import oracle as O
    from paper_2205_03532_b200.geometry import broadphase_batched, broadphase_pairs
    from paper_2205_03532_b200.geometry.broadphase import MAX_BODIES

    rng = np.random.default_rng(33)
    n = MAX_BODIES
    c = rng.uniform(-0.5, 0.5, (n, 3))
    ext = rng.uniform(0.002, 0.02, (n, 3))
    lo, hi = c - ext, c + ext
    lo[10, 0], hi[10, 0] = hi[10, 0], lo[10, 0]
    lo[11, 0] = lo[12, 0] = lo[13, 0]
    ids = rng.permutation(n * 2)[:n]
    got = broadphase_pairs([((lo[i], hi[i]), int(ids[i])) for i in range(n)], 1e-3)
    ref = [tuple(int(x) for x in p) for p in O.broadphase_pairs(lo, hi, ids, 1e-3)]
    assert got == ref and len(ref) > 100
    # scene 0 fine, scene 1 over the cap (3), scene 2 duplicate ids (4), scene 3 NaN (1)
    m = n + 1
    lo2 = np.concatenate([lo[:5], rng.uniform(-1, 1, (m, 3)), lo[:3], lo[:3]])
    hi2 = lo2 + 0.01
    hi2[-1, 1] = np.nan
    ids2 = np.concatenate([np.arange(5), np.arange(m), [1, 2, 1], [0, 1, 2]])
    off = np.array([0, 5, 5 + m, 8 + m, 11 + m])
    _, _, n_pairs, status = broadphase_batched(lo2, hi2, off, np.zeros(4), ids2)
    assert status.cpu().tolist() == [0, 3, 4, 1]
