"""GPU: the edges of the drop-in boundary that round 2 hardened.

* the exact face bound at cd = 0, tiny cd and at faces outside the grid (the
  outside-distance term), every output against the oracle (per-env digests);
* SDF files straight to the device store (cs_sdf_register_file) against the
  reference-written file and the host loader;
* bounded, thread-keyed plan caches that release assets;
* argument checks (shapes, stream hand-off, solver body limit, shared-memory limit).
"""

import gc
import os

import numpy as np
import pytest

from conftest import GOLDEN, env_digests

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def P():
    import paper_2205_03532_b200 as P
    from paper_2205_03532_b200 import _native

    _native.lib()
    return P


@pytest.fixture(scope="module")
def grid64(P, grid64_npz):
    d = grid64_npz
    return P.SignedDistanceGrid(d["origin"], float(d["voxel"]), d["dims"], d["values"], (d["aabb_lo"], d["aabb_hi"]))


@pytest.fixture(scope="module")
def nut(P, meshes):
    return P.TriMesh(meshes["nut_v"], meshes["nut_t"])


def _digest_case(P, grid, nut, sp, mp, cd):
    from oracle import oracle as O

    E = len(mp)
    res = P.collide([P.register_sdf(grid)] * E, [P.register_mesh(nut)] * E, sp, mp, cd)
    og = O.Grid(grid.values, grid.dims, grid.origin, grid.voxel_size, *grid.mesh_aabb)
    odig = O.collide_digest(og, nut.vertices, nut.triangles, sp, mp, cd)
    ost = O.collide_batched(og, nut.vertices, nut.triangles, sp, mp, cd)
    dig = env_digests(res.plan)
    assert np.array_equal(res.n_cand.cpu().numpy(), ost[:, 0].astype(np.int64))
    bad = np.nonzero(dig != odig)[0]
    assert len(bad) == 0, f"envs {bad.tolist()} differ"
    return ost


def test_bound_at_zero_and_tiny_contact_distance(P, grid64, nut, gen64):
    """cd = 0 and cd -> 0: the face bound's margin is absolute (max |value| 2^-40),
    so skipping stays exact where the minimum corner is near zero."""
    envs = list(gen64["envs"])
    sp = np.stack([gen64[f"e{e}_sdf_pose"] for e in envs])
    mp = np.stack([gen64[f"e{e}_mesh_pose"] for e in envs])
    v = grid64.voxel_size
    for cd in (0.0, 1e-15, 1e-12, 1e-9, 0.05 * v, 0.5 * v):
        _digest_case(P, grid64, nut, sp, mp, np.full(len(envs), cd))


def test_faces_outside_the_grid(P, grid64, nut, gen64):
    """The nut lifted through the grid's top face and pushed out sideways: samples
    clamp to boundary cells and add the outside distance (sdf/_kernels.py:299-308);
    with a large cd those faces become candidates. Every output vs the oracle."""
    e0 = int(gen64["envs"][0])
    base = gen64[f"e{e0}_mesh_pose"]
    top = grid64.origin[2] + (grid64.dims[2] - 1) * grid64.voxel_size
    side = grid64.origin[0] + (grid64.dims[0] - 1) * grid64.voxel_size
    poses = []
    for dz in (-0.004, -0.002, 0.0, 0.003):
        p = base.copy()
        p[2] = top + dz
        poses.append(p)
    for dx in (0.0, 0.004):
        p = base.copy()
        p[0] = side + dx
        poses.append(p)
    mp = np.stack(poses)
    sp = np.tile(gen64[f"e{e0}_sdf_pose"], (len(mp), 1))
    for cd in (2.0 * grid64.voxel_size, 0.004):
        ost = _digest_case(P, grid64, nut, sp, mp, np.full(len(mp), cd))
    assert (ost[:, 0] > 0).sum() >= 3  # the outside-term faces produce candidates at cd = 4 mm


def test_load_device_matches_reference_file(P):
    import json

    from paper_2205_03532_b200.sdf.grid import SignedDistanceGrid, load_device

    meta = json.load(open(os.path.join(GOLDEN, "sdf_file.json")))
    path = os.path.join(GOLDEN, meta["file"])
    host = SignedDistanceGrid.load(path)
    dev = load_device(path)
    assert dev.dims == host.dims and np.array_equal(dev.origin, host.origin) and dev.voxel_size == host.voxel_size
    assert np.array_equal(dev.mesh_aabb[0], host.mesh_aabb[0]) and np.array_equal(dev.mesh_aabb[1], host.mesh_aabb[1])
    assert np.array_equal(dev.values, host.values)
    pts = np.random.default_rng(0).uniform(host.origin - 0.002, host.origin + np.array(host.dims) * host.voxel_size,
                                           (512, 3))
    assert np.array_equal(dev.sample(pts), host.sample(pts))
    assert np.array_equal(dev.gradient(pts), host.gradient(pts))


def test_load_device_errors(P, tmp_path):
    from paper_2205_03532_b200.sdf.grid import load_device

    with pytest.raises(OSError):
        load_device(tmp_path / "missing.sdf")
    data = open(os.path.join(GOLDEN, "ref_peg_r64.sdf"), "rb").read()
    (tmp_path / "bad.sdf").write_bytes(b"XXXXXXXX" + data[8:])
    with pytest.raises(ValueError, match="not an SDF grid file"):
        load_device(tmp_path / "bad.sdf")
    (tmp_path / "short.sdf").write_bytes(data[:-4])
    with pytest.raises(ValueError):
        load_device(tmp_path / "short.sdf")


def test_collide_with_file_registered_grid(P, grid64, nut, gen64, tmp_path):
    """A grid registered from its file behaves exactly like the host-registered one,
    and cached_sdf(device=True) returns it for a cache hit."""
    from paper_2205_03532_b200.sdf.grid import DeviceSignedDistanceGrid, SdfResolutionSpec, cached_sdf, load_device

    path = tmp_path / "bolt64.sdf"
    grid64.save(path)
    dg = load_device(path)
    envs = list(gen64["envs"])
    sp = np.stack([gen64[f"e{e}_sdf_pose"] for e in envs])
    mp = np.stack([gen64[f"e{e}_mesh_pose"] for e in envs])
    cd = np.full(len(envs), float(gen64["cd"]))
    a = P.collide([P.register_sdf(grid64)] * len(envs), [P.register_mesh(nut)] * len(envs), sp, mp, cd)
    da = env_digests(a.plan)
    b = P.collide([P.register_sdf(dg)] * len(envs), [P.register_mesh(nut)] * len(envs), sp, mp, cd)
    assert np.array_equal(env_digests(b.plan), da)
    from paper_2205_03532_b200.geometry import TriMesh

    bolt = TriMesh(*(np.load(os.path.join(GOLDEN, "meshes.npz"))[k] for k in ("bolt_v", "bolt_t")))
    key = tmp_path / f"{bolt.content_digest()}_r64_p4.sdf"
    os.replace(path, key)
    hit = cached_sdf(bolt, SdfResolutionSpec(64, 4), cache_dir=tmp_path, device=True)
    assert isinstance(hit, DeviceSignedDistanceGrid) and np.array_equal(hit.values, grid64.values)


def test_plan_caches_release_assets(P, grid64, nut, gen64):
    """The per-pair drop-in's cached plan is dropped when its grid is finalised, so
    the grid's deferred device free completes."""
    from paper_2205_03532_b200.contacts import generation as gen

    g = P.SignedDistanceGrid(grid64.origin, grid64.voxel_size, grid64.dims, grid64.values.copy(), grid64.mesh_aabb)
    e = int(gen64["envs"][0])
    sp = P.Transform.from_pose(gen64[f"e{e}_sdf_pose"][:3], gen64[f"e{e}_sdf_pose"][3:])
    mp = P.Transform.from_pose(gen64[f"e{e}_mesh_pose"][:3], gen64[f"e{e}_mesh_pose"][3:])
    cs = P.generate_contacts(P.CollisionPairing(0, 1), g, nut, sp, mp, float(gen64["cd"]))
    assert len(cs) > 0
    h = g.device_handle()
    cache = gen._gen_plans()
    assert any(h in s for (s, _) in cache._assets.values())
    del g
    gc.collect()
    assert not any(h in s for (s, _) in cache._assets.values())
    # the device copy is released: the handle no longer names a live grid
    import ctypes

    from paper_2205_03532_b200 import _native

    ptr = ctypes.c_void_p()
    assert _native.lib().cs_sdf_values(h, ctypes.byref(ptr)) == _native.CS_ERR_HANDLE
    g2 = P.SignedDistanceGrid(grid64.origin, grid64.voxel_size, grid64.dims, grid64.values, grid64.mesh_aabb)
    # bounded: many distinct pairs never keep more than maxsize plans
    for _ in range(cache.maxsize + 4):
        m = P.TriMesh(nut.vertices, nut.triangles)
        P.generate_contacts(P.CollisionPairing(0, 1), g2, m, sp, mp, float(gen64["cd"]))
    assert len(cache) <= cache.maxsize


def test_argument_checks(P, grid64, nut):
    from paper_2205_03532_b200 import _native
    from paper_2205_03532_b200.collide import Plan
    from paper_2205_03532_b200.dynamics import BatchedSolverState

    plan = Plan([P.register_sdf(grid64)] * 4, [P.register_mesh(nut)] * 4, None)
    d = lambda *s: torch.zeros(s, dtype=torch.float64, device="cuda")  # noqa: E731
    with pytest.raises(ValueError, match="sdf_pose"):
        plan.collide(d(3, 7), d(4, 7), d(4))
    with pytest.raises(ValueError, match="mesh_pose"):
        plan.collide(d(4, 7), d(4, 12), d(4))
    with pytest.raises(ValueError, match="contact_distance"):
        plan.collide(d(4, 7), d(4, 7), d(5))
    with pytest.raises(ValueError):
        plan.collide_host(np.zeros((4, 7)), np.zeros((4, 7)), np.zeros(2))
    with pytest.raises(ValueError, match="state.ref"):
        plan.solve(BatchedSolverState(4, 3), d(4), d(4), d(4))
    with pytest.raises(ValueError, match="mu"):
        plan.solve(BatchedSolverState(4, 2), d(3), d(4), d(4))
    # k_reduce's shared memory: refused at plan creation with a clear message
    with pytest.raises(ValueError, match="shared memory"):
        Plan([P.register_sdf(grid64)], [P.register_mesh(nut)], P.ReductionParams(max_patches=4096, batch_size=16384))
    # the device solver's body limit is explicit
    from paper_2205_03532_b200.dynamics.solver import SOLVER_MAX_BODIES, check_solver_bodies

    with pytest.raises(ValueError, match="bodies"):
        check_solver_bodies(SOLVER_MAX_BODIES + 1)
    assert _native.CS_ERR_IO == 7


def test_collide_on_a_side_stream(P, grid64, nut, gen64):
    """collide(stream=s): the inputs staged on the current stream are handed to s
    (wait + record_stream) and check() waits for s."""
    envs = list(gen64["envs"])
    E = len(envs)
    sp = np.stack([gen64[f"e{e}_sdf_pose"] for e in envs])
    mp = np.stack([gen64[f"e{e}_mesh_pose"] for e in envs])
    cd = np.full(E, float(gen64["cd"]))
    hs, hm = [P.register_sdf(grid64)] * E, [P.register_mesh(nut)] * E
    ref = env_digests(P.collide(hs, hm, sp, mp, cd).plan)
    from paper_2205_03532_b200.collide import clear_plan_cache

    clear_plan_cache()
    s = torch.cuda.Stream()
    res = P.collide(hs, hm, sp, mp, cd, stream=s)  # check() syncs s
    s.synchronize()
    assert np.array_equal(env_digests(res.plan), ref)
    bad = mp.copy()
    bad[1, 0] = np.nan
    from paper_2205_03532_b200.errors import NonFiniteStateError

    with pytest.raises(NonFiniteStateError):
        P.collide(hs, hm, sp, bad, cd, stream=s)


def test_collide_host_graph_replay(P, grid64, nut, gen64):
    """cs_collide_host replays the step from a CUDA graph after its first call: every call
    (eager, capture, replays, a pose-format switch) gives the device path's results."""
    from paper_2205_03532_b200 import _native
    from paper_2205_03532_b200.collide import Plan

    envs = list(gen64["envs"])
    E = len(envs)
    cd = np.full(E, float(gen64["cd"]))
    sp = np.ascontiguousarray(np.stack([gen64[f"e{e}_sdf_pose"] for e in envs]))
    mp = np.ascontiguousarray(np.stack([gen64[f"e{e}_mesh_pose"] for e in envs]))
    host = Plan([P.register_sdf(grid64)] * E, [P.register_mesh(nut)] * E, P.ReductionParams())
    dev = Plan([P.register_sdf(grid64)] * E, [P.register_mesh(nut)] * E, P.ReductionParams())
    rng = np.random.default_rng(7)
    def same(k):  # the valid outputs (padding past n_cand / n_patch is never written)
        assert np.array_equal(host.n_cand.cpu().numpy(), dev.n_cand.cpu().numpy()), k
        rh, rd = P.ReducedContacts(host), P.ReducedContacts(dev)
        for e in range(E):
            a, b = rh.contact_set(e), rd.contact_set(e)
            assert np.array_equal(a.points, b.points) and np.array_equal(a.normals, b.normals), (k, e)
            assert np.array_equal(a.depths, b.depths) and np.array_equal(a.face_indices, b.face_indices), (k, e)
            pa, pb = rh.patches(e), rd.patches(e)
            assert len(pa) == len(pb), (k, e)
            for x, y in zip(pa, pb):
                assert np.array_equal(x.member_indices, y.member_indices) and np.array_equal(x.points, y.points)
                assert x.area_metric == y.area_metric and x.weight_sum == y.weight_sum, (k, e)

    for k in range(5):
        mpk = mp.copy()
        mpk[:, :3] += rng.uniform(-2e-4, 2e-4, size=(E, 3))  # a different step each call
        stats = host.collide_host(sp, mpk, cd)
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
        dev.collide(t(sp), t(mpk), t(cd))
        torch.cuda.synchronize()
        assert np.array_equal(stats, dev.stats.cpu().numpy())
        same(k)
    # the 12-value pose format: a new capture
    def pose12(p7):
        return np.stack([P.Transform.from_pose(p[:3], p[3:]).pose12() for p in p7])
    for _ in range(2):
        stats = host.collide_host(np.ascontiguousarray(pose12(sp)), np.ascontiguousarray(pose12(mp)), cd,
                                  pose_format=_native.CS_POSE12)
        dev.collide(torch.from_numpy(pose12(sp)).cuda(), torch.from_numpy(pose12(mp)).cuda(),
                    torch.from_numpy(cd).cuda(), pose_format=_native.CS_POSE12)
        torch.cuda.synchronize()
        assert np.array_equal(stats, dev.stats.cpu().numpy())
        same("pose12")
