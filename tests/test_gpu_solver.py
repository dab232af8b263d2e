"""GPU parity of the contact solver (csrc/cs_solver.cu through
libcontactsim_b200.so): bit-exact against the reference's golden outputs
(tests/golden/solver.npz: ContactConstraints.build, gauss_seidel_sweeps,
body_wrenches) and, for the batched Plan.solve on collide's device-resident
reduced contacts, against the pinned oracle."""

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

G = golden("solver.npz")
CASES = [str(c) for c in G["cases"]]
BUILD_KEYS = ("ra", "rb", "tan1", "tan2", "kn", "kt1", "kt2", "bias_target", "restitution_target")


def case(name):
    return {k[len(name) + 1:]: G[k] for k in G.files if k.startswith(name + "_")}


def same(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and a.tobytes() == b.tobytes()


@pytest.fixture(scope="module")
def P():
    import paper_2205_03532_b200 as P
    from paper_2205_03532_b200 import _native

    _native.lib()
    return P


def rows_of(c):
    m = int(c["m"])
    return [{"body_a": int(c["body_a"][i]), "body_b": int(c["body_b"][i]), "point": c["point"][i],
             "normal": c["normal"][i], "depth": float(c["depth"][i]), "mu": float(c["mu"][i]),
             "restitution": float(c["restitution"][i]), "slop": float(c["slop"][i])} for i in range(m)]


@pytest.mark.parametrize("name", CASES)
def test_solver_dropin_matches_reference(P, name):
    """The reference's per-scene calls, one after the other as Scene._substep makes them."""
    from paper_2205_03532_b200.dynamics import ContactConstraints, SolverState

    c = case(name)
    nb = int(c["nb"])
    st = SolverState(nb)
    st.ref[...] = c["ref"]
    st.w_mat[...] = c["w_mat"]
    st.vel[...] = c["vel0"]
    con = ContactConstraints.build(rows_of(c), st, float(c["h"]), float(c["bias"]))
    for k in BUILD_KEYS:
        assert same(getattr(con, k), c[k].reshape(getattr(con, k).shape)), f"{name}: build {k}"
    pos_it, vel_it = (int(x) for x in c["iters"])
    con.position_sweeps(st, pos_it)
    assert same(st.vel, c["vel_pos"]) and same(st.impulse, c["imp_pos"]), name
    assert same(con.lam_n, c["lam_n"]), name
    con.velocity_sweeps(st, vel_it)
    assert same(st.vel, c["vel_end"]) and same(st.impulse, c["imp_end"]), name
    for k in ("lam_vel", "lam_t1", "lam_t2"):
        assert same(getattr(con, k), c[k]), f"{name}: {k}"
    assert same(con.body_wrenches(nb, float(c["h"])), c["wrench"]), name


def test_solver_batched_abi_ragged_systems(P):
    """Seven systems in single launches through the raw C ABI (CSR rows): the six
    golden M16 env systems (ragged row counts) and an empty one in the middle;
    build, position sweeps, velocity sweeps and wrenches each in one launch."""
    from paper_2205_03532_b200 import _native

    names = ["r64e0", "r64e1", "r64e2", None, "r256e0", "r256e1", "r256e2"]
    cs = [case(n) if n else None for n in names]
    c0 = cs[0]
    h, bias = float(c0["h"]), float(c0["bias"])
    pit, vit = (int(x) for x in c0["iters"])
    for c in cs:
        if c is not None:
            assert (float(c["h"]), float(c["bias"]), int(c["nb"])) == (h, bias, 2)
    S = len(cs)
    ms = [int(c["m"]) if c is not None else 0 for c in cs]
    off = np.concatenate([[0], np.cumsum(ms)]).astype(np.int64)
    R = int(off[-1])
    live = [c for c in cs if c is not None]
    cat = lambda k, shape: np.concatenate([np.asarray(c[k], np.float64).reshape(shape) for c in live])  # noqa: E731
    ref = np.zeros((S, 2, 3)); W = np.zeros((S, 2, 6, 6)); vel = np.zeros((S, 2, 6))
    for s, c in enumerate(cs):
        if c is not None:
            ref[s], W[s], vel[s] = c["ref"], c["w_mat"], c["vel0"]
        else:
            vel[s] = np.arange(12).reshape(2, 6)  # untouched: no rows
    d = lambda a, dt=torch.float64: torch.from_numpy(np.ascontiguousarray(a)).to(dt).cuda()  # noqa: E731
    ba = d(np.concatenate([c["body_a"] for c in live]).astype(np.int64), torch.int64)
    bb = d(np.concatenate([c["body_b"] for c in live]).astype(np.int64), torch.int64)
    point, normal = d(cat("point", (-1, 3))), d(cat("normal", (-1, 3)))
    depth, rest, slop, mu = (d(cat(k, (-1,))) for k in ("depth", "restitution", "slop", "mu"))
    outs = {k: torch.zeros((R, 3) if k in ("ra", "rb", "tan1", "tan2") else (R,), dtype=torch.float64,
                           device="cuda") for k in BUILD_KEYS}
    lam = {k: torch.zeros(R, dtype=torch.float64, device="cuda") for k in ("lam_n", "lam_vel", "lam_t1", "lam_t2")}
    dref, dW, dvel, doff = d(ref), d(W), d(vel), d(off, torch.int64)
    dimp = torch.zeros_like(dvel)
    wr = torch.zeros((S, 2, 6), dtype=torch.float64, device="cuda")
    st = _native.stream_handle()
    _native.call("cs_constraints_build", S, 2, doff.data_ptr(), ba.data_ptr(), bb.data_ptr(), point.data_ptr(),
                 normal.data_ptr(), depth.data_ptr(), rest.data_ptr(), slop.data_ptr(), dref.data_ptr(),
                 dW.data_ptr(), dvel.data_ptr(), h, bias, *(outs[k].data_ptr() for k in BUILD_KEYS), st)
    geo = (ba, bb, outs["ra"], outs["rb"], normal, outs["tan1"], outs["tan2"], outs["kn"], outs["kt1"], outs["kt2"])
    for it, target, ln, fr in ((pit, "bias_target", "lam_n", 1), (vit, "restitution_target", "lam_vel", 0)):
        _native.call("cs_gauss_seidel_sweeps", S, 2, doff.data_ptr(), it, dW.data_ptr(), dvel.data_ptr(),
                     dimp.data_ptr(), *(a.data_ptr() for a in geo), outs[target].data_ptr(), mu.data_ptr(),
                     lam[ln].data_ptr(), lam["lam_t1"].data_ptr(), lam["lam_t2"].data_ptr(), fr, st)
    _native.call("cs_body_wrenches", S, 2, doff.data_ptr(), ba.data_ptr(), bb.data_ptr(), outs["ra"].data_ptr(),
                 outs["rb"].data_ptr(), normal.data_ptr(), outs["tan1"].data_ptr(), outs["tan2"].data_ptr(),
                 lam["lam_n"].data_ptr(), lam["lam_vel"].data_ptr(), lam["lam_t1"].data_ptr(),
                 lam["lam_t2"].data_ptr(), h, wr.data_ptr(), st)
    got = {k: v.cpu().numpy() for k, v in outs.items()}
    gl = {k: v.cpu().numpy() for k, v in lam.items()}
    gv, gi, gw = dvel.cpu().numpy(), dimp.cpu().numpy(), wr.cpu().numpy()
    for s, c in enumerate(cs):
        if c is None:
            assert same(gv[s], vel[s]) and not gi[s].any() and not gw[s].any()
            continue
        a, b = off[s], off[s + 1]
        for k in BUILD_KEYS:
            assert same(got[k][a:b], c[k].reshape(got[k][a:b].shape)), (names[s], k)
        assert same(gv[s], c["vel_end"]) and same(gi[s], c["imp_end"]), names[s]
        for k in ("lam_n", "lam_vel", "lam_t1", "lam_t2"):
            assert same(gl[k][a:b], c[k]), (names[s], k)
        assert same(gw[s], c["wrench"]), names[s]


def test_plan_solve_matches_oracle(P, grid64_npz, meshes):
    """collide -> Plan.solve on the device-resident reduced contacts, against the
    oracle fed the same patches in Scene row order (scene.py:228-243)."""
    from oracle import oracle as O
    from paper_2205_03532_b200.dynamics import BatchedSolverState, SolverParams

    gen64 = golden("gen_r64.npz")
    d = grid64_npz
    grid = P.SignedDistanceGrid(d["origin"], float(d["voxel"]), d["dims"], d["values"], (d["aabb_lo"], d["aabb_hi"]))
    nut = P.TriMesh(meshes["nut_v"], meshes["nut_t"])
    envs = list(gen64["envs"])
    E = len(envs) * 3
    sp = np.concatenate([np.stack([gen64[f"e{e}_sdf_pose"] for e in envs])] * 3)
    mp = np.concatenate([np.stack([gen64[f"e{e}_mesh_pose"] for e in envs])] * 3)
    cd = np.full(E, float(gen64["cd"]))
    res = P.collide([P.register_sdf(grid)] * E, [P.register_mesh(nut)] * E, sp, mp, cd)
    plan = res.plan
    rng = np.random.default_rng(3)
    ref = np.zeros((E, 2, 3)); W = np.zeros((E, 2, 6, 6)); vel = np.zeros((E, 2, 6))
    for e in range(E):
        for b in range(2):
            if b == 0 and e % 3 == 0:
                continue  # static SDF body in a third of the envs
            m = rng.uniform(0.005, 0.05)
            ref[e, b] = mp[e, :3] if b else rng.standard_normal(3) * 1e-3
            W[e, b, :3, :3] = np.eye(3) / m
            A = rng.standard_normal((3, 3))
            W[e, b, 3:, 3:] = np.linalg.inv(A @ A.T * 1e-6 + np.eye(3) * 1e-7)
            vel[e, b] = rng.standard_normal(6) * np.array([0.05] * 3 + [0.5] * 3)
        vel[e, 1, 2] -= 0.4 + (e % 4) * 0.3  # some impacts above the restitution threshold
    mu = rng.uniform(0.0, 0.8, E); mu[::5] = 0.0
    rest = rng.uniform(0.0, 0.6, E)
    slop = np.full(E, 0.5 * float(d["voxel"]))
    st = BatchedSolverState.from_numpy(ref, W, vel)
    prm = SolverParams(dt=1 / 120, substeps=2, pos_iterations=10, vel_iterations=2)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float64)).cuda()  # noqa: E731
    wrench = plan.solve(st, t(mu), t(rest), t(slop), prm).cpu().numpy()
    gvel, gimp = st.vel.cpu().numpy(), st.impulse.cpu().numpy()
    n_kept = res.n_kept.cpu().numpy()
    h = prm.dt / prm.substeps
    for e in range(E):
        pt = res.patches(e)
        pts = np.concatenate([p.points for p in pt]) if pt else np.zeros((0, 3))
        nrm = np.concatenate([p.normals for p in pt]) if pt else np.zeros((0, 3))
        dep = np.concatenate([p.depths for p in pt]) if pt else np.zeros(0)
        m = len(dep)
        assert m == n_kept[e]
        a = np.zeros(m, np.int64); b = np.ones(m, np.int64)
        con = O.constraints_build(a, b, pts, nrm, dep, rest[e], slop[e], ref[e], W[e], vel[e], h, prm.bias_factor)
        rows = plan.solver_rows(e)
        for k in ("kn", "kt1", "kt2", "bias_target", "restitution_target", "ra", "rb", "tan1", "tan2"):
            assert same(rows[k], con[k]), (e, k)
        assert same(rows["point"], pts) and same(rows["depth"], dep), e
        v = np.array(vel[e]); imp = np.zeros((2, 6))
        lam = {k: np.zeros(m) for k in ("n", "t1", "t2", "v")}
        args = (a, b, con["ra"], con["rb"], nrm, con["tan1"], con["tan2"], con["kn"], con["kt1"], con["kt2"])
        if m:
            O.gauss_seidel_sweeps(prm.pos_iterations, W[e], v, imp, *args, con["bias_target"], mu[e], lam["n"],
                                  lam["t1"], lam["t2"], True)
            O.gauss_seidel_sweeps(prm.vel_iterations, W[e], v, imp, *args, con["restitution_target"], mu[e],
                                  lam["v"], lam["t1"], lam["t2"], False)
        assert same(gvel[e], v) and same(gimp[e], imp), e
        wr = O.body_wrenches(2, a, b, con["ra"], con["rb"], nrm, con["tan1"], con["tan2"], lam["n"], lam["v"],
                             lam["t1"], lam["t2"], h)
        assert same(wrench[e], wr), e


def test_solver_errors(P):
    from paper_2205_03532_b200 import _native

    with pytest.raises(ValueError):
        _native.call("cs_gauss_seidel_sweeps", 1, 99, 0, 1, *([0] * 18), 1, _native.stream_handle())
    from paper_2205_03532_b200.dynamics import SolverParams

    with pytest.raises(ValueError):
        SolverParams(dt=0.0)
    with pytest.raises(ValueError):
        SolverParams(vel_iterations=-1)


@pytest.mark.parametrize("nb", [6, 13, 40])
def test_solver_many_body_system_vs_oracle(P, nb):
    """Systems above four bodies take the shared-memory state path (6), above eight the
    global-memory one (13, 40: the reference has no body limit): random rows between
    dynamic and static bodies against the oracle."""
    from oracle import oracle as O
    from paper_2205_03532_b200.dynamics import ContactConstraints, SolverState

    rng = np.random.default_rng(21 + nb)
    m = 15 * nb
    st = SolverState(nb)
    for b in sorted({0, 2, nb - 1} | set(range(3, nb, 3))):  # the rigid-body mobility layout; the last a full 6x6
        mass = rng.uniform(0.01, 0.05)
        st.ref[b] = rng.standard_normal(3) * 0.01
        st.w_mat[b, :3, :3] = np.eye(3) / mass
        A = rng.standard_normal((3, 3))
        st.w_mat[b, 3:, 3:] = np.linalg.inv(A @ A.T * 1e-6 + np.eye(3) * 1e-7)
        st.vel[b] = rng.standard_normal(6) * 0.1
    B = rng.standard_normal((6, 6))
    st.w_mat[nb - 1] = B @ B.T * 10.0
    rows = []
    for c in range(m):
        a, b = rng.choice(nb, size=2, replace=False)
        n = rng.standard_normal(3)
        n /= np.linalg.norm(n)
        rows.append({"body_a": int(a), "body_b": int(b), "point": rng.standard_normal(3) * 0.01, "normal": n,
                     "depth": float(rng.uniform(-2e-4, 4e-4)), "mu": 0.5, "restitution": 0.3, "slop": 5e-5})
    vel0 = st.vel.copy()
    con = ContactConstraints.build(rows, st, 1 / 240, 0.2)
    con.position_sweeps(st, 10)
    con.velocity_sweeps(st, 2)
    wr = con.body_wrenches(nb, 1 / 240)
    ba = np.array([r["body_a"] for r in rows]); bb = np.array([r["body_b"] for r in rows])
    pts = np.array([r["point"] for r in rows]); nrm = np.array([r["normal"] for r in rows])
    dep = np.array([r["depth"] for r in rows])
    oc = O.constraints_build(ba, bb, pts, nrm, dep, 0.3, 5e-5, st.ref, st.w_mat, vel0, 1 / 240, 0.2)
    for k in ("kn", "kt1", "kt2", "bias_target", "restitution_target"):
        assert np.array_equal(getattr(con, k), oc[k]), k
    v, imp = np.array(vel0), np.zeros((nb, 6))
    ln, l1, l2, lv = (np.zeros(m) for _ in range(4))
    geo = (ba, bb, oc["ra"], oc["rb"], nrm, oc["tan1"], oc["tan2"], oc["kn"], oc["kt1"], oc["kt2"])
    O.gauss_seidel_sweeps(10, st.w_mat, v, imp, *geo, oc["bias_target"], 0.5, ln, l1, l2, True)
    O.gauss_seidel_sweeps(2, st.w_mat, v, imp, *geo, oc["restitution_target"], 0.5, lv, l1, l2, False)
    assert st.vel.tobytes() == v.tobytes() and st.impulse.tobytes() == imp.tobytes()
    assert con.lam_n.tobytes() == ln.tobytes() and con.lam_vel.tobytes() == lv.tobytes()
    owr = O.body_wrenches(nb, ba, bb, oc["ra"], oc["rb"], nrm, oc["tan1"], oc["tan2"], ln, lv, l1, l2, 1 / 240)
    assert np.array_equal(wr, owr)
