"""The REFERENCE's own CPU path, timed on the host cores.

This is the unmodified reference package (`contactsim`, pkg/src/contactsim), installed
once as a build artefact with

    python -m pip install --no-index --no-build-isolation --no-deps \
        --find-links /opt/wheelhouse --target baseline/_ref <copy of /root/reference/pkg>

(`baseline/_ref` is git-ignored; it travels to the GPU box with the repo snapshot).
Nothing here imports this repo's package or its CUDA library: assets are built with
the reference's own `generate_iso_thread` / `generate_sdf`, and each env is
`generate_contacts` + `reduce_contacts` called exactly as `Scene._collect_contacts`
does (pkg/src/contactsim/dynamics/scene.py:206-226): cd = 2 voxel,
ReductionParams(min_depth=-cd).

Modes:
  A: serial env loop in this process, numba's own thread pool (NUMBA_NUM_THREADS = cores);
  B: a process pool of `cores` workers over env shards, NUMBA_NUM_THREADS=1 each.
The first (JIT) call of every process is discarded.
"""

from __future__ import annotations

import multiprocessing as mp
import os
import sys
import tempfile
import time

import numpy as np

REF_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_ref")


def cores() -> int:
    return len(os.sched_getaffinity(0))


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _import_ref():
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tempfile.gettempdir(), "cs_ref_numba_cache"))
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import contactsim  # noqa: F401  (the reference package)

    return contactsim


def available() -> str | None:
    """None if the reference package imports from baseline/_ref, else the reason."""
    if not os.path.isdir(os.path.join(REF_DIR, "contactsim")):
        return "baseline/_ref (pip install of the reference) is absent"
    try:
        _import_ref()
    except Exception as exc:  # noqa: BLE001
        return f"reference import failed: {exc!r}"
    return None


def build_assets(res: int = 256, segments_per_turn: int = 80):
    """The headline assets with the reference's own generators (one-time setup, untimed)."""
    _import_ref()
    from contactsim.geometry.threads import ThreadSpec, bolt_thread_base_z, generate_iso_thread
    from contactsim.sdf.grid import SdfResolutionSpec, generate_sdf

    nut = generate_iso_thread(ThreadSpec.standard("M16", "nut", "tight", segments_per_turn=segments_per_turn))
    bolt_spec = ThreadSpec.standard("M16", "bolt", "tight", segments_per_turn=segments_per_turn)
    bolt = generate_iso_thread(bolt_spec)
    grid = generate_sdf(bolt, SdfResolutionSpec(res, 4))
    return {"nut": nut, "grid": grid, "bolt_tris": len(bolt), "pitch": bolt_spec.pitch,
            "z0": float(bolt_thread_base_z(bolt_spec))}


def assets_from_arrays(values, dims, origin, voxel, lo, hi, nut_v, nut_t, bolt_tris: int):
    """The reference's SignedDistanceGrid / TriMesh around given arrays (a grid that
    generate_sdf produced elsewhere, e.g. the GPU arm's bit-identical one)."""
    _import_ref()
    from contactsim.geometry.mesh import TriMesh
    from contactsim.sdf.grid import SignedDistanceGrid

    grid = SignedDistanceGrid(np.asarray(origin), float(voxel), tuple(int(d) for d in dims), np.asarray(values),
                              (np.asarray(lo), np.asarray(hi)))
    return {"nut": TriMesh(nut_v, nut_t), "grid": grid, "bolt_tris": int(bolt_tris)}


def nut_poses(n: int, seed: int, pitch: float, z0: float) -> np.ndarray:
    """The SURVEY §8(d) pose distribution (the GPU arm's paper_2205_03532_b200.scenes.nut_poses),
    drawn with the reference's own quaternion helpers (math3d.py)."""
    _import_ref()
    from contactsim.math3d import quat_from_axis_angle, quat_multiply

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


def _collect(grid, nut, sdf7, mesh7, bolt_tris=1):
    """One env, as Scene._collect_contacts (scene.py:206-226). Returns (t_gen, t_red, n_cand)."""
    from contactsim.contacts.generation import BodyShape, assign_roles, generate_contacts
    from contactsim.contacts.reduction import reduce_contacts
    from contactsim.contacts.types import ReductionParams
    from contactsim.math3d import Transform

    pairing = assign_roles(BodyShape(0, bolt_tris, True), BodyShape(1, len(nut), False))  # bolt = SDF body
    cd = 2.0 * grid.voxel_size
    t0 = time.perf_counter()
    cs = generate_contacts(pairing, grid, nut, Transform.from_pose(sdf7[:3], sdf7[3:]),
                           Transform.from_pose(mesh7[:3], mesh7[3:]), cd)
    t1 = time.perf_counter()
    reduce_contacts(cs, ReductionParams(min_depth=-cd))
    t2 = time.perf_counter()
    return t1 - t0, t2 - t1, len(cs)


_W = {}


def _worker_init(grid_file, meta, nut_file):
    os.environ["NUMBA_NUM_THREADS"] = "1"
    _import_ref()
    from contactsim.geometry.mesh import TriMesh
    from contactsim.sdf.grid import SignedDistanceGrid

    vals = np.load(grid_file)
    g = SignedDistanceGrid(meta["origin"], meta["voxel"], meta["dims"], vals, (meta["lo"], meta["hi"]))
    d = np.load(nut_file)
    nut = TriMesh(d["v"], d["t"])
    _W["grid"], _W["nut"], _W["bt"] = g, nut, meta["bolt_tris"]
    _collect(g, nut, meta["warm_sdf"], meta["warm_mesh"], meta["bolt_tris"])  # JIT / first call, discarded


def _worker_env(args):
    sdf7, mesh7 = args
    return _collect(_W["grid"], _W["nut"], sdf7, mesh7, _W["bt"])


def mode_b(assets, sdf7, mesh7, n_proc: int | None = None) -> dict:
    """Mode B: n_proc worker processes (1 numba thread each) over the envs."""
    n_proc = n_proc or cores()
    grid, nut = assets["grid"], assets["nut"]
    tmp = tempfile.mkdtemp(prefix="cs_ref_")
    gf, nf = os.path.join(tmp, "grid.npy"), os.path.join(tmp, "nut.npz")
    np.save(gf, np.asarray(grid.values))
    np.savez(nf, v=nut.vertices, t=nut.triangles)
    lo, hi = grid.mesh_aabb
    meta = {"origin": np.asarray(grid.origin), "voxel": float(grid.voxel_size), "dims": tuple(grid.dims),
            "lo": np.asarray(lo), "hi": np.asarray(hi), "warm_sdf": sdf7[0], "warm_mesh": mesh7[0],
            "bolt_tris": assets["bolt_tris"]}
    ctx = mp.get_context("spawn")
    # one thread per worker: numba's pool and the BLAS pools (numpy @ in the reduction)
    # inherit these before the spawned workers load them
    one = ("NUMBA_NUM_THREADS", "OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS")
    saved = {k: os.environ.get(k) for k in one}
    for k in one:
        os.environ[k] = "1"
    try:
        with ctx.Pool(n_proc, initializer=_worker_init, initargs=(gf, meta, nf)) as pool:
            pool.map(_worker_env, [(sdf7[0], mesh7[0])] * n_proc)  # every worker warm
            t0 = time.perf_counter()
            res = pool.map(_worker_env, list(zip(sdf7, mesh7)), chunksize=1)
            wall = time.perf_counter() - t0
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    g = np.array([r[0] for r in res]); r_ = np.array([r[1] for r in res]); c = np.array([r[2] for r in res])
    return {"mode": "B", "procs": n_proc, "envs": len(res), "wall_s": wall, "ms_per_env_wall": wall / len(res) * 1e3,
            "gen_ms_per_env_core": float(g.mean() * 1e3), "red_ms_per_env_core": float(r_.mean() * 1e3),
            "candidates_per_env": float(c.mean())}


def mode_a(assets, sdf7, mesh7) -> dict:
    """Mode A: a serial env loop in this process (numba threads = its default pool)."""
    grid, nut = assets["grid"], assets["nut"]
    bt = assets["bolt_tris"]
    _collect(grid, nut, sdf7[0], mesh7[0], bt)  # JIT, discarded
    t0 = time.perf_counter()
    res = [_collect(grid, nut, s, m, bt) for s, m in zip(sdf7, mesh7)]
    wall = time.perf_counter() - t0
    g = np.array([r[0] for r in res]); r_ = np.array([r[1] for r in res])
    from numba import config

    return {"mode": "A", "numba_threads": int(config.NUMBA_NUM_THREADS), "envs": len(res), "wall_s": wall,
            "ms_per_env_wall": wall / len(res) * 1e3, "gen_ms_per_env": float(g.mean() * 1e3),
            "red_ms_per_env": float(r_.mean() * 1e3)}


def measure(assets, sdf7, mesh7, faces: int, envs_b: int, envs_a: int) -> dict:
    """Both modes on bounded samples of the workload; the faster one is the baseline."""
    b = mode_b(assets, sdf7[:envs_b], mesh7[:envs_b])
    a = mode_a(assets, sdf7[:envs_a], mesh7[:envs_a])
    best = b if b["ms_per_env_wall"] <= a["ms_per_env_wall"] else a
    return {"value": faces / (best["ms_per_env_wall"] * 1e-3), "unit": "queries/s", "cores": cores(),
            "cpu_model": cpu_model(), "best_mode": best["mode"],
            "ms_per_1024_envs": best["ms_per_env_wall"] * 1024, "mode_a": a, "mode_b": b}
