"""The drop-in boundary from plain C (examples/collide_demo.c): a C host registers
the grid and the mesh, runs one collide step through cs_collide_host and prints
per-env stats, which must equal the Python path's on the same inputs."""

import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT, golden

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def test_c_host_matches_python(tmp_path, grid64_npz, meshes):
    import paper_2205_03532_b200 as P
    from paper_2205_03532_b200 import _native

    _native.lib()
    exe = tmp_path / "collide_demo"
    lib_dir = os.path.dirname(_native.LIB_PATH)
    subprocess.run(["gcc", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"), os.path.join(ROOT, "examples",
                    "collide_demo.c"), "-L", lib_dir, "-lcontactsim_b200", f"-Wl,-rpath,{lib_dir}", "-o", str(exe)],
                   check=True)
    d, gen = grid64_npz, golden("gen_r64.npz")
    envs = list(gen["envs"])
    E = len(envs)
    sp = np.stack([gen[f"e{e}_sdf_pose"] for e in envs])
    mp = np.stack([gen[f"e{e}_mesh_pose"] for e in envs])
    cd = np.full(E, float(gen["cd"]))
    v, t = np.ascontiguousarray(meshes["nut_v"], np.float64), np.ascontiguousarray(meshes["nut_t"], np.int32)
    nx, ny, nz = (int(x) for x in d["dims"])
    blob = b"".join([
        np.array([len(v), len(t), nx, ny, nz, E], np.int64).tobytes(),
        np.concatenate([d["origin"], [float(d["voxel"])], d["aabb_lo"], d["aabb_hi"]]).astype(np.float64).tobytes(),
        v.tobytes(), t.tobytes(), np.ascontiguousarray(d["values"], np.float32).reshape(-1).tobytes(),
        sp.astype(np.float64).tobytes(), mp.astype(np.float64).tobytes(), cd.tobytes()])
    inp = tmp_path / "input.bin"
    inp.write_bytes(blob)
    out = subprocess.run([str(exe), str(inp)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    got = np.array([[float(x) for x in line.split()] for line in out.stdout.strip().splitlines()])
    grid = P.SignedDistanceGrid(d["origin"], float(d["voxel"]), d["dims"], d["values"], (d["aabb_lo"], d["aabb_hi"]))
    nut = P.TriMesh(v, t)  # registered handles live as long as their asset objects
    res = P.collide([P.register_sdf(grid)] * E, [P.register_mesh(nut)] * E, sp, mp, cd)
    ref = res.stats.cpu().numpy()
    assert got.shape == (E, 4)
    assert np.array_equal(got[:, :3], ref[:, :3].astype(np.float64))
    assert np.array_equal(got[:, 3].astype(np.float32), ref[:, 3])
    assert (got[:, 0] > 0).all()
