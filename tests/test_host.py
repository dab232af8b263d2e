"""Host-side logic on CPU: fixtures vs the reference meshes, parameter
validation, role assignment, seeded workloads, env sharding and the stats
all-gather over a world-size-2 gloo group."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import golden


def test_fixture_meshes_match_reference(meshes):
    from paper_2205_03532_b200.geometry import ThreadSpec, generate_iso_thread, generate_peg_hole

    nut = generate_iso_thread(ThreadSpec.standard("M16", "nut", "tight", segments_per_turn=80))
    bolt = generate_iso_thread(ThreadSpec.standard("M16", "bolt", "tight", segments_per_turn=80))
    peg, hole = generate_peg_hole(0.004, 0.104e-3, 0.03)
    for name, m in (("nut", nut), ("bolt", bolt), ("peg", peg), ("hole", hole)):
        assert np.array_equal(m.vertices, meshes[name + "_v"]), name
        assert np.array_equal(m.triangles, meshes[name + "_t"]), name
        assert m.is_watertight()
    assert (len(nut.vertices), len(nut.triangles)) == (8652, 17304)


def test_grid_layout_matches_reference(meshes):
    import json

    from paper_2205_03532_b200.geometry import TriMesh
    from paper_2205_03532_b200.sdf.grid import SdfResolutionSpec, grid_layout

    from conftest import GOLDEN

    meta = json.load(open(os.path.join(GOLDEN, "grids.json")))
    bolt = TriMesh(meshes["bolt_v"], meshes["bolt_t"])
    for res in (64, 128, 256):
        dims, origin, voxel = grid_layout(bolt, SdfResolutionSpec(res, 4))
        m = meta[f"bolt_r{res}"]
        assert list(dims) == m["dims"] and list(origin) == m["origin"] and voxel == m["voxel"]


def test_poses_match_golden_draw():
    from paper_2205_03532_b200.scenes import nut_poses

    p = golden("poses.npz")
    mine = nut_poses(64, 0, float(p["pitch"]), float(p["z0"]))
    np.testing.assert_allclose(mine, p["nut_pose"], rtol=0, atol=1e-15)


def test_reduction_params_validation():
    from paper_2205_03532_b200 import ReductionParams

    for kw in (dict(max_patches=0), dict(per_patch_cap=0), dict(normal_cone_cos=1.5), dict(batch_size=0)):
        with pytest.raises(ValueError):
            ReductionParams(**kw)
    c = ReductionParams(min_depth=-1e-4).to_c()
    assert c.max_patches == 128 and c.per_patch_cap == 6 and c.has_min_depth == 1 and c.min_depth == -1e-4


def test_assign_roles_rules():
    from paper_2205_03532_b200.contacts import BodyShape, assign_roles

    a, b = BodyShape(0, 100, True), BodyShape(1, 50, False)
    assert assign_roles(a, b).sdf_body == 0
    assert assign_roles(BodyShape(0, 10, False), BodyShape(1, 50, True)).sdf_body == 1
    p = assign_roles(BodyShape(3, 10, True), BodyShape(1, 10, True))
    assert (p.sdf_body, p.mesh_body, p.fallback) == (1, 3, False)
    p = assign_roles(BodyShape(0, 10, False), BodyShape(1, 20, False))
    assert (p.sdf_body, p.fallback) == (1, True)


def test_shard_ranges_partition():
    from paper_2205_03532_b200.scenes import shard_range

    for n in (1, 7, 1024, 1025):
        for world in (1, 2, 3, 8):
            cover = [i for r in range(world) for i in range(*shard_range(n, r, world))]
            assert cover == list(range(n))


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _gather_worker(rank, world, port, n_envs, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2205_03532_b200.distributed import env_shard, gather_env_stats, step_report

    lo, hi = env_shard(n_envs)
    local = torch.stack([torch.arange(lo, hi, dtype=torch.float32) + c for c in (0, 1000, 2000, 0.5)], dim=1)
    allst = gather_env_stats(local, n_envs)
    q.put((rank, allst.numpy(), step_report(allst)))
    dist.destroy_process_group()


def test_stats_allgather_gloo_world2():
    n_envs, world = 11, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, world, port, n_envs, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    expect = np.stack([np.arange(n_envs) + c for c in (0, 1000, 2000, 0.5)], axis=1).astype(np.float32)
    for rank, arr, rep in outs:
        assert np.array_equal(arr, expect)
        assert rep["contacts_before"] == int(expect[:, 0].sum())


def _bench(*args, env=None):
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    e = dict(os.environ, **(env or {}))
    e.pop("WORLD_SIZE", None) if env is None or "WORLD_SIZE" not in env else None
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), *args], capture_output=True, text=True,
                       timeout=300, env=e, cwd=root)
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    return r.returncode, (json.loads(lines[-1]) if lines else None), r.stderr


def test_bench_launcher_two_ranks():
    """`bench.py --gpus 2` outside torchrun launches two ranks (torch.distributed.run on
    127.0.0.1); they shard the envs and all-gather every env's stats in order (gloo)."""
    rc, out, err = _bench("--gpus", "2", "--dry-run", "--steps", "2", "--envs", "7")
    assert rc == 0, err[-2000:]
    assert out["n_gpus"] == 2 and out["envs_total"] == 14 and out["shards"] == [[0, 7], [7, 14]]
    assert out["gather_ok"] and out["scaling"] == "weak"


def test_bench_strong_scaling_shards():
    """--envs-total: the same total work split over the ranks (uneven shards padded in the gather)."""
    rc, out, err = _bench("--gpus", "2", "--dry-run", "--steps", "1", "--envs-total", "1023")
    assert rc == 0, err[-2000:]
    assert out["shards"] == [[0, 512], [512, 1023]] and out["scaling"] == "strong" and out["gather_ok"]


def test_bench_rejects_world_size_mismatch():
    rc, out, err = _bench("--gpus", "4", "--dry-run", env={"WORLD_SIZE": "1", "RANK": "0", "LOCAL_RANK": "0"})
    assert rc != 0 and "WORLD_SIZE" in err
