"""SDF on-disk format and cache on CPU, against a file the
REFERENCE wrote (tests/golden/make_sdf_file_golden.py: SignedDistanceGrid.save,
/root/reference/pkg/src/contactsim/sdf/grid.py:138-160) and the reference's
cache keys (cached_sdf, grid.py:247-267). Also the host-side plan cache."""

import json
import logging
import os
import sys

import numpy as np
import pytest

from conftest import GOLDEN, golden

REF_SRC = "/root/reference/pkg/src"


@pytest.fixture(scope="module")
def meta():
    return json.load(open(os.path.join(GOLDEN, "sdf_file.json")))


@pytest.fixture(scope="module")
def ref_file(meta):
    return os.path.join(GOLDEN, meta["file"])


def test_load_reference_written_file(ref_file):
    from paper_2205_03532_b200.sdf.grid import SignedDistanceGrid

    g = golden("grid_peg_r64.npz")
    grid = SignedDistanceGrid.load(ref_file)
    assert grid.dims == tuple(int(d) for d in g["dims"])
    assert np.array_equal(grid.values, g["values"].reshape(-1))
    assert np.array_equal(grid.origin, g["origin"]) and grid.voxel_size == float(g["voxel"])
    assert np.array_equal(grid.mesh_aabb[0], g["aabb_lo"]) and np.array_equal(grid.mesh_aabb[1], g["aabb_hi"])
    assert not grid.values.flags.writeable


def test_save_is_byte_identical_to_reference(ref_file, tmp_path):
    from paper_2205_03532_b200.sdf.grid import SignedDistanceGrid

    out = tmp_path / "ours.sdf"
    SignedDistanceGrid.load(ref_file).save(out)
    assert out.read_bytes() == open(ref_file, "rb").read()


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference sources not present")
def test_reference_loads_our_file(tmp_path):
    from paper_2205_03532_b200.sdf.grid import SignedDistanceGrid

    g = golden("grid_bolt_r64.npz")
    ours = SignedDistanceGrid(g["origin"], float(g["voxel"]), g["dims"], g["values"], (g["aabb_lo"], g["aabb_hi"]))
    ours.save(tmp_path / "b.sdf")
    sys.path.insert(0, REF_SRC)
    try:
        from contactsim.sdf.grid import SignedDistanceGrid as RefGrid
    finally:
        sys.path.remove(REF_SRC)
    ref = RefGrid.load(tmp_path / "b.sdf")
    assert tuple(ref.dims) == ours.dims and np.array_equal(ref.values, ours.values)
    assert np.array_equal(ref.origin, ours.origin) and ref.voxel_size == ours.voxel_size


def test_errors_match_reference(tmp_path, ref_file):
    from paper_2205_03532_b200.sdf.grid import SignedDistanceGrid

    bad = tmp_path / "bad.sdf"
    data = open(ref_file, "rb").read()
    bad.write_bytes(b"NOTASDF!" + data[8:])
    with pytest.raises(ValueError, match="not an SDF grid file"):
        SignedDistanceGrid.load(bad)
    short = tmp_path / "short.sdf"
    short.write_bytes(data[:-4])
    with pytest.raises(ValueError):
        SignedDistanceGrid.load(short)
    with pytest.raises(OSError):
        SignedDistanceGrid.load(tmp_path / "missing.sdf")


def test_cache_keys_match_reference(meta, meshes):
    from paper_2205_03532_b200.geometry import TriMesh

    for name, digest in meta["mesh_digests"].items():
        assert TriMesh(meshes[f"{name}_v"], meshes[f"{name}_t"]).content_digest() == digest, name


def _peg(meshes):
    from paper_2205_03532_b200.geometry import TriMesh

    return TriMesh(meshes["peg_v"], meshes["peg_t"])


def test_cached_sdf_hit_miss_and_unreadable(meshes, meta, ref_file, tmp_path, monkeypatch, caplog):
    from paper_2205_03532_b200.sdf import grid as G

    peg = _peg(meshes)
    spec = G.SdfResolutionSpec(64, 4)
    path = tmp_path / f"{meta['mesh_digests']['peg']}_r64_p4.sdf"
    calls = []
    ref = G.SignedDistanceGrid.load(ref_file)

    def fake_generate(mesh, s):
        calls.append(s)
        return ref

    monkeypatch.setattr(G, "generate_sdf", fake_generate)
    # no cache directory: always generated
    monkeypatch.delenv(G.CACHE_ENV_VAR, raising=False)
    G.cached_sdf(peg, spec)
    assert len(calls) == 1
    # a reference-written entry under the reference's key is a hit: not regenerated
    path.write_bytes(open(ref_file, "rb").read())
    hit = G.cached_sdf(peg, spec, cache_dir=tmp_path)
    assert len(calls) == 1 and np.array_equal(hit.values, ref.values)
    # the environment variable names the directory too
    monkeypatch.setenv(G.CACHE_ENV_VAR, str(tmp_path))
    G.cached_sdf(peg, spec)
    assert len(calls) == 1
    # an unreadable entry is discarded with a warning, regenerated and rewritten
    path.write_bytes(b"garbage!" + b"\0" * 200)
    with caplog.at_level(logging.WARNING, logger=G.log.name):
        G.cached_sdf(peg, spec, cache_dir=tmp_path)
    assert len(calls) == 2
    assert any("discarding unreadable SDF cache entry" in r.getMessage() for r in caplog.records)
    assert path.read_bytes() == open(ref_file, "rb").read()
    # a miss writes the entry (a new directory is created)
    sub = tmp_path / "new" / "dir"
    G.cached_sdf(peg, spec, cache_dir=sub)
    assert len(calls) == 3 and (sub / path.name).read_bytes() == open(ref_file, "rb").read()


def test_plan_cache_lru_threads_and_eviction():
    import threading

    from paper_2205_03532_b200.collide import PlanCache, evict_asset_plans

    c = PlanCache(maxsize=3)
    made = []

    def mk(tag):
        def f():
            made.append(tag)
            return object()
        return f

    a = c.get(("a",), mk("a"), (1,), (10,))
    assert c.get(("a",), mk("a2"), (1,), (10,)) is a and made == ["a"]
    c.get(("b",), mk("b"), (2,), (10,))
    c.get(("c",), mk("c"), (3,), (11,))
    c.get(("a",), mk("-"), (1,), (10,))  # a is now most recent
    c.get(("d",), mk("d"), (4,), (12,))  # evicts b (least recent)
    assert len(c) == 3 and made == ["a", "b", "c", "d"]
    c.get(("b",), mk("b2"), (2,), (10,))
    assert made[-1] == "b2"
    # another thread never shares this thread's plans
    box = []
    t = threading.Thread(target=lambda: box.append(c.get(("a",), mk("a-t"), (1,), (10,))))
    t.start()
    t.join()
    assert box[0] is not a and made[-1] == "a-t"
    # finalising an asset drops every plan that names it
    evict_asset_plans(mesh=10)
    assert all(10 not in m for (_, m) in c._assets.values())
    evict_asset_plans(sdf=4)
    assert all(4 not in s for (s, _) in c._assets.values())
    c.clear()
    assert len(c) == 0
