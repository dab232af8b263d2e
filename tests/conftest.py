import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: longer-running check")


def golden(name: str):
    return np.load(os.path.join(GOLDEN, name))


@pytest.fixture(scope="session")
def meshes():
    return golden("meshes.npz")


@pytest.fixture(scope="session")
def grid64_npz():
    return golden("grid_bolt_r64.npz")


@pytest.fixture(scope="session")
def gen64():
    return golden("gen_r64.npz")


@pytest.fixture(scope="session")
def gen256():
    return golden("gen_r256.npz")


@pytest.fixture(scope="session")
def synth():
    return golden("red_synth.npz")


@pytest.fixture(scope="session")
def kat():
    return golden("kat.npz")


@pytest.fixture(scope="session")
def sdf_query():
    return golden("sdf_query.npz")


PATCH_KEYS = ("rep", "nkept", "member_offsets", "members", "kept_faces", "kept_points", "kept_normals",
              "kept_depths", "wsum", "wp", "wn", "wt", "area", "maxd")
CS_KEYS = ("points", "normals", "depths", "faces")


def pack_patch_list(patches, cap: int) -> dict:
    """Same layout as tests/golden/make_golden.py pack_patches()."""
    P = len(patches)
    K = max(cap, 1)
    d = {
        "rep": np.zeros((P, 3)), "nkept": np.zeros(P, np.int64), "kept_points": np.zeros((P, K, 3)),
        "kept_normals": np.zeros((P, K, 3)), "kept_depths": np.zeros((P, K)), "kept_faces": np.full((P, K), -1, np.int64),
        "wsum": np.zeros(P), "wp": np.zeros((P, 3)), "wn": np.zeros((P, 3)), "wt": np.zeros((P, 3)),
        "area": np.zeros(P), "maxd": np.zeros(P),
    }
    moff = [0]
    members = []
    for i, p in enumerate(patches):
        k = len(p)
        d["rep"][i] = p.representative_normal
        d["nkept"][i] = k
        d["kept_points"][i, :k] = p.points
        d["kept_normals"][i, :k] = p.normals
        d["kept_depths"][i, :k] = p.depths
        d["kept_faces"][i, :k] = p.face_indices
        members.extend(np.asarray(p.member_indices).tolist())
        moff.append(len(members))
        d["wsum"][i] = p.weight_sum
        d["wp"][i] = p.weighted_point_sum
        d["wn"][i] = p.weighted_normal_sum
        d["wt"][i] = p.weighted_torque_sum
        d["area"][i] = p.area_metric
        d["maxd"][i] = p.max_depth
    d["member_offsets"] = np.array(moff, np.int64)
    d["members"] = np.array(members, np.int64)
    return d


def assert_same(got: dict, ref, prefix: str, keys, label: str = "") -> None:
    """Bit-exact comparison (NaN-aware) of dict-of-arrays against golden npz entries."""
    for k in keys:
        a = np.asarray(got[k])
        b = np.asarray(ref[prefix + k])
        if k.startswith("kept_") and b.ndim >= 2 and a.ndim >= 2 and a.shape[1] != b.shape[1]:
            w = min(a.shape[1], b.shape[1])
            a, b = a[:, :w], b[:, :w]
        assert a.shape == b.shape, f"{label}{k}: shape {a.shape} != {b.shape}"
        if a.dtype.kind == "f":
            same = (a == b) | (np.isnan(a) & np.isnan(b))
        else:
            same = a == b
        if not same.all():
            bad = np.argwhere(~same)
            raise AssertionError(f"{label}{k}: {len(bad)} mismatches, first at {bad[:3].tolist()}: "
                                 f"{a[tuple(bad[0])]!r} vs {b[tuple(bad[0])]!r}")
