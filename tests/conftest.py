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
def merge():
    """Reduction cases that take _add_patch's merge branch (tests/golden/make_merge_golden.py)."""
    return golden("red_merge.npz")


@pytest.fixture(scope="session")
def nan_cases():
    """Reduction cases with NaN points, normals and depths (tests/golden/make_nan_golden.py)."""
    return golden("red_nan.npz")


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


_DIG_K = np.uint64(0x9E3779B97F4A7C15)


def _digest_words(words: np.ndarray) -> int:
    w = np.ascontiguousarray(words).view(np.uint64)
    i = np.arange(len(w), dtype=np.uint64)
    with np.errstate(over="ignore"):
        return int(np.sum((w ^ _DIG_K) * (np.uint64(2) * i + np.uint64(1)), dtype=np.uint64))


def digest_env(P, Nn, D, F, rep, nk, kept, moff, mem, ws, wp, wn, wt, ar, md) -> int:
    """One env's digest from its candidate arrays (C rows) and patch arrays (q patches;
    kept/members as candidate indices): the word stream of og_collide_digest."""
    u = lambda a: np.asarray(a, dtype=np.int64).view(np.uint64).ravel()  # noqa: E731
    f = lambda a: np.asarray(a, dtype=np.float64).view(np.uint64).ravel()  # noqa: E731
    c = len(D)
    parts = [u([c]), f(P), f(Nn), f(D), u(F)]
    q = len(nk) if c > 0 else 0
    parts.append(u([q]))
    for j in range(q):
        m0, m1 = int(moff[j]), int(moff[j + 1])
        parts += [f(rep[j]), u([nk[j]]), u(kept[j][: nk[j]]), u([m1 - m0]), u(mem[m0:m1]), f([ws[j]]), f(wp[j]),
                  f(wn[j]), f(wt[j]), f([ar[j]]), f([md[j]])]
    return _digest_words(np.concatenate(parts))


def env_digests(plan) -> np.ndarray:
    """Per env digest of every output of a collide (the word stream of the oracle's
    og_collide_digest, oracle/cs_oracle.c): candidates, then per patch the normal,
    kept candidates, members, aggregates, area and max depth."""
    E = plan.n_envs
    base = plan.cand_base.cpu().numpy()
    nc = plan.n_cand.cpu().numpy().astype(np.int64)
    npch = plan.n_patch.cpu().numpy().astype(np.int64)
    P, Nn, D = plan.cand_point.cpu().numpy(), plan.cand_normal.cpu().numpy(), plan.cand_depth.cpu().numpy()
    F = plan.cand_face.cpu().numpy()
    rep, nk, kc = plan.patch_normal.cpu().numpy(), plan.patch_nkept.cpu().numpy(), plan.kept_cand.cpu().numpy()
    mo, mem = plan.member_offsets.cpu().numpy(), plan.members.cpu().numpy()
    ws, wp, wn, wt = (plan.w_sum.cpu().numpy(), plan.wp_sum.cpu().numpy(), plan.wn_sum.cpu().numpy(),
                      plan.wt_sum.cpu().numpy())
    ar, md = plan.area.cpu().numpy(), plan.max_depth.cpu().numpy()
    out = np.zeros(E, np.uint64)
    for e in range(E):
        b, c, q = int(base[e]), int(nc[e]), int(npch[e])
        out[e] = digest_env(P[b:b + c], Nn[b:b + c], D[b:b + c], F[b:b + c], rep[e, :q], nk[e, :q], kc[e, :q],
                            mo[e, : q + 1], mem[b:b + c], ws[e, :q], wp[e, :q], wn[e, :q], wt[e, :q], ar[e, :q],
                            md[e, :q])
    return out
