"""ORACLE — test infrastructure only.

ctypes front end for oracle/cs_oracle.c, the plain-C restatement of the
reference hot path (contactsim generate_contacts / reduce_contacts and the
SDF sampling kernels), and oracle/cs_oracle_solver.c, the contact solver that
consumes its output (dynamics/solver.py ContactConstraints.build,
dynamics/_kernels.py gauss_seidel_sweeps). Imported only by tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline leg, as the checker. The product package never imports
this module.

Each function cites the reference code it restates; tests/test_oracle.py pins
every one of them bit-for-bit against tests/golden/ (outputs of the reference).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "libcs_oracle.so")

_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _SO


def lib():
    global _lib
    if _lib is None:
        srcs = [os.path.join(_HERE, f) for f in ("cs_oracle.c", "cs_oracle_solver.c", "cs_oracle_broadphase.c")]
        if not os.path.exists(_SO) or os.path.getmtime(_SO) < max(os.path.getmtime(f) for f in srcs if os.path.exists(f)):
            build()
        _lib = ctypes.CDLL(_SO)
        _lib.og_generate_contacts.restype = ctypes.c_int64
        _lib.og_reduce_contacts.restype = ctypes.c_int
        _lib.og_num_threads.restype = ctypes.c_int
        _lib.og_sum.restype = ctypes.c_double
        _lib.og_broadphase.restype = ctypes.c_int64
    return _lib


def _p(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


class Grid:
    """Just the fields of contactsim.sdf.grid.SignedDistanceGrid the path reads (grid.py:48-68)."""

    def __init__(self, values, dims, origin, voxel, aabb_lo, aabb_hi):
        self.values = np.ascontiguousarray(values, dtype=np.float32).reshape(-1)
        self.dims = tuple(int(d) for d in dims)
        self.origin = _f64(origin)
        self.voxel = float(voxel)
        self.aabb_lo = _f64(aabb_lo)
        self.aabb_hi = _f64(aabb_hi)

    @classmethod
    def from_npz(cls, d) -> "Grid":
        return cls(d["values"], d["dims"], d["origin"], float(d["voxel"]), d["aabb_lo"], d["aabb_hi"])

    def _args(self):
        nx, ny, nz = self.dims
        return [_p(self.values), ctypes.c_int64(nx), ctypes.c_int64(ny), ctypes.c_int64(nz),
                ctypes.c_double(self.origin[0]), ctypes.c_double(self.origin[1]), ctypes.c_double(self.origin[2]),
                ctypes.c_double(self.voxel)]


def sample(grid: Grid, points) -> np.ndarray:
    """sample_batch (sdf/_kernels.py:330-335) at grid-frame points."""
    pts = _f64(points).reshape(-1, 3)
    out = np.empty(len(pts))
    lib().og_sample_batch(*grid._args(), _p(pts), ctypes.c_int64(len(pts)), _p(out))
    return out


def gradient(grid: Grid, points) -> np.ndarray:
    """gradient_batch (sdf/_kernels.py:338-346), unnormalised."""
    pts = _f64(points).reshape(-1, 3)
    out = np.empty((len(pts), 3))
    lib().og_gradient_batch(*grid._args(), _p(pts), ctypes.c_int64(len(pts)), _p(out))
    return out


def face_contacts(grid: Grid, tri_verts, contact_distance, max_iters=12, tol=None):
    """numba face_contacts (contacts/_kernels.py:11-87); returns (point, phi, grad, found)."""
    tv = _f64(tri_verts).reshape(-1, 3, 3)
    m = len(tv)
    tol = 0.1 * grid.voxel if tol is None else tol
    op = np.zeros((m, 3))
    ophi = np.zeros(m)
    ogr = np.zeros((m, 3))
    ofd = np.zeros(m, np.uint8)
    lib().og_face_contacts(*grid._args(), _p(tv), ctypes.c_int64(m), ctypes.c_double(contact_distance),
                           ctypes.c_int(max_iters), ctypes.c_double(tol), _p(op), _p(ophi), _p(ogr), _p(ofd))
    return op, ophi, ogr, ofd


def quat_to_matrix(q) -> np.ndarray:
    q = _f64(q)
    R = np.empty(9)
    lib().og_quat_to_matrix(_p(q), _p(R))
    return R.reshape(3, 3)


def to_grid(sdf_pose7, mesh_pose7):
    """sdf_pose.inverse().compose(mesh_pose) (generation.py:70)."""
    s, m = _f64(sdf_pose7), _f64(mesh_pose7)
    R = np.empty(9)
    t = np.empty(3)
    lib().og_to_grid(_p(s), _p(m), _p(R), _p(t))
    return R.reshape(3, 3), t


def tri_verts(sdf_pose7, mesh_pose7, vertices, triangles) -> np.ndarray:
    """verts_grid[triangles] as generate_contacts builds it (generation.py:70-72)."""
    v = _f64(vertices)
    t = np.ascontiguousarray(triangles, dtype=np.int32)
    out = np.empty((len(t), 3, 3))
    lib().og_tri_verts(_p(_f64(sdf_pose7)), _p(_f64(mesh_pose7)), _p(v), ctypes.c_int64(len(v)), _p(t),
                       ctypes.c_int64(len(t)), _p(out))
    return out


def generate_contacts(grid: Grid, vertices, triangles, sdf_pose7, mesh_pose7, contact_distance, threads=True):
    """generate_contacts (generation.py:54-114): dict(points, normals, depths, faces)."""
    v = _f64(vertices)
    t = np.ascontiguousarray(triangles, dtype=np.int32)
    nt = len(t)
    pts = np.empty((max(nt, 1), 3))
    nrm = np.empty((max(nt, 1), 3))
    dep = np.empty(max(nt, 1))
    fac = np.empty(max(nt, 1), np.int64)
    c = lib().og_generate_contacts(*grid._args(), _p(grid.aabb_lo), _p(grid.aabb_hi), _p(v), ctypes.c_int64(len(v)),
                                   _p(t), ctypes.c_int64(nt), _p(_f64(sdf_pose7)), _p(_f64(mesh_pose7)),
                                   ctypes.c_double(contact_distance), _p(pts), _p(nrm), _p(dep), _p(fac),
                                   ctypes.c_int(1 if threads else 0))
    if c == -2:
        raise ValueError("contact_distance must be non-negative")
    if c == -1:
        raise RuntimeError("non-finite pose in contact generation")
    return {"points": pts[:c].copy(), "normals": nrm[:c].copy(), "depths": dep[:c].copy(), "faces": fac[:c].copy()}


def reduce_contacts(points, normals, depths, faces=None, max_patches=128, per_patch_cap=6,
                    normal_cone_cos=float(np.cos(np.radians(20.0))), min_depth=None, batch_size=1024) -> dict:
    """reduce_contacts (reduction.py:45-236); same dict layout as tests/golden pack_patches()."""
    P = _f64(points).reshape(-1, 3)
    Nn = _f64(normals).reshape(-1, 3)
    D = _f64(depths).reshape(-1)
    n = len(D)
    N, K = int(max_patches), int(per_patch_cap)
    rep = np.zeros((N, 3))
    nkept = np.zeros(N, np.int64)
    kept = np.full((N, K), -1, np.int64)
    moff = np.zeros(N + 1, np.int64)
    members = np.zeros(max(n, 1), np.int64)
    wsum = np.zeros(N)
    wp = np.zeros((N, 3))
    wn = np.zeros((N, 3))
    wt = np.zeros((N, 3))
    area = np.zeros(N)
    maxd = np.zeros(N)
    npatch = lib().og_reduce_contacts(
        ctypes.c_int64(n), _p(P), _p(Nn), _p(D), ctypes.c_int(N), ctypes.c_int(K), ctypes.c_double(normal_cone_cos),
        ctypes.c_double(0.0 if min_depth is None else min_depth), ctypes.c_int(0 if min_depth is None else 1),
        ctypes.c_int(int(batch_size)), _p(rep), _p(nkept), _p(kept), _p(moff), _p(members), _p(wsum), _p(wp),
        _p(wn), _p(wt), _p(area), _p(maxd))
    q = npatch
    out = {
        "rep": rep[:q], "nkept": nkept[:q], "kept": kept[:q], "member_offsets": moff[: q + 1],
        "members": members[: moff[q]], "wsum": wsum[:q], "wp": wp[:q], "wn": wn[:q], "wt": wt[:q],
        "area": area[:q], "maxd": maxd[:q],
    }
    kidx = np.where(out["kept"] >= 0, out["kept"], 0)
    mask = out["kept"] >= 0
    out["kept_points"] = np.where(mask[..., None], P[kidx], 0.0)
    out["kept_normals"] = np.where(mask[..., None], Nn[kidx], 0.0)
    out["kept_depths"] = np.where(mask, D[kidx], 0.0)
    if faces is not None:
        F = np.asarray(faces, dtype=np.int64)
        out["kept_faces"] = np.where(mask, F[kidx], -1)
    return out


class EnvStats(ctypes.Structure):
    _fields_ = [("n_cand", ctypes.c_int64), ("n_patch", ctypes.c_int64), ("n_kept", ctypes.c_int64),
                ("max_depth", ctypes.c_double)]


def collide_batched(grid: Grid, vertices, triangles, sdf_pose7, mesh_pose7, contact_distance, max_patches=128,
                    per_patch_cap=6, normal_cone_cos=float(np.cos(np.radians(20.0))), batch_size=1024) -> np.ndarray:
    """Per env generate_contacts + reduce_contacts as Scene._collect_contacts does
    (dynamics/scene.py:206-226), OpenMP over envs. Returns (E, 4) stats
    [n_cand, n_patch, n_kept, max_kept_depth]."""
    s7 = _f64(sdf_pose7).reshape(-1, 7)
    m7 = _f64(mesh_pose7).reshape(-1, 7)
    E = len(m7)
    cd = _f64(np.broadcast_to(np.asarray(contact_distance, dtype=np.float64), (E,)))
    v = _f64(vertices)
    t = np.ascontiguousarray(triangles, dtype=np.int32)
    stats = (EnvStats * E)()
    lib().og_collide_batched(ctypes.c_int64(E), *grid._args(), _p(grid.aabb_lo), _p(grid.aabb_hi), _p(v),
                             ctypes.c_int64(len(v)), _p(t), ctypes.c_int64(len(t)), _p(s7), _p(m7), _p(cd),
                             ctypes.c_int(max_patches), ctypes.c_int(per_patch_cap), ctypes.c_double(normal_cone_cos),
                             ctypes.c_int(batch_size), stats)
    return np.array([[s.n_cand, s.n_patch, s.n_kept, s.max_depth] for s in stats], dtype=np.float64)


def collide_digest(grid: Grid, vertices, triangles, sdf_pose7, mesh_pose7, contact_distance, max_patches=128,
                   per_patch_cap=6, normal_cone_cos=float(np.cos(np.radians(20.0))), batch_size=1024) -> np.ndarray:
    """Per env digest (uint64) of every output of generate_contacts + reduce_contacts
    (og_collide_digest; the word stream is documented there), OpenMP over envs."""
    s7 = _f64(sdf_pose7).reshape(-1, 7)
    m7 = _f64(mesh_pose7).reshape(-1, 7)
    E = len(m7)
    cd = _f64(np.broadcast_to(np.asarray(contact_distance, dtype=np.float64), (E,)))
    v = _f64(vertices)
    t = np.ascontiguousarray(triangles, dtype=np.int32)
    out = np.zeros(E, np.uint64)
    lib().og_collide_digest(ctypes.c_int64(E), *grid._args(), _p(grid.aabb_lo), _p(grid.aabb_hi), _p(v),
                            ctypes.c_int64(len(v)), _p(t), ctypes.c_int64(len(t)), _p(s7), _p(m7), _p(cd),
                            ctypes.c_int(max_patches), ctypes.c_int(per_patch_cap), ctypes.c_double(normal_cone_cos),
                            ctypes.c_int(batch_size), _p(out))
    return out


def num_threads() -> int:
    return int(lib().og_num_threads())


# ---------------------------------------------------------------- contact solver (cs_oracle_solver.c)

def _i64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


def constraints_build(body_a, body_b, point, normal, depth, restitution, slop, ref, w_mat, vel, h, bias_factor):
    """ContactConstraints.build (dynamics/solver.py:105-141) for one system; rows in
    sweep order. Returns dict of ra, rb, tan1, tan2, kn, kt1, kt2, bias_target,
    restitution_target."""
    m = len(depth)
    ba, bb = _i64(body_a), _i64(body_b)
    pt, nr = _f64(point).reshape(m, 3), _f64(normal).reshape(m, 3)
    dep = _f64(depth)
    rest = _f64(np.broadcast_to(np.asarray(restitution, dtype=np.float64), (m,)))
    sl = _f64(np.broadcast_to(np.asarray(slop, dtype=np.float64), (m,)))
    ref_, W, v = _f64(ref), _f64(w_mat), _f64(vel)
    out = {k: np.zeros((m, 3)) for k in ("ra", "rb", "tan1", "tan2")}
    out.update({k: np.zeros(m) for k in ("kn", "kt1", "kt2", "bias_target", "restitution_target")})
    lib().og_constraints_build(ctypes.c_int64(m), _p(ba), _p(bb), _p(pt), _p(nr), _p(dep), _p(rest), _p(sl),
                               _p(ref_), _p(W), _p(v), ctypes.c_double(h), ctypes.c_double(bias_factor),
                               *(_p(out[k]) for k in ("ra", "rb", "tan1", "tan2", "kn", "kt1", "kt2", "bias_target",
                                                       "restitution_target")))
    return out


def gauss_seidel_sweeps(iters, w_mat, vel, imp, body_a, body_b, ra, rb, nrm, tan1, tan2, kn, kt1, kt2, target_vn,
                        mu, lam_n, lam_t1, lam_t2, with_friction):
    """dynamics/_kernels.py:52-115, same argument list; vel, imp, lam_* are updated
    in place (they must be C-contiguous float64 arrays)."""
    m = len(kn)
    for a in (vel, imp, lam_n, lam_t1, lam_t2):
        assert a.dtype == np.float64 and a.flags.c_contiguous
    ba, bb = _i64(body_a), _i64(body_b)
    args = [_f64(x) for x in (ra, rb, nrm, tan1, tan2, kn, kt1, kt2, target_vn,
                              np.broadcast_to(np.asarray(mu, dtype=np.float64), (m,)))]
    W = _f64(w_mat)
    lib().og_gauss_seidel_sweeps(ctypes.c_int64(iters), _p(W), _p(vel), _p(imp), ctypes.c_int64(m), _p(ba),
                                 _p(bb), *(_p(a) for a in args), _p(lam_n), _p(lam_t1), _p(lam_t2),
                                 ctypes.c_int(1 if with_friction else 0))


def body_wrenches(n_bodies, body_a, body_b, ra, rb, nrm, tan1, tan2, lam_n, lam_vel, lam_t1, lam_t2, h):
    """ContactConstraints.body_wrenches (dynamics/solver.py:154-163)."""
    m = len(lam_n)
    out = np.zeros((n_bodies, 6))
    ba, bb = _i64(body_a), _i64(body_b)
    arrs = [_f64(x) for x in (ra, rb, nrm, tan1, tan2, lam_n, lam_vel, lam_t1, lam_t2)]
    lib().og_body_wrenches(ctypes.c_int64(m), _p(ba), _p(bb), *(_p(a) for a in arrs),
                           ctypes.c_double(h), _p(out))
    return out


# ---------------------------------------------------------------- broadphase (cs_oracle_broadphase.c)

def world_aabb(mesh_lo, mesh_hi, pose7):
    """RigidBody.world_aabb (dynamics/body.py:77-83) for n bodies: (lo, hi) (n, 3)."""
    ml, mh, p = _f64(mesh_lo).reshape(-1, 3), _f64(mesh_hi).reshape(-1, 3), _f64(pose7).reshape(-1, 7)
    n = len(ml)
    lo, hi = np.zeros((n, 3)), np.zeros((n, 3))
    lib().og_world_aabb(ctypes.c_int64(n), _p(ml), _p(mh), _p(p), _p(lo), _p(hi))
    return lo, hi


def broadphase_pairs(lo, hi, ids, margin):
    """geometry/broadphase.py:25-44 for one scene: (P, 2) int64 sorted (id_a, id_b)."""
    lo_, hi_ = _f64(lo).reshape(-1, 3), _f64(hi).reshape(-1, 3)
    ids_ = _i64(ids)
    n = len(ids_)
    out = np.zeros((max(n * (n - 1) // 2, 1), 2), np.int64)
    k = lib().og_broadphase(ctypes.c_int64(n), _p(lo_), _p(hi_), _p(ids_), ctypes.c_double(margin), _p(out))
    if k < 0:
        raise ValueError("non-finite AABB in broadphase input")
    return out[:k]
