"""Batched collide: SDF contact generation + contact reduction for E envs per call.

This is the vectorised body of contactsim's per-pair loop in
Scene._collect_contacts (/root/reference/pkg/src/contactsim/dynamics/scene.py:188-227):
for every env e, generate_contacts(sdf_e, mesh_e, poses_e, cd_e) followed by
reduce_contacts(candidates, ReductionParams(min_depth=-cd_e)). Results stay on
the device in a padded layout (ReducedContacts); `patches(e)` rebuilds the
reference's list[ContactPatch] for one env.

    register_sdf(grid) -> int          device SDF store handle (uploaded once)
    register_mesh(mesh) -> int         device mesh store handle
    collide(sdf_handles, mesh_handles, sdf_pose, mesh_pose, contact_distance, params)
        -> ReducedContacts
"""

from __future__ import annotations

import ctypes
import threading
import weakref
from collections import OrderedDict

import numpy as np

from . import _native
from .contacts.types import ContactPatch, ContactSet, ReductionParams
from .errors import NonFiniteStateError
from .geometry.mesh import TriMesh
from .sdf.grid import SignedDistanceGrid



class PlanCache:
    """Bounded, thread-safe LRU of plans keyed by (thread, assets, params).

    The per-pair drop-ins and collide() reuse one plan per configuration instead of
    allocating device buffers on every call. Keys carry the calling thread's id, so
    two threads never share a plan's buffers (a plan is re-entrant per stream, not
    across concurrent callers). At most `maxsize` plans are kept; when an SDF or mesh
    asset is finalised its plans are dropped first, so the deferred free of its device
    copy completes and its handle is reused."""

    _all: "weakref.WeakSet[PlanCache]" = weakref.WeakSet()

    def __init__(self, maxsize: int = 8):
        self.maxsize = maxsize
        self._d: OrderedDict = OrderedDict()
        self._assets: dict = {}
        self._lock = threading.Lock()
        PlanCache._all.add(self)

    def get(self, key, make, sdf_handles=(), mesh_handles=()):
        key = (threading.get_ident(),) + tuple(key)
        with self._lock:
            plan = self._d.get(key)
            if plan is not None:
                self._d.move_to_end(key)
                return plan
        plan = make()
        with self._lock:
            self._d[key] = plan
            self._assets[key] = (frozenset(int(h) for h in sdf_handles), frozenset(int(h) for h in mesh_handles))
            while len(self._d) > self.maxsize:
                old, _ = self._d.popitem(last=False)
                self._assets.pop(old, None)
        return plan

    def evict(self, sdf: int | None = None, mesh: int | None = None) -> None:
        with self._lock:
            for k in [k for k, (s, m) in self._assets.items() if (sdf is not None and sdf in s) or
                      (mesh is not None and mesh in m)]:
                self._d.pop(k, None)
                self._assets.pop(k, None)

    def clear(self) -> None:
        with self._lock:
            self._d.clear()
            self._assets.clear()

    def __len__(self) -> int:
        return len(self._d)


def evict_asset_plans(sdf: int | None = None, mesh: int | None = None) -> None:
    """Drop every cached plan that uses SDF handle `sdf` / mesh handle `mesh`."""
    for c in list(PlanCache._all):
        c.evict(sdf, mesh)


def _free_mesh(h: int) -> None:
    try:
        evict_asset_plans(mesh=h)
        _native.lib().cs_mesh_free(h)
    except Exception:
        pass


def register_sdf(grid: SignedDistanceGrid) -> int:
    """SDF asset registration: upload the grid once; every env naming it shares it."""
    return grid.device_handle()


def register_mesh(mesh: TriMesh) -> int:
    """Upload the mesh to the device mesh store once; freed with the TriMesh."""
    h = mesh._device_handle
    if h is None:
        out = ctypes.c_int32(-1)
        _native.call("cs_mesh_register", mesh.vertices.ctypes.data, len(mesh.vertices), mesh.triangles.ctypes.data,
                     len(mesh.triangles), ctypes.byref(out))
        h = mesh._device_handle = int(out.value)
        weakref.finalize(mesh, _free_mesh, h)
    return h


def pin_sdf_in_l2(grid: SignedDistanceGrid, hit_ratio: float = 1.0, stream=None) -> None:
    """Persist the grid in L2 for launches on `stream` (cudaAccessPolicyWindow)."""
    _native.call("cs_sdf_l2_persist", grid.device_handle(), _native.stream_handle(stream), float(hit_ratio))


def _destroy_plan(ptr: int) -> None:
    try:
        _native.lib().cs_plan_destroy(ptr)
    except Exception:
        pass


class _PlanHandle:
    """Owns a cs_plan's device memory. The plan's tensor views keep this handle (not
    the Plan) alive, so dropping a Plan frees its buffers at once unless a view of
    them is still held (no Plan <-> view reference cycle waiting for the GC)."""

    def __init__(self, ptr: int):
        self.ptr = ptr
        weakref.finalize(self, _destroy_plan, ptr)


class Plan:
    """Owns the device buffers of one env configuration (cs_plan_create)."""

    def __init__(self, sdf_handles, mesh_handles, params: ReductionParams | None, stages: int = _native.CS_STAGE_ALL,
                 capacity=None):
        lib = _native.lib()
        ptr = ctypes.c_void_p()
        self.params = params or ReductionParams()
        cparams = self.params.to_c()
        if stages == _native.CS_STAGE_REDUCE:
            cap = np.ascontiguousarray(capacity, dtype=np.int64)
            self.n_envs = len(cap)
            _native.check(lib.cs_plan_create_reduce(self.n_envs, cap.ctypes.data, ctypes.byref(cparams), ctypes.byref(ptr)))
        else:
            s = np.ascontiguousarray(sdf_handles, dtype=np.int32)
            m = np.ascontiguousarray(mesh_handles, dtype=np.int32)
            if s.shape != m.shape or s.ndim != 1:
                raise ValueError("sdf_handles and mesh_handles must be 1-D of equal length")
            self.n_envs = len(s)
            _native.check(lib.cs_plan_create(self.n_envs, s.ctypes.data, m.ctypes.data, ctypes.byref(cparams),
                                             stages, ctypes.byref(ptr)))
        self.ptr = int(ptr.value)
        self.stages = stages
        self._handle = _PlanHandle(self.ptr)
        o = _native.OutputsC()
        _native.check(lib.cs_plan_outputs(self.ptr, ctypes.byref(o)))
        self.c = o
        E, N, K, cap = o.n_envs, o.max_patches, o.per_patch_cap, o.total_capacity
        v = lambda name, shape, dt: _native.device_view(getattr(o, name), shape, dt, self._handle)  # noqa: E731
        self.cand_base = v("cand_base", (E,), "i8")
        self.env_status = v("env_status", (E,), "i4")
        self.n_cand = v("n_cand", (E,), "i4")
        self.cand_point = v("cand_point", (cap, 3), "f8")
        self.cand_normal = v("cand_normal", (cap, 3), "f8")
        self.cand_depth = v("cand_depth", (cap,), "f8")
        self.cand_face = v("cand_face", (cap,), "i4")
        if o.face_work:
            self.face_work = v("face_work", (4,), "i4")  # diagnostics of the last step's descent
        if stages & _native.CS_STAGE_REDUCE:
            self.n_patch = v("n_patch", (E,), "i4")
            self.n_kept = v("n_kept", (E,), "i4")
            self.stats = v("stats", (E, 4), "f4")
            self.patch_normal = v("patch_normal", (E, N, 3), "f8")
            self.patch_nkept = v("patch_nkept", (E, N), "i4")
            self.kept_cand = v("kept_cand", (E, N, K), "i4")
            self.kept_point = v("kept_point", (E, N, K, 3), "f8")
            self.kept_normal = v("kept_normal", (E, N, K, 3), "f8")
            self.kept_depth = v("kept_depth", (E, N, K), "f8")
            self.kept_face = v("kept_face", (E, N, K), "i4")
            self.w_sum = v("w_sum", (E, N), "f8")
            self.wp_sum = v("wp_sum", (E, N, 3), "f8")
            self.wn_sum = v("wn_sum", (E, N, 3), "f8")
            self.wt_sum = v("wt_sum", (E, N, 3), "f8")
            self.area = v("area", (E, N), "f8")
            self.max_depth = v("max_depth", (E, N), "f8")
            self.member_offsets = v("member_offsets", (E, N + 1), "i4")
            self.members = v("members", (cap,), "i4")

    def collide(self, sdf_pose, mesh_pose, contact_distance, pose_format: int = _native.CS_POSE7, stream=None):
        """One step on device tensors (float64, contiguous). Stream-ordered, no sync."""
        for t in (sdf_pose, mesh_pose, contact_distance):
            if not (t.is_cuda and t.dtype.is_floating_point and t.element_size() == 8 and t.is_contiguous()):
                raise ValueError("poses and contact_distance must be contiguous float64 CUDA tensors")
        self._check_pose_shapes(sdf_pose, mesh_pose, contact_distance, pose_format)
        _native.hand_to_stream(stream, sdf_pose, mesh_pose, contact_distance)
        _native.call("cs_collide", self.ptr, sdf_pose.data_ptr(), mesh_pose.data_ptr(), pose_format,
                     contact_distance.data_ptr(), _native.stream_handle(stream))

    def _check_pose_shapes(self, sdf_pose, mesh_pose, contact_distance, pose_format) -> None:
        """The C side reads E poses of 7 (or 12) doubles and E contact distances."""
        if not (self.stages & _native.CS_STAGE_GENERATE):
            raise ValueError("plan has no generate stage")
        width = 7 if pose_format == _native.CS_POSE7 else 12 if pose_format == _native.CS_POSE12 else None
        if width is None:
            raise ValueError(f"unknown pose format {pose_format}")
        E = self.n_envs
        for name, t in (("sdf_pose", sdf_pose), ("mesh_pose", mesh_pose)):
            if tuple(t.shape) not in ((E, width), (E * width,)):
                raise ValueError(f"{name} must have shape ({E}, {width}), got {tuple(t.shape)}")
        n_cd = contact_distance.numel() if hasattr(contact_distance, "numel") else contact_distance.size
        if n_cd != E:
            raise ValueError(f"contact_distance must hold {E} values, got {n_cd}")

    def collide_host(self, sdf_pose: np.ndarray, mesh_pose: np.ndarray, contact_distance: np.ndarray,
                     pose_format: int = _native.CS_POSE7, stats_out: np.ndarray | None = None, stream=None):
        """End-to-end call with host buffers: H2D poses, collide, D2H stats [E,4], synchronise."""
        st = stats_out if stats_out is not None else np.empty((self.n_envs, 4), np.float32)
        for a in (sdf_pose, mesh_pose, contact_distance, st):
            if not (isinstance(a, np.ndarray) and a.flags.c_contiguous):
                raise ValueError("collide_host takes C-contiguous numpy arrays")
        if sdf_pose.dtype != np.float64 or mesh_pose.dtype != np.float64 or contact_distance.dtype != np.float64 \
                or st.dtype != np.float32 or st.size != 4 * self.n_envs:
            raise ValueError("collide_host: float64 poses / contact_distance and a float32 (E, 4) stats buffer")
        self._check_pose_shapes(sdf_pose, mesh_pose, contact_distance, pose_format)
        _native.call("cs_collide_host", self.ptr, sdf_pose.ctypes.data, mesh_pose.ctypes.data, pose_format,
                     contact_distance.ctypes.data, st.ctypes.data, _native.stream_handle(stream))
        return st

    def reduce(self, stream=None):
        _native.call("cs_reduce", self.ptr, _native.stream_handle(stream))

    PHASES = ("env_xf", "face_prep", "face_pgd", "compact", "reduce", "finalize", "total")

    def enable_timing(self, slots: int) -> None:
        """Record CUDA events around each phase of the next `slots` collide calls (0 disables)."""
        _native.call("cs_plan_timing", self.ptr, int(slots))

    @property
    def device_bytes(self) -> int:
        """Device memory the plan holds (cs_plan_device_bytes): about 4.3 MB per env
        of the M16 nut (17 304 faces), for sizing env counts per GPU."""
        n = ctypes.c_int64(0)
        _native.call("cs_plan_device_bytes", self.ptr, ctypes.byref(n))
        return int(n.value)

    def read_timing(self, max_steps: int) -> np.ndarray:
        """(steps, 7) ms per phase (Plan.PHASES), oldest first."""
        out = np.zeros((max_steps, len(self.PHASES)), np.float32)
        n = ctypes.c_int32(0)
        _native.call("cs_plan_timing_read", self.ptr, out.ctypes.data, int(max_steps), ctypes.byref(n))
        return out[: n.value]

    def solve(self, state, mu, restitution, slop, params=None, wrench=None, stream=None):
        """Contact solve of one substep on the last collide's reduced contacts
        (cs_plan_solve): per env the two-body system of Scene._substep
        (dynamics/scene.py:130-145) — rows in (patch, kept) order, pos_iterations
        sweeps with friction toward the bias targets, then vel_iterations toward the
        restitution targets. state: dynamics.BatchedSolverState (vel and impulse
        updated in place); mu, restitution, slop: (E,) float64 CUDA tensors.
        Returns the body wrenches (E,2,6)."""
        import torch

        from .dynamics.solver import SolverParams

        if not self.stages & _native.CS_STAGE_REDUCE:
            raise ValueError("plan has no reduce stage")
        params = params or SolverParams()
        for t in (state.ref, state.w_mat, state.vel, state.impulse, mu, restitution, slop):
            if not (t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
                raise ValueError("solver state and per-env parameters must be contiguous float64 CUDA tensors")
        E = self.n_envs
        want = {"ref": (E, 2, 3), "w_mat": (E, 2, 6, 6), "vel": (E, 2, 6), "impulse": (E, 2, 6)}
        for name, shape in want.items():
            got = tuple(getattr(state, name).shape)
            if got != shape:
                raise ValueError(f"state.{name} must have shape {shape} (one two-body system per env), got {got}")
        for name, t in (("mu", mu), ("restitution", restitution), ("slop", slop)):
            if t.numel() != E:
                raise ValueError(f"{name} must hold {E} values, got {t.numel()}")
        if wrench is not None and not (wrench.is_cuda and wrench.dtype == torch.float64 and wrench.is_contiguous()
                                       and tuple(wrench.shape) == (E, 2, 6)):
            raise ValueError(f"wrench must be a contiguous float64 CUDA tensor of shape ({E}, 2, 6)")
        _native.hand_to_stream(stream, state.ref, state.w_mat, state.vel, state.impulse, mu, restitution, slop, wrench)
        if wrench is None:
            wrench = torch.empty((self.n_envs, 2, 6), dtype=torch.float64, device="cuda")
        cp = params.to_c()
        _native.call("cs_plan_solve", self.ptr, state.ref.data_ptr(), state.w_mat.data_ptr(), state.vel.data_ptr(),
                     state.impulse.data_ptr(), mu.data_ptr(), restitution.data_ptr(), slop.data_ptr(),
                     ctypes.byref(cp), wrench.data_ptr(), _native.stream_handle(stream))
        return wrench

    def solver_rows(self, e: int | None = None) -> dict:
        """The solver rows of the last solve (cs_plan_solver_rows). With e: env e's
        rows in sweep order as host arrays; without: the raw device views
        (interleaved layout, include/contactsim_b200.h cs_solver_rows)."""
        r = _native.SolverRowsC()
        _native.call("cs_plan_solver_rows", self.ptr, ctypes.byref(r))
        R = r.planes
        out = {"stride": int(r.stride), "planes": int(R)}
        vec = ("point", "normal", "ra", "rb", "tan1", "tan2")
        for k in ("body_a", "body_b"):
            out[k] = _native.device_view(getattr(r, k), (R,), "i8", self._handle)
        for k in vec:
            out[k] = _native.device_view(getattr(r, k), (3, R), "f8", self._handle)
        for k in ("depth", "mu", "restitution", "slop", "kn", "kt1", "kt2", "bias_target", "restitution_target",
                  "lam_n", "lam_vel", "lam_t1", "lam_t2"):
            out[k] = _native.device_view(getattr(r, k), (R,), "f8", self._handle)
        if e is None:
            return out
        m = int(self.n_kept[e].item())
        idx = ((e // 32 * r.stride + np.arange(m)) * 32 + e % 32).astype(np.int64)
        it = __import__("torch").from_numpy(idx).cuda()
        return {k: (v[:, it].T if k in vec else v[it]).cpu().numpy() for k, v in out.items()
                if k not in ("stride", "planes")}

    def count_samples(self, sdf_pose, mesh_pose, contact_distance, pose_format: int = _native.CS_POSE7):
        """Exact trilinear SDF samples of one collide step (counting builds):
        (k_face_prep samples, k_face_pgd samples)."""
        _native.call("cs_plan_count_samples", self.ptr, 1, None)
        self.collide(sdf_pose, mesh_pose, contact_distance, pose_format)
        c = (ctypes.c_uint64 * 2)()
        _native.call("cs_plan_count_samples", self.ptr, 0, c)
        return int(c[0]), int(c[1])


class ReducedContacts:
    """Device-resident result of one collide step (views into the plan's buffers;
    valid until the plan runs again)."""

    def __init__(self, plan: Plan, body_ids=None, stream=None):
        self.plan = plan
        self.body_ids = body_ids
        self.stream = stream  # the stream the step ran on (check() waits for it)

    def __getattr__(self, name):
        return getattr(self.plan, name)

    @property
    def n_envs(self) -> int:
        return self.plan.n_envs

    def check(self) -> None:
        """Raise the reference's errors for envs flagged on device (waits for the step's stream)."""
        _native.sync_stream(self.stream)
        st = self.plan.env_status.cpu().numpy()
        if (st == 1).any():
            raise NonFiniteStateError(f"non-finite pose in contact generation (envs {np.nonzero(st == 1)[0][:8].tolist()})")
        if (st == 2).any():
            raise ValueError("contact_distance must be non-negative")

    def contact_set(self, e: int, body_a: int = -1, body_b: int = -1) -> ContactSet:
        p = self.plan
        base_n = _native.fetch(p.cand_base[e: e + 1], p.n_cand[e: e + 1])
        base, n = int(base_n[0][0]), int(base_n[1][0])
        sl = slice(base, base + n)
        pt, nr, dp, fc = _native.fetch(p.cand_point[sl], p.cand_normal[sl], p.cand_depth[sl], p.cand_face[sl])
        return ContactSet(pt, nr, dp, fc.astype(np.int64), body_a, body_b)

    def patches(self, e: int, face_indices: np.ndarray | None = None) -> list[ContactPatch]:
        """list[ContactPatch] of env e in slot order (reduction.py:75)."""
        p = self.plan
        # two synchronisations: the env's counts and offsets, then every field at once
        np_, base, moff = _native.fetch(p.n_patch[e: e + 1], p.cand_base[e: e + 1], p.member_offsets[e])
        P, base = int(np_[0]), int(base[0])
        if P == 0:
            return []
        moff = moff[: P + 1].astype(np.int64)
        keys = ("patch_normal", "patch_nkept", "kept_cand", "kept_point", "kept_normal", "kept_depth", "kept_face",
                "w_sum", "wp_sum", "wn_sum", "wt_sum", "area", "max_depth")
        got = _native.fetch(p.members[base: base + int(moff[-1])], *(getattr(p, k)[e, :P] for k in keys))
        members = got[0].astype(np.int64)
        host = dict(zip(keys, got[1:]))
        out = []
        for q in range(P):
            k = int(host["patch_nkept"][q])
            if face_indices is not None:
                faces = np.asarray(face_indices, dtype=np.int64)[host["kept_cand"][q, :k].astype(np.int64)]
            else:
                faces = host["kept_face"][q, :k].astype(np.int64)
            out.append(ContactPatch(
                representative_normal=host["patch_normal"][q].copy(),
                points=host["kept_point"][q, :k].copy(),
                normals=host["kept_normal"][q, :k].copy(),
                depths=host["kept_depth"][q, :k].copy(),
                face_indices=faces,
                member_indices=members[moff[q]: moff[q + 1]].copy(),
                weight_sum=float(host["w_sum"][q]),
                weighted_point_sum=host["wp_sum"][q].copy(),
                weighted_normal_sum=host["wn_sum"][q].copy(),
                weighted_torque_sum=host["wt_sum"][q].copy(),
                area_metric=float(host["area"][q]),
                max_depth=float(host["max_depth"][q]),
            ))
        return out


_plan_cache = PlanCache(maxsize=4)


def clear_plan_cache() -> None:
    """Drop every cached plan: collide()'s and the per-pair drop-ins' (their device
    memory is freed once no result view of them is held)."""
    for c in list(PlanCache._all):
        c.clear()


def get_plan(sdf_handles, mesh_handles, params: ReductionParams | None) -> Plan:
    params = params or ReductionParams()
    s = tuple(np.asarray(sdf_handles).tolist())
    m = tuple(np.asarray(mesh_handles).tolist())
    key = (s, m, params.max_patches, params.per_patch_cap, params.normal_cone_cos, params.min_depth,
           params.batch_size)
    return _plan_cache.get(key, lambda: Plan(sdf_handles, mesh_handles, params), set(s), set(m))


def collide(sdf_handles, mesh_handles, sdf_pose, mesh_pose, contact_distance, params: ReductionParams | None = None,
            check: bool = True, stream=None) -> ReducedContacts:
    """Generate + reduce contacts for E envs.

    sdf_handles / mesh_handles: (E,) ints from register_sdf / register_mesh.
    sdf_pose / mesh_pose: (E, 7) float64 (px, py, pz, qw, qx, qy, qz), host or CUDA.
    contact_distance: (E,) or scalar float64.
    params: ReductionParams shared by every env. As in Scene._collect_contacts
    (scene.py:215-225), min_depth=None means "-contact_distance per env"; pass
    params with min_depth set to override.
    """
    import torch

    E = len(sdf_handles)
    plan = get_plan(sdf_handles, mesh_handles, params if params is not None else ReductionParams())
    dev = lambda x: torch.as_tensor(np.asarray(x, dtype=np.float64) if not torch.is_tensor(x) else x,  # noqa: E731
                                    dtype=torch.float64).cuda().contiguous()
    sp, mp = dev(sdf_pose).reshape(E, 7), dev(mesh_pose).reshape(E, 7)
    cd = dev(contact_distance).reshape(-1)
    if cd.numel() == 1:
        cd = cd.expand(E).contiguous()
    plan.collide(sp, mp, cd, _native.CS_POSE7, stream)  # hands the staged inputs to `stream`
    res = ReducedContacts(plan, stream=stream)
    if check:
        res.check()
    return res
