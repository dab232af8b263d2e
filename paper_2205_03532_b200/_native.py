"""ctypes binding of libcontactsim_b200.so (include/contactsim_b200.h).

This is the only way the package reaches the GPU. There is no CPU fallback:
if the library or a CUDA device is missing, `lib()` raises.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import threading

from .errors import MeshValidationError, NonFiniteStateError

_HERE = os.path.dirname(os.path.abspath(__file__))
# CS_LIB_PATH: developer override (build variants for A/B timing); the default is the in-tree build
LIB_PATH = os.environ.get("CS_LIB_PATH") or os.path.join(_HERE, "_lib", "libcontactsim_b200.so")
CSRC = os.path.join(_HERE, "csrc")

CS_OK, CS_ERR_VALUE, CS_ERR_NONFINITE, CS_ERR_MESH, CS_ERR_HANDLE, CS_ERR_CUDA, CS_ERR_OOM, CS_ERR_IO = range(8)
CS_POSE7, CS_POSE12 = 0, 1
CS_STAGE_GENERATE, CS_STAGE_REDUCE, CS_STAGE_ALL = 1, 2, 3

_i32, _i64, _f32, _f64, _vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_float, ctypes.c_double, ctypes.c_void_p


class ReductionParamsC(ctypes.Structure):
    _fields_ = [("max_patches", _i32), ("per_patch_cap", _i32), ("batch_size", _i32), ("has_min_depth", _i32),
                ("normal_cone_cos", _f64), ("min_depth", _f64)]


class OutputsC(ctypes.Structure):
    _fields_ = [
        ("n_envs", _i64), ("max_patches", _i32), ("per_patch_cap", _i32), ("total_capacity", _i64),
        ("cand_base", _vp), ("env_status", _vp), ("n_cand", _vp), ("n_patch", _vp), ("n_kept", _vp), ("stats", _vp),
        ("cand_point", _vp), ("cand_normal", _vp), ("cand_depth", _vp), ("cand_face", _vp),
        ("patch_normal", _vp), ("patch_nkept", _vp), ("kept_cand", _vp), ("kept_point", _vp), ("kept_normal", _vp),
        ("kept_depth", _vp), ("kept_face", _vp), ("w_sum", _vp), ("wp_sum", _vp), ("wn_sum", _vp), ("wt_sum", _vp),
        ("area", _vp), ("max_depth", _vp), ("member_offsets", _vp), ("members", _vp), ("face_work", _vp),
    ]


class SdfFileInfoC(ctypes.Structure):
    _fields_ = [("dims", _i32 * 3), ("origin", _f64 * 3), ("voxel", _f64), ("aabb_lo", _f64 * 3), ("aabb_hi", _f64 * 3)]


class SolverParamsC(ctypes.Structure):
    _fields_ = [("h", _f64), ("bias_factor", _f64), ("pos_iterations", _i32), ("vel_iterations", _i32)]


class SolverRowsC(ctypes.Structure):
    _fields_ = [("stride", _i64), ("planes", _i64)] + [(k, _vp) for k in (
        "body_a", "body_b", "point", "normal", "depth", "mu", "restitution", "slop", "ra", "rb", "tan1", "tan2",
        "kn", "kt1", "kt2", "bias_target", "restitution_target", "lam_n", "lam_vel", "lam_t1", "lam_t2")]


_SIGS = {
    "cs_last_error": ([], ctypes.c_char_p),
    "cs_abi_version": ([], ctypes.c_int),
    "cs_device_info": ([ctypes.POINTER(_i32), ctypes.POINTER(_i64), ctypes.POINTER(_i64)], ctypes.c_int),
    "cs_bench_gather": ([_i32, _i64, _i32, ctypes.POINTER(_f64)], ctypes.c_int),
    "cs_sdf_register": ([_vp, ctypes.c_int, _i32, _i32, _i32, _vp, _f64, _vp, _vp, ctypes.POINTER(_i32)], ctypes.c_int),
    "cs_sdf_register_file": ([ctypes.c_char_p, ctypes.POINTER(_i32), ctypes.POINTER(SdfFileInfoC)], ctypes.c_int),
    "cs_sdf_free": ([_i32], ctypes.c_int),
    "cs_sdf_values": ([_i32, ctypes.POINTER(_vp)], ctypes.c_int),
    "cs_sdf_l2_persist": ([_i32, _vp, _f32], ctypes.c_int),
    "cs_mesh_register": ([_vp, _i64, _vp, _i64, ctypes.POINTER(_i32)], ctypes.c_int),
    "cs_mesh_free": ([_i32], ctypes.c_int),
    "cs_face_contacts": ([_vp, _i64, _i64, _i64, _f64, _f64, _f64, _f64, _vp, _i64, _f64, _i32, _f64, _vp, _vp, _vp,
                          _vp, _vp], ctypes.c_int),
    "cs_sdf_sample": ([_vp, _i64, _i64, _i64, _f64, _f64, _f64, _f64, _vp, _i64, _vp, _vp], ctypes.c_int),
    "cs_sdf_gradient": ([_vp, _i64, _i64, _i64, _f64, _f64, _f64, _f64, _vp, _i64, _vp, _vp], ctypes.c_int),
    "cs_plan_create": ([_i64, _vp, _vp, ctypes.POINTER(ReductionParamsC), _i32, ctypes.POINTER(_vp)], ctypes.c_int),
    "cs_plan_create_reduce": ([_i64, _vp, ctypes.POINTER(ReductionParamsC), ctypes.POINTER(_vp)], ctypes.c_int),
    "cs_plan_destroy": ([_vp], ctypes.c_int),
    "cs_plan_device_bytes": ([_vp, ctypes.POINTER(ctypes.c_int64)], ctypes.c_int),
    "cs_plan_outputs": ([_vp, ctypes.POINTER(OutputsC)], ctypes.c_int),
    "cs_collide": ([_vp, _vp, _vp, _i32, _vp, _vp], ctypes.c_int),
    "cs_reduce": ([_vp, _vp], ctypes.c_int),
    "cs_plan_count_samples": ([_vp, _i32, ctypes.POINTER(ctypes.c_uint64)], ctypes.c_int),
    "cs_plan_timing": ([_vp, _i32], ctypes.c_int),
    "cs_plan_timing_read": ([_vp, _vp, _i32, ctypes.POINTER(_i32)], ctypes.c_int),
    "cs_collide_host": ([_vp, _vp, _vp, _i32, _vp, _vp, _vp], ctypes.c_int),
    "cs_sdf_generate": ([_vp, _i64, _vp, _i64, _i32, _i32, _i32, _vp, _f64, _vp], ctypes.c_int),
    "cs_constraints_build": ([_i64, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _f64, _f64]
                             + [_vp] * 9 + [_vp], ctypes.c_int),
    "cs_gauss_seidel_sweeps": ([_i64, _i32, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                _vp, _vp, _vp, _vp, _vp, _vp, _i32, _vp], ctypes.c_int),
    "cs_body_wrenches": ([_i64, _i32, _vp] + [_vp] * 11 + [_f64, _vp, _vp], ctypes.c_int),
    "cs_plan_solve": ([_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, ctypes.POINTER(SolverParamsC), _vp, _vp], ctypes.c_int),
    "cs_plan_solver_rows": ([_vp, ctypes.POINTER(SolverRowsC)], ctypes.c_int),
    "cs_multipair_solve": ([_vp, _i64, _i32, _vp, _vp, _vp, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                            ctypes.POINTER(SolverParamsC), _vp, _vp], ctypes.c_int),
    "cs_plan_multipair_rows": ([_vp, ctypes.POINTER(SolverRowsC), ctypes.POINTER(_vp)], ctypes.c_int),
    "cs_world_aabb": ([_i64, _vp, _vp, _vp, _vp, _vp, _vp], ctypes.c_int),
    "cs_broadphase": ([_i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp], ctypes.c_int),
    "cs_pair_slots_active": ([_i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp], ctypes.c_int),
    "cs_collide_active": ([_vp, _vp, _vp, _i32, _vp, _vp, _vp], ctypes.c_int),
}

EXPORTED = tuple(_SIGS)

_lib = None
_lock = threading.Lock()


def build(verbose: bool = False) -> str:
    """Compile the sm_100a library in-tree (nvcc cross-compiles without a GPU)."""
    out = subprocess.run(["make", "-C", CSRC, "-j8"], capture_output=not verbose, text=True)
    if out.returncode != 0:
        raise RuntimeError(f"building libcontactsim_b200.so failed:\n{out.stdout}\n{out.stderr}")
    return LIB_PATH


def load_symbols_only() -> ctypes.CDLL:
    """dlopen the library and bind every ABI symbol without touching the GPU."""
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing; run __graft_entry__.build() (no CPU fallback exists)")
    so = ctypes.CDLL(LIB_PATH)
    for name, (args, res) in _SIGS.items():
        fn = getattr(so, name)
        fn.argtypes = args
        fn.restype = res
    return so


def lib() -> ctypes.CDLL:
    """The loaded library, bound to a CUDA device. Raises if either is missing."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            import torch

            if not torch.cuda.is_available():
                raise RuntimeError("paper_2205_03532_b200 needs a CUDA device (sm_100a); there is no CPU path")
            torch.cuda.init()
            so = load_symbols_only()
            if so.cs_abi_version() != 1:
                raise ImportError("libcontactsim_b200.so ABI version mismatch")
            _lib = so
    return _lib


def check(status: int) -> None:
    """Map a cs_status to the reference's exception classes (errors.py)."""
    if status == CS_OK:
        return
    msg = _lib.cs_last_error().decode() if _lib is not None else f"status {status}"
    if status == CS_ERR_VALUE:
        raise ValueError(msg)
    if status == CS_ERR_NONFINITE:
        raise NonFiniteStateError(msg)
    if status == CS_ERR_MESH:
        raise MeshValidationError(msg)
    if status == CS_ERR_OOM:
        raise MemoryError(msg)
    if status == CS_ERR_IO:
        raise OSError(msg)
    raise RuntimeError(msg)


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args))


def stream_handle(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def hand_to_stream(stream, *tensors) -> None:
    """Make tensors staged on the current stream safe to read on `stream`: `stream`
    waits for the current stream's work so far, and the caching allocator is told the
    tensors are in use there (record_stream), so their memory is not reused until
    `stream`'s kernels are done. No-op when `stream` is None or the current stream."""
    import torch

    if stream is None:
        return
    cur = torch.cuda.current_stream()
    if int(stream.cuda_stream) == int(cur.cuda_stream):
        return
    stream.wait_stream(cur)
    for t in tensors:
        if t is not None:
            t.record_stream(stream)


def fetch(*tensors) -> list:
    """Device tensors to numpy with ONE synchronisation: every copy is queued
    asynchronously (into pinned host memory) on the current stream, then the stream is
    waited for once (instead of a blocking .cpu() per tensor)."""
    import torch

    host = [t.to("cpu", non_blocking=True) for t in tensors]
    torch.cuda.current_stream().synchronize()
    return [h.numpy() for h in host]


def sync_stream(stream=None) -> None:
    """Block until `stream` (default: the current stream) has finished."""
    import torch

    (stream if stream is not None else torch.cuda.current_stream()).synchronize()


class DevArray:
    """Zero-copy __cuda_array_interface__ view of plan-owned device memory."""

    _TYPESTR = {"f8": "<f8", "f4": "<f4", "i4": "<i4", "i8": "<i8", "u1": "|u1"}

    def __init__(self, ptr: int, shape, dtype: str, owner):
        self.__cuda_array_interface__ = {
            "shape": tuple(int(s) for s in shape),
            "typestr": self._TYPESTR[dtype],
            "data": (int(ptr), False),
            "version": 3,
            "strides": None,
            "stream": None,
        }
        self._owner = owner


def device_view(ptr: int, shape, dtype: str, owner):
    import torch

    t = torch.as_tensor(DevArray(ptr, shape, dtype, owner), device="cuda")
    t._cs_owner = owner  # keep the plan alive while the view exists
    return t
