"""Drop-in for the reference's sweep kernel (contactsim/dynamics/_kernels.py:52-115).

`gauss_seidel_sweeps` keeps the reference's argument list and in-place
semantics: vel, imp, lam_n, lam_t1, lam_t2 are updated. The sweep runs on the GPU
(cs_gauss_seidel_sweeps, csrc/cs_solver.cu) and is bit-identical to the numba
kernel. Arguments may be numpy arrays (copied to the device and back) or
contiguous float64 / int64 CUDA tensors (updated in place on the device).
"""

from __future__ import annotations

import numpy as np

from .. import _native

_IN_OUT = ("vel", "imp", "lam_n", "lam_t1", "lam_t2")


def _dev(x, dtype):
    import torch

    if isinstance(x, torch.Tensor):
        if not x.is_cuda or x.dtype != dtype or not x.is_contiguous():
            raise ValueError("CUDA tensors passed to the solver must be contiguous and of the reference's dtype")
        return x
    return torch.from_numpy(np.array(x, dtype=np.float64 if dtype.is_floating_point else np.int64, order="C")).cuda()


def gauss_seidel_sweeps(iters, w_mat, vel, imp, body_a, body_b, ra, rb, nrm, tan1, tan2, kn, kt1, kt2, target_vn, mu,
                        lam_n, lam_t1, lam_t2, with_friction):
    import torch

    f64, i64 = torch.float64, torch.int64
    m = len(kn)
    args = dict(w_mat=w_mat, vel=vel, imp=imp, ra=ra, rb=rb, nrm=nrm, tan1=tan1, tan2=tan2, kn=kn, kt1=kt1, kt2=kt2,
                target_vn=target_vn, mu=np.broadcast_to(np.asarray(mu, np.float64), (m,)) if not
                isinstance(mu, torch.Tensor) else mu, lam_n=lam_n, lam_t1=lam_t1, lam_t2=lam_t2)
    d = {k: _dev(v, f64) for k, v in args.items()}
    ba, bb = _dev(body_a, i64), _dev(body_b, i64)
    nb = int(d["vel"].shape[0])
    if m == 0 or iters <= 0:
        return
    from .solver import check_solver_bodies

    check_solver_bodies(nb)
    off = torch.tensor([0, m], dtype=i64, device="cuda")
    p = lambda k: d[k].data_ptr()  # noqa: E731
    _native.call("cs_gauss_seidel_sweeps", 1, nb, off.data_ptr(), int(iters), p("w_mat"), p("vel"), p("imp"),
                 ba.data_ptr(), bb.data_ptr(), p("ra"), p("rb"), p("nrm"), p("tan1"), p("tan2"), p("kn"), p("kt1"),
                 p("kt2"), p("target_vn"), p("mu"), p("lam_n"), p("lam_t1"), p("lam_t2"), 1 if with_friction else 0,
                 _native.stream_handle())
    for k in _IN_OUT:  # numpy in/out arguments get the device results
        if isinstance(args[k], np.ndarray):
            args[k][...] = d[k].cpu().numpy().reshape(args[k].shape)
