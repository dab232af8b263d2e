"""Per-phase CTA cycle split of k_reduce (developer tool; needs a -DRED_PROF build):
    CS_LIB_PATH=_variants/redprof/libcontactsim_b200.so python scripts/red_prof.py
"""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import paper_2205_03532_b200 as P
    from paper_2205_03532_b200 import _native
    from paper_2205_03532_b200.scenes import m16_workload

    n = 1024
    w = m16_workload(n)
    plan = P.Plan([P.register_sdf(w["grid"])] * n, [P.register_mesh(w["nut"])] * n, P.ReductionParams())
    sp, mp, cd = (torch.from_numpy(np.ascontiguousarray(w[k])).cuda() for k in ("sdf_pose", "mesh_pose", "cd"))
    lib = _native.lib()
    buf = (ctypes.c_ulonglong * 8)()
    plan.collide(sp, mp, cd)
    torch.cuda.synchronize()
    lib.cs_debug_red_prof(buf)
    a = np.array(buf[:], dtype=np.float64)
    reps = 10
    for _ in range(reps):
        plan.collide(sp, mp, cd)
    torch.cuda.synchronize()
    lib.cs_debug_red_prof(buf)
    b = (np.array(buf[:], dtype=np.float64) - a) / reps / n
    names = ["setup (cull check)", "stage + assign", "after batches", "seed loops (per batch)", "outputs + CSR count",
             "CSR scatter (warp 0)"]
    tot = b[:6].sum()
    for i, nm in enumerate(names):
        print(f"{nm:24s} {b[i] / 1e3:10.1f} kcycles per env  {100 * b[i] / tot:5.1f}%")


if __name__ == "__main__":
    main()
