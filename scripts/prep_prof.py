"""Per-phase CTA cycle split of k_face_prep (developer tool; needs a -DPREP_PROF build):
    CS_LIB_PATH=_variants/prof/libcontactsim_b200.so python scripts/prep_prof.py
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
    buf = (ctypes.c_ulonglong * 16)()
    plan.collide(sp, mp, cd)
    torch.cuda.synchronize()
    lib.cs_debug_prep_prof(buf)
    a = np.array(buf[:], dtype=np.float64)
    reps = 10
    for _ in range(reps):
        plan.collide(sp, mp, cd)
    torch.cuda.synchronize()
    lib.cs_debug_prep_prof(buf)
    b = (np.array(buf[:], dtype=np.float64) - a) / reps
    names = ["load env", "transform", "bound+queue faces", "queue verts", "samples", "prune+scan+write"]
    tot = b[:6].sum()
    for i, nm in enumerate(names):
        print(f"{nm:20s} {b[i] / 1e6:10.2f} Mcycles (sum over CTAs)  {100 * b[i] / tot:5.1f}%")
    if b[8]:  # -DPREP_STATS: face outcomes (the bound is evaluated but not applied)
        for i, nm in zip(range(8, 14), ["faces", "aabb near", "bound culls", "prune culls", "both cull", "neither"]):
            print(f"{nm:12s} {b[i]:12.0f}  {100 * b[i] / b[8]:5.1f}%")
        bs = (ctypes.c_ulonglong * 4)()
        lib.cs_debug_bound_stat.restype = ctypes.c_int
        lib.cs_debug_bound_stat(bs)
        x = np.array(bs[:], dtype=np.float64) / (reps + 1)
        print(f"brick passes {x[0]:.0f}, settled by bricks {x[1]:.0f}; cell passes {x[2]:.0f}; "
              f"boxes too large for the cell pass {x[3]:.0f}")


if __name__ == "__main__":
    main()
