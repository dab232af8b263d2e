"""How large is the box of grid cells a k_face_prep chunk samples (developer tool; needs a
-DBOX_STATS build): could the chunk's samples read their corners from shared memory?
    CS_LIB_PATH=_variants/box/libcontactsim_b200.so python scripts/box_stats.py"""
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
    lib.cs_debug_box_stat(buf)
    a = np.array(buf[:], dtype=np.float64)
    plan.collide(sp, mp, cd)
    torch.cuda.synchronize()
    lib.cs_debug_box_stat(buf)
    b = np.array(buf[:], dtype=np.float64) - a
    ch = b[0]
    print(f"chunks with samples {ch:.0f}: mean box {b[1] / ch:.0f} cells (4 B each) for {b[5] / ch:.0f} samples; "
          f"boxes <= 4096 cells {100 * b[2] / ch:.1f}%, <= 8192 {100 * b[3] / ch:.1f}%, <= 16384 {100 * b[4] / ch:.1f}%")


if __name__ == "__main__":
    main()
