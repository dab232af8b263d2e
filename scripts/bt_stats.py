"""Backtracking statistics of the descent (developer tool; needs a -DBT_STATS build):
    CS_LIB_PATH=_variants/bt/libcontactsim_b200.so python scripts/bt_stats.py
Per backtrack call (k_pgd_first's iteration 0 and k_pgd_rest's later ones): the try
that was accepted (0..3) or none, and how many projections were known (same point)
versus sampled."""
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
    lib.cs_debug_bt_stat(buf)
    a = np.array(buf[:], dtype=np.float64)
    plan.collide(sp, mp, cd)
    torch.cuda.synchronize()
    lib.cs_debug_bt_stat(buf)
    b = np.array(buf[:], dtype=np.float64) - a
    calls = b[:5].sum()
    print(f"backtrack calls {calls:.0f}: accepted at try 0..3 " +
          " ".join(f"{100 * b[i] / calls:.1f}%" for i in range(4)) + f", no move {100 * b[4] / calls:.1f}%")
    print(f"projections {b[5] + b[6]:.0f}: known {100 * b[5] / (b[5] + b[6]):.1f}%, sampled {100 * b[6] / (b[5] + b[6]):.1f}%")
    print(f"k_pgd_first: no move from a centroid start {b[8]:.0f}, from a vertex start {b[9]:.0f}; "
          f"moved from a centroid {b[10]:.0f}, from a vertex {b[11]:.0f}; projections equal to p {b[12]:.0f}; "
          f"no move at vertex a / b / c: {b[13]:.0f} / {b[14]:.0f} / {b[15]:.0f}")
    tries = b[0] * 1 + b[1] * 2 + b[2] * 3 + b[3] * 4 + b[4] * 4
    print(f"mean tries per call {tries / calls:.2f} (a warp runs the max of its lanes: 4 whenever one lane moves late "
          f"or not at all)")


if __name__ == "__main__":
    main()
