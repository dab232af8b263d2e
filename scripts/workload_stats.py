"""Workload statistics of the headline config on the GPU (developer tool):
candidates per env, patches per env, patch-size distribution, hull sizes.

    python scripts/workload_stats.py [--envs 1024]
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--envs", type=int, default=1024)
    args = ap.parse_args()
    import torch

    import paper_2205_03532_b200 as P
    from paper_2205_03532_b200.scenes import m16_workload

    w = m16_workload(args.envs)
    plan = P.Plan([P.register_sdf(w["grid"])] * args.envs, [P.register_mesh(w["nut"])] * args.envs, P.ReductionParams())
    sp, mp, cd = (torch.from_numpy(np.ascontiguousarray(w[k])).cuda() for k in ("sdf_pose", "mesh_pose", "cd"))
    plan.collide(sp, mp, cd)
    torch.cuda.synchronize()
    nc = plan.n_cand.cpu().numpy()
    npch = plan.n_patch.cpu().numpy()
    mo = plan.member_offsets.cpu().numpy()
    sizes = np.concatenate([np.diff(mo[e, : npch[e] + 1]) for e in range(args.envs)])
    print(f"envs {args.envs}: candidates/env mean {nc.mean():.0f} min {nc.min()} max {nc.max()}")
    print(f"patches/env mean {npch.mean():.1f} max {npch.max()}  total {len(sizes)}")
    qs = [50, 75, 90, 95, 99, 99.9, 100]
    print("patch members percentiles", {q: int(np.percentile(sizes, q)) for q in qs})
    for lim in (32, 64, 128, 256, 512, 1024, 2048, 4096):
        sel = sizes > lim
        print(f"  > {lim:5d}: {sel.sum():6d} patches ({100 * sel.mean():5.1f}%), {sizes[sel].sum():8d} members "
              f"({100 * sizes[sel].sum() / sizes.sum():5.1f}%)")
    fw = plan.face_work.cpu().numpy()
    print(f"face descent: {fw[0]} faces ({fw[0] / args.envs:.0f}/env), {fw[2]} moved by iteration 0, {fw[3]} still moving")
    nk = plan.patch_nkept.cpu().numpy()
    print("kept per env mean", nk.sum(1).mean())


if __name__ == "__main__":
    main()
