"""Developer check: run the same collide step repeatedly (eager and CUDA-graph replay)
and report every output element that differs between runs, including padding.
    python scripts/determinism_check.py [reps]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2205_03532_b200 as P  # noqa: E402

G = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    g = np.load(os.path.join(G, "grid_bolt_r64.npz"))
    m = np.load(os.path.join(G, "meshes.npz"))
    gen = np.load(os.path.join(G, "gen_r64.npz"))
    grid = P.SignedDistanceGrid(g["origin"], float(g["voxel"]), g["dims"], g["values"], (g["aabb_lo"], g["aabb_hi"]))
    nut = P.TriMesh(m["nut_v"], m["nut_t"])
    envs = list(gen["envs"])
    E = len(envs)
    plan = P.Plan([P.register_sdf(grid)] * E, [P.register_mesh(nut)] * E, P.ReductionParams())
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float64)).cuda()  # noqa: E731
    sp = d(np.stack([gen[f"e{e}_sdf_pose"] for e in envs]))
    mp = d(np.stack([gen[f"e{e}_mesh_pose"] for e in envs]))
    cd = d(np.full(E, float(gen["cd"])))
    keys = ("n_cand", "cand_point", "cand_normal", "cand_face", "n_patch", "patch_normal", "patch_nkept", "n_kept", "kept_point",
            "kept_normal", "kept_depth", "kept_face", "w_sum", "area", "max_depth")
    keys = [k for k in keys if hasattr(plan, k)]

    def snap():
        torch.cuda.synchronize()
        return {k: getattr(plan, k).clone() for k in keys}

    plan.collide(sp, mp, cd)
    ref = snap()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=s):
        plan.collide(sp, mp, cd, stream=s)
    nbad = 0
    for r in range(reps):
        if r % 2:
            gr.replay()
        else:
            plan.collide(sp, mp, cd)
        got = snap()
        for k in keys:
            a, b = got[k], ref[k]
            if not torch.equal(a, b):
                diff = (a != b) & ~(torch.isnan(a) & torch.isnan(b)) if a.is_floating_point() else (a != b)
                idx = torch.nonzero(diff)
                nbad += 1
                print(f"rep {r} ({'graph' if r % 2 else 'eager'}): {k} differs at {idx.shape[0]} elements, first "
                      f"{idx[:4].tolist()} got {a[tuple(idx[0])].tolist()} ref {b[tuple(idx[0])].tolist()}", flush=True)
    print(f"{reps} reps, {nbad} differing (rep, field) pairs; n_kept {plan.n_kept.sum().item() if hasattr(plan, 'n_kept') else '?'}")


if __name__ == "__main__":
    main()
