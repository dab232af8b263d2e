"""Config 3 measured: 4096 envs over pegs 4/8/12/16 mm in tight
holes and M4..M20 nuts on bolts (scenes.suite_workload), one collide per step.

    python scripts/bench_config3.py [--envs 4096 --steps 20 --warmup 3]
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import ClockSampler  # noqa: E402  (nvidia-smi clocks during the timed steps)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--envs", type=int, default=4096)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    args = ap.parse_args()
    import torch

    import paper_2205_03532_b200 as P
    from paper_2205_03532_b200.scenes import suite_workload

    E = args.envs
    w = suite_workload(E, seed=1)
    A, asset = w["assets"], w["asset"]
    hs = [P.register_sdf(a["grid"]) for a in A]
    hm = [P.register_mesh(a["mesh"]) for a in A]
    plan = P.Plan([hs[k] for k in asset], [hm[k] for k in asset], P.ReductionParams())
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float64)).cuda()  # noqa: E731
    sp, mp, cd = dev(w["sdf_pose"]), dev(w["mesh_pose"]), dev(w["cd"])
    for _ in range(args.warmup):
        plan.collide(sp, mp, cd)
    torch.cuda.synchronize()
    plan.enable_timing(args.steps)
    clocks = ClockSampler(torch.cuda.current_device())
    for _ in range(args.steps):
        plan.collide(sp, mp, cd)
    torch.cuda.synchronize()
    clk = clocks.stop()
    ph = plan.read_timing(args.steps)
    t = float(ph[:, plan.PHASES.index("total")].mean())
    faces = int(sum(len(A[k]["mesh"].triangles) for k in asset))
    nc = plan.n_cand.cpu().numpy()
    line = {"workload": f"config 3: {E} envs, pegs 4/8/12/16 mm + M4..M20 nut/bolt (9 assets, res 256)",
            "ms_per_step": t, "face_queries_per_s": faces / (t * 1e-3),
            "phase_ms": {n: float(ph[:, i].mean()) for i, n in enumerate(plan.PHASES)},
            "candidates_per_env": {a["name"]: float(nc[asset == k].mean()) for k, a in enumerate(A)},
            "grids": {a["name"]: list(a["grid"].dims) for a in A},
            "steps": args.steps, "warmup": args.warmup, "dtype": "f64", "clocks": clk,
            "timing": "CUDA events around each eager collide (Plan.enable_timing)",
            "data": "synthetic (seeded poses, procedural assets)"}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
