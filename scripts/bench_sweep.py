"""Config 5 measured: SDF resolution x env count on one GPU
(M16 nut on bolt, seeded poses), one collide per step, CUDA-event phase timing.

    python scripts/bench_sweep.py [--res 64 128 256 512] [--envs 1024 4096 16384]

Prints one JSON line per (res, envs). A plan takes 4.3 MB per env (scripts/plan_memory.py),
so one B200 holds about 43 k envs; beyond that, shard envs over GPUs (bench.py --gpus N).
"""
import argparse
import gc
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import ClockSampler  # noqa: E402  (nvidia-smi clocks during the timed steps)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--res", type=int, nargs="+", default=[64, 128, 256, 512])
    ap.add_argument("--envs", type=int, nargs="+", default=[1024, 4096, 16384])
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    args = ap.parse_args()
    if len(args.res) * len(args.envs) > 1:  # one process per point: every plan's buffers are released
        import subprocess

        for res in args.res:
            for E in args.envs:
                out = subprocess.run([sys.executable, os.path.abspath(__file__), "--res", str(res), "--envs", str(E),
                                      "--steps", str(args.steps), "--warmup", str(args.warmup)],
                                     capture_output=True, text=True)
                lines = [x for x in out.stdout.splitlines() if x.startswith("{")]
                print(lines[-1] if lines else json.dumps({"res": res, "envs": E, "error": out.stderr[-300:]}),
                      flush=True)
        return
    import torch

    import paper_2205_03532_b200 as P
    from paper_2205_03532_b200.scenes import m16_meshes, m16_workload
    from paper_2205_03532_b200.sdf.grid import SdfResolutionSpec, generate_sdf

    nut, bolt, _ = m16_meshes()
    F = len(nut.triangles)
    hm = P.register_mesh(nut)
    for res in args.res:
        grid = generate_sdf(bolt, SdfResolutionSpec(res, 4))
        hs = P.register_sdf(grid)
        for E in args.envs:
            w = m16_workload(E, grid=grid)
            plan = P.Plan([hs] * E, [hm] * E, P.ReductionParams())
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
            nc = plan.n_cand.cpu().numpy()
            print(json.dumps({"res": res, "dims": list(grid.dims), "grid_mb": grid.values.nbytes / 1e6, "envs": E,
                              "ms_per_step": t, "face_queries_per_s": E * F / (t * 1e-3),
                              "candidates_per_env": float(nc.mean()),
                              "phase_ms": {n: float(ph[:, i].mean()) for i, n in enumerate(plan.PHASES)},
                              "clocks": clk, "timing": "CUDA events around each eager collide"}), flush=True)
            del plan, sp, mp, cd  # frees the plan's buffers (collide._PlanHandle)
            gc.collect()
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
