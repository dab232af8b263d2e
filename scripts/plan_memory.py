"""Device memory of a collide plan per env (M16 nut on the res-256 bolt), measured
with cudaMemGetInfo around Plan creation. Sizes the largest env count one GPU holds.

    python scripts/plan_memory.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2205_03532_b200 as P  # noqa: E402
from paper_2205_03532_b200.scenes import m16_workload  # noqa: E402


def main():
    w = m16_workload(16, seed=0, resolution=256)
    hs, hm = P.register_sdf(w["grid"]), P.register_mesh(w["nut"])
    torch.cuda.synchronize()
    free0, total = torch.cuda.mem_get_info()
    for E in (1024, 4096):
        f0 = torch.cuda.mem_get_info()[0]
        plan = P.Plan([hs] * E, [hm] * E, P.ReductionParams())
        torch.cuda.synchronize()
        used = f0 - torch.cuda.mem_get_info()[0]
        print(json.dumps({"envs": E, "plan_bytes": used, "per_env_mb": used / E / 1e6,
                          "max_envs_estimate": int(free0 * 0.97 / (used / E)), "gpu_total_bytes": total}))
        del plan


if __name__ == "__main__":
    main()
