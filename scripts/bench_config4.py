"""Config 4: multi-pair scenes, one device pipeline per step.

    python scripts/bench_config4.py [--scenes 2048 --steps 20 --warmup 3]

Each scene: static bolt (SDF, res 256), dynamic M16 nut (mesh), two chain-driven
finger pads (make_box((0.004, 0.016, 0.008), subdivisions=8), SDF res 64) against
the nut's flats at x = +-(14 mm - 0.05 mm) in the nut frame. A step is
MultiPairScenes.step: world AABBs -> broadphase -> pair-slot mask -> collide over
every candidate pair slot (bolt-nut, pad-nut x2). Prints one JSON line.
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
    ap.add_argument("--scenes", type=int, default=2048)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    args = ap.parse_args()
    import torch

    import paper_2205_03532_b200 as P
    from paper_2205_03532_b200.geometry import make_box
    from paper_2205_03532_b200.math3d import quat_to_matrix
    from paper_2205_03532_b200.multipair import MultiPairScenes, SceneBody
    from paper_2205_03532_b200.scenes import m16_workload

    S = args.scenes
    w = m16_workload(S)
    bolt, nut, grid = w["bolt"], w["nut"], w["grid"]
    pad = make_box((0.004, 0.016, 0.008), subdivisions=8)
    pad_grid = P.generate_sdf(pad, P.SdfResolutionSpec(64, 4))
    hb, hbm, hn = P.register_sdf(grid), P.register_mesh(bolt), P.register_mesh(nut)
    hp, hpm = P.register_sdf(pad_grid), P.register_mesh(pad)
    scene = lambda: [  # noqa: E731
        SceneBody(0, hbm, bolt.aabb(), len(bolt.triangles), hb, grid.voxel_size, True, True),
        SceneBody(1, hn, nut.aabb(), len(nut.triangles), None, None, False, False),
        SceneBody(2, hpm, pad.aabb(), len(pad.triangles), hp, pad_grid.voxel_size, True, True),
        SceneBody(3, hpm, pad.aabb(), len(pad.triangles), hp, pad_grid.voxel_size, True, True)]
    mps = MultiPairScenes([scene() for _ in range(S)])
    poses = np.zeros((S, 4, 7))
    poses[:, 0] = w["sdf_pose"]
    poses[:, 1] = w["mesh_pose"]
    for i in range(S):
        mp = w["mesh_pose"][i]
        R = quat_to_matrix(mp[3:])
        for b, sgn in ((2, 1.0), (3, -1.0)):
            poses[i, b, :3] = mp[:3] + R @ np.array([sgn * (0.014 - 0.00005), 0.0, 0.0])
            poses[i, b, 3:] = mp[3:]
    dp = torch.from_numpy(poses.reshape(-1, 7)).cuda()
    res = mps.step(dp)  # checked once
    for _ in range(args.warmup):
        mps.step(dp, check=False)
    torch.cuda.synchronize()
    ms = []
    clocks = ClockSampler(torch.cuda.current_device())
    for _ in range(args.steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        mps.step(dp, check=False)
        b.record()
        b.synchronize()
        ms.append(a.elapsed_time(b))
    clk = clocks.stop()
    # the substep's contact solve of every scene (4 bodies; nut dynamic, bolt static, pads chain-driven)
    from paper_2205_03532_b200.dynamics import BatchedSolverState, SolverParams

    ref = np.zeros((S, 4, 3)); W = np.zeros((S, 4, 6, 6)); vel = np.zeros((S, 4, 6))
    ref[:, 1] = w["mesh_pose"][:, :3]
    W[:, 1, :3, :3] = np.eye(3) / 0.03
    W[:, 1, 3:, 3:] = np.diag(1.0 / np.array([2.4e-6, 2.4e-6, 3.9e-6]))
    vel[:, 1, 2] = -0.05
    st = BatchedSolverState.from_numpy(ref, W, vel)
    vel0 = st.vel.clone()
    prm = SolverParams()
    mps.step(dp, check=False)
    sms = []
    for it in range(args.warmup + args.steps):
        st.vel.copy_(vel0); st.impulse.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        mps.solve(st, prm)
        b.record()
        b.synchronize()
        if it >= args.warmup:
            sms.append(a.elapsed_time(b))
    nc = res.n_cand.cpu().numpy()
    act = mps.active.cpu().numpy().astype(bool)
    kind = np.where(mps.slot_sdf_body == 0, "bolt-nut", "pad-nut")
    t = float(np.median(ms))
    F = len(nut.triangles)
    line = {"workload": f"config 4: {S} scenes x (bolt r256, nut, 2 pads r64), 3 pair slots each",
            "ms_per_step": t, "pair_slots": int(mps.n_slots), "active_pairs": int(act.sum()),
            "face_queries_per_s": float(act.sum() * F / (t * 1e-3)),
            "candidates_per_pair": {k: float(nc[(kind == k) & act].mean()) for k in ("bolt-nut", "pad-nut")},
            "patches_per_pair": {k: float(res.n_patch.cpu().numpy()[(kind == k) & act].mean())
                                 for k in ("bolt-nut", "pad-nut")},
            "solve_ms": float(np.median(sms)), "solve": "MultiPairScenes.solve: 16 pos + 1 vel sweeps per scene",
            "steps": args.steps, "warmup": args.warmup, "dtype": "f64", "clocks": clk,
            "timing": "CUDA events around each eager MultiPairScenes.step / solve (median)",
            "data": "synthetic (seeded SURVEY §8(d) poses, procedural assets)"}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
