"""Experiment: split the 1024 envs into G plans on G streams and time the step."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2205_03532_b200 as P
from paper_2205_03532_b200.scenes import m16_workload

E = 1024
w = m16_workload(E)
hs, hm = P.register_sdf(w["grid"]), P.register_mesh(w["nut"])
sp_all = torch.from_numpy(np.ascontiguousarray(w["sdf_pose"])).cuda()
mp_all = torch.from_numpy(np.ascontiguousarray(w["mesh_pose"])).cuda()
cd_all = torch.from_numpy(np.ascontiguousarray(w["cd"])).cuda()
P.pin_sdf_in_l2(w["grid"], 1.0, torch.cuda.current_stream())
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for G in (1, 2, 4, 8):
    n = E // G
    plans = [P.Plan([hs] * n, [hm] * n, P.ReductionParams()) for _ in range(G)]
    streams = [torch.cuda.Stream() for _ in range(G)]
    for s in streams:
        P.pin_sdf_in_l2(w["grid"], 1.0, s)
    sl = [(sp_all[g * n:(g + 1) * n].contiguous(), mp_all[g * n:(g + 1) * n].contiguous(), cd_all[g * n:(g + 1) * n].contiguous()) for g in range(G)]
    main = torch.cuda.current_stream()
    def step():
        ev = torch.cuda.Event()
        ev.record(main)
        for g in range(G):
            streams[g].wait_event(ev)
            with torch.cuda.stream(streams[g]):
                plans[g].collide(*sl[g], stream=streams[g])
        for g in range(G):
            main.wait_stream(streams[g])
    for _ in range(5):
        step()
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(main); step(); b.record(main); b.synchronize()
        ts.append(a.elapsed_time(b))
    print(f"G={G}: {np.median(ts):.3f} ms per 1024-env step (median of 20)", flush=True)
    del plans
    torch.cuda.synchronize()
