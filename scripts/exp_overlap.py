"""Experiment: the 1024-env step as K concurrent sub-plans of 1024/K envs on K streams
(one CUDA graph, fork/join), to measure how much the phases' different limiters
overlap. Prints ms per step for each K."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2205_03532_b200 as P  # noqa: E402
from paper_2205_03532_b200.scenes import m16_workload  # noqa: E402

E = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
w = m16_workload(E, seed=0)
hs, hm = P.register_sdf(w["grid"]), P.register_mesh(w["nut"])
sp = torch.from_numpy(np.ascontiguousarray(w["sdf_pose"])).cuda()
mp = torch.from_numpy(np.ascontiguousarray(w["mesh_pose"])).cuda()
cd = torch.from_numpy(np.ascontiguousarray(w["cd"])).cuda()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
main = torch.cuda.current_stream()
SEQ = len(sys.argv) > 2 and sys.argv[2] == "seq"  # sub-plans one after the other on one stream
for K in (1, 2, 4, 8, 16):
    n = E // K
    plans = [P.Plan([hs] * n, [hm] * n, P.ReductionParams()) for _ in range(K)]
    sl = [(k * n, (k + 1) * n) for k in range(K)]
    args = [(sp[a:b].contiguous(), mp[a:b].contiguous(), cd[a:b].contiguous()) for a, b in sl]
    streams = [torch.cuda.Stream() for _ in range(K)]
    for pl, a in zip(plans, args):
        pl.collide(*a)  # eager first call (lazy setup outside capture)
    torch.cuda.synchronize()
    cap = torch.cuda.Stream()
    cap.wait_stream(main)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=cap):
        for s in streams:
            s.wait_stream(cap)
        for pl, s, a in zip(plans, streams, args):
            pl.collide(*a, stream=cap if SEQ else s)
        for s in streams:
            cap.wait_stream(s)
    for _ in range(5):
        g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(main)
        g.replay()
        b.record(main)
        ts.append((a, b))
    torch.cuda.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in ts) / len(ts)
    ncand = sum(int(pl.n_cand.sum()) for pl in plans)
    print(f"K={K} envs/plan={n} ms/step={ms:.3f} n_cand={ncand}", flush=True)
    del g, plans
    torch.cuda.synchronize()
