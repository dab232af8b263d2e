"""Run the synthetic reduction goldens case by case (for compute-sanitizer)."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2205_03532_b200 as P

s = np.load("tests/golden/red_synth.npz")
for c in s["cases"]:
    pre = f"c{c}_"
    N, K, cone, md, bs = s[pre + "params"]
    cs = P.ContactSet(s[pre + "cs_points"], s[pre + "cs_normals"], s[pre + "cs_depths"], s[pre + "cs_faces"], 0, 1)
    rp = P.ReductionParams(int(N), int(K), float(cone), None if np.isnan(md) else float(md), int(bs))
    print("case", c, "n", len(cs), "params", (int(N), int(K), float(cone), md, int(bs)), flush=True)
    patches = P.reduce_contacts(cs, rp)
    print("  ok", len(patches), flush=True)
