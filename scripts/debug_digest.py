"""Developer tool: field-by-field comparison of chosen envs of the headline workload
against the oracle (where per-env digests disagree)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import paper_2205_03532_b200 as P
    from conftest import env_digests, pack_patch_list
    from oracle import oracle as O
    from paper_2205_03532_b200.scenes import m16_workload

    envs = [int(x) for x in sys.argv[1:]] or [43, 47, 53]
    E = 1024
    w = m16_workload(E, seed=0)
    grid, nut = w["grid"], w["nut"]
    res = P.collide([P.register_sdf(grid)] * E, [P.register_mesh(nut)] * E, w["sdf_pose"], w["mesh_pose"], w["cd"])
    og = O.Grid(grid.values, grid.dims, grid.origin, grid.voxel_size, *grid.mesh_aabb)
    dig = env_digests(res.plan)
    odig = O.collide_digest(og, nut.vertices, nut.triangles, w["sdf_pose"], w["mesh_pose"], w["cd"])
    bad = np.nonzero(dig != odig)[0].tolist()
    print("differing envs:", bad)
    for e in (bad[:4] or envs):
        cd = float(w["cd"][e])
        ref = O.generate_contacts(og, nut.vertices, nut.triangles, w["sdf_pose"][e], w["mesh_pose"][e], cd)
        cs = res.contact_set(e)
        for k, a, b in (("points", cs.points, ref["points"]), ("normals", cs.normals, ref["normals"]),
                        ("depths", cs.depths, ref["depths"]), ("faces", cs.face_indices, ref["faces"])):
            if a.shape != b.shape or not np.array_equal(a, b):
                print(e, "cand", k, a.shape, b.shape)
        r = O.reduce_contacts(ref["points"], ref["normals"], ref["depths"], ref["faces"], min_depth=-cd)
        got = pack_patch_list(res.patches(e), 6)
        for k in ("rep", "nkept", "members", "kept_faces", "wsum", "wp", "wn", "wt", "area", "maxd"):
            a, b = np.asarray(got[k]), np.asarray(r[k])
            if a.shape != b.shape or not np.array_equal(a, b):
                print(e, "patch", k, a.shape, b.shape, np.argwhere(a != b)[:5].tolist() if a.shape == b.shape else "")
        kc = res.plan.kept_cand.cpu().numpy()[e]
        nk = res.plan.patch_nkept.cpu().numpy()[e]
        for q in range(len(r["nkept"])):
            if not np.array_equal(kc[q, : nk[q]], r["kept"][q, : r["nkept"][q]]):
                print(e, "kept_cand", q, kc[q, : nk[q]], r["kept"][q, : r["nkept"][q]])
                break


if __name__ == "__main__":
    main()
