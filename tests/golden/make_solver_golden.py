"""Generate tests/golden/solver.npz by running the REFERENCE contact solver.

Run here (the build container), never on the GPU box:

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \\
        python tests/golden/make_solver_golden.py

SURVEY §8(f) row 1: the solver that consumes the reduced contacts. For each case it
records the reference's own outputs of
  ContactConstraints.build      (dynamics/solver.py:105-141)
  position_sweeps / velocity_sweeps -> gauss_seidel_sweeps (dynamics/_kernels.py:52-115)
  body_wrenches                 (dynamics/solver.py:154-163)
on rows laid out exactly as Scene._collect_contacts lays them out
(dynamics/scene.py:228-243: pair, patch slot, kept contact). The contact rows are the
reference's reduced patches of the golden M16 envs (gen_r64.npz / gen_r256.npz),
plus synthetic systems for the cold branches (restitution above the threshold,
static-static rows with k = 0, mu = 0, several bodies, empty systems).
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from contactsim.dynamics.solver import ContactConstraints, SolverState  # noqa: E402
from contactsim.math3d import quat_to_matrix  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def random_inertia(rng, m):
    # a box-like principal inertia, rotated: SPD
    d = m * rng.uniform(1e-6, 5e-6, 3)
    q = rng.standard_normal(4)
    q /= np.linalg.norm(q)
    r = quat_to_matrix(q)
    return r @ np.diag(d) @ r.T


def make_state(rng, nb, dynamic, com):
    st = SolverState(nb)
    for i in range(nb):
        if not dynamic[i]:
            continue
        m = rng.uniform(0.005, 0.05)
        st.ref[i] = com[i]
        st.w_mat[i, 0, 0] = st.w_mat[i, 1, 1] = st.w_mat[i, 2, 2] = 1.0 / m
        st.w_mat[i, 3:, 3:] = np.linalg.inv(random_inertia(rng, m))
        st.vel[i, :3] = rng.standard_normal(3) * 0.05
        st.vel[i, 3:] = rng.standard_normal(3) * 0.5
    return st


def rows_from_patches(g, e, body_a, body_b, mu, rest, slop):
    nk = g[f"e{e}_pt_nkept"]
    rows = []
    for p in range(len(nk)):
        for k in range(int(nk[p])):
            rows.append({"body_a": body_a, "body_b": body_b, "point": g[f"e{e}_pt_kept_points"][p, k].copy(),
                         "normal": g[f"e{e}_pt_kept_normals"][p, k].copy(),
                         "depth": float(g[f"e{e}_pt_kept_depths"][p, k]), "mu": mu, "restitution": rest,
                         "slop": slop})
    return rows


def run_case(out, name, rows, st, h, bias, pos_it, vel_it):
    m = len(rows)
    out[f"{name}_m"] = np.int64(m)
    out[f"{name}_nb"] = np.int64(len(st.vel))
    out[f"{name}_h"] = np.float64(h)
    out[f"{name}_bias"] = np.float64(bias)
    out[f"{name}_iters"] = np.array([pos_it, vel_it], np.int64)
    for k in ("body_a", "body_b"):
        out[f"{name}_{k}"] = np.array([r[k] for r in rows], np.int64).reshape(m)
    for k in ("point", "normal"):
        out[f"{name}_{k}"] = np.array([r[k] for r in rows], np.float64).reshape(m, 3)
    for k in ("depth", "mu", "restitution", "slop"):
        out[f"{name}_{k}"] = np.array([r[k] for r in rows], np.float64).reshape(m)
    out[f"{name}_ref"] = st.ref.copy()
    out[f"{name}_w_mat"] = st.w_mat.copy()
    out[f"{name}_vel0"] = st.vel.copy()
    con = ContactConstraints.build(rows, st, h, bias)
    for k in ("ra", "rb", "tan1", "tan2", "kn", "kt1", "kt2", "bias_target", "restitution_target"):
        out[f"{name}_{k}"] = getattr(con, k).copy()
    con.position_sweeps(st, pos_it)
    out[f"{name}_vel_pos"] = st.vel.copy()
    out[f"{name}_imp_pos"] = st.impulse.copy()
    out[f"{name}_lam_n"] = con.lam_n.copy()
    con.velocity_sweeps(st, vel_it)
    out[f"{name}_vel_end"] = st.vel.copy()
    out[f"{name}_imp_end"] = st.impulse.copy()
    for k in ("lam_vel", "lam_t1", "lam_t2"):
        out[f"{name}_{k}"] = getattr(con, k).copy()
    out[f"{name}_wrench"] = con.body_wrenches(len(st.vel), h)


def main():
    rng = np.random.default_rng(7)
    out = {}
    names = []
    h = 1.0 / 60.0
    for res in (64, 256):
        g = np.load(os.path.join(HERE, f"gen_r{res}.npz"))
        envs = int(g["envs"]) if np.ndim(g["envs"]) == 0 else len(g["envs"])
        voxel = float(g["cd"]) / 2.0 if np.ndim(g["cd"]) == 0 else float(np.asarray(g["cd"]).ravel()[0]) / 2.0
        for e in range(min(envs, 3)):
            # bolt (body 0) static, nut (body 1) dynamic: the Factory pair (scene.py:228-243)
            com = [np.zeros(3), g[f"e{e}_mesh_pose"][:3].copy()]
            st = make_state(rng, 2, [False, True], com)
            st.vel[1, 2] = -0.3  # approaching
            rows = rows_from_patches(g, e, 0, 1, float(np.sqrt(0.5 * 0.5)), 0.0, 0.5 * voxel)
            name = f"r{res}e{e}"
            run_case(out, name, rows, st, h, 0.2, 16, 1)
            names.append(name)
        # both dynamic, restitution and fast impact, several iterations
        com = [np.array([0.0, 0.0, 0.01]), g["e0_mesh_pose"][:3].copy()]
        st = make_state(rng, 2, [True, True], com)
        st.vel[1, 2] = -1.5
        rows = rows_from_patches(g, 0, 0, 1, 0.3, 0.4, 0.5 * voxel)
        name = f"r{res}dyn"
        run_case(out, name, rows, st, h / 4, 0.2, 8, 3)
        names.append(name)
    # synthetic: 3 bodies, two pairs sharing body 1; mu = 0 rows; static-static rows (k = 0)
    m = 60
    rows = []
    for c in range(m):
        n = rng.standard_normal(3)
        n /= np.linalg.norm(n)
        pair = c % 3
        ba, bb = [(0, 1), (2, 1), (0, 2)][pair]
        rows.append({"body_a": ba, "body_b": bb, "point": rng.standard_normal(3) * 0.01, "normal": n,
                     "depth": float(rng.uniform(-2e-4, 4e-4)), "mu": 0.0 if c % 5 == 0 else 0.6,
                     "restitution": 0.5, "slop": 5e-5})
    st = make_state(rng, 3, [True, True, False], [rng.standard_normal(3) * 0.01 for _ in range(3)])
    st.vel[:2] *= 20.0
    run_case(out, "multi", rows, st, h, 0.25, 12, 2)
    names.append("multi")
    st = make_state(rng, 2, [False, False], [np.zeros(3), np.zeros(3)])
    run_case(out, "static", [dict(r, body_a=0, body_b=1) for r in rows[:10]], st, h, 0.2, 4, 1)
    names.append("static")
    st = make_state(rng, 2, [False, True], [np.zeros(3), np.zeros(3)])
    run_case(out, "empty", [], st, h, 0.2, 4, 1)
    names.append("empty")
    out["cases"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "solver.npz"), **out)
    print("wrote solver.npz:", ", ".join(f"{n}({int(out[n + '_m'])} rows)" for n in names))


if __name__ == "__main__":
    main()
