"""Contact solver oracle (oracle/cs_oracle_solver.c) pinned bit for bit against the
reference's own outputs (tests/golden/solver.npz, tests/golden/make_solver_golden.py):
ContactConstraints.build (dynamics/solver.py:105-141), gauss_seidel_sweeps
(dynamics/_kernels.py:52-115) and body_wrenches (solver.py:154-163)."""

import numpy as np
import pytest

from conftest import golden
from oracle import oracle as O

BUILD_KEYS = ("ra", "rb", "tan1", "tan2", "kn", "kt1", "kt2", "bias_target", "restitution_target")
G = golden("solver.npz")
CASES = [str(c) for c in G["cases"]]


def case(name):
    return {k[len(name) + 1:]: G[k] for k in G.files if k.startswith(name + "_")}


def same(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and a.tobytes() == b.tobytes()


def run_oracle(c):
    con = O.constraints_build(c["body_a"], c["body_b"], c["point"], c["normal"], c["depth"], c["restitution"],
                              c["slop"], c["ref"], c["w_mat"], c["vel0"], float(c["h"]), float(c["bias"]))
    m, nb = int(c["m"]), int(c["nb"])
    vel = np.array(c["vel0"], dtype=np.float64, order="C")
    imp = np.zeros((nb, 6))
    lam = {k: np.zeros(m) for k in ("lam_n", "lam_t1", "lam_t2", "lam_vel")}
    pos_it, vel_it = (int(x) for x in c["iters"])
    args = (c["body_a"], c["body_b"], con["ra"], con["rb"], c["normal"], con["tan1"], con["tan2"], con["kn"],
            con["kt1"], con["kt2"])
    if m:
        O.gauss_seidel_sweeps(pos_it, c["w_mat"], vel, imp, *args, con["bias_target"], c["mu"], lam["lam_n"],
                              lam["lam_t1"], lam["lam_t2"], True)
    out = {"con": con, "vel_pos": vel.copy(), "imp_pos": imp.copy(), "lam_n": lam["lam_n"].copy()}
    if m:
        O.gauss_seidel_sweeps(vel_it, c["w_mat"], vel, imp, *args, con["restitution_target"], c["mu"],
                              lam["lam_vel"], lam["lam_t1"], lam["lam_t2"], False)
    out.update(vel_end=vel, imp_end=imp, lam=lam)
    out["wrench"] = O.body_wrenches(nb, c["body_a"], c["body_b"], con["ra"], con["rb"], c["normal"], con["tan1"],
                                    con["tan2"], lam["lam_n"], lam["lam_vel"], lam["lam_t1"], lam["lam_t2"],
                                    float(c["h"]))
    return out


@pytest.mark.parametrize("name", CASES)
def test_solver_oracle_bit_exact(name):
    c = case(name)
    r = run_oracle(c)
    for k in BUILD_KEYS:
        assert same(r["con"][k], c[k].reshape(r["con"][k].shape)), f"{name}: build {k}"
    assert same(r["vel_pos"], c["vel_pos"]), f"{name}: velocities after the position sweeps"
    assert same(r["imp_pos"], c["imp_pos"]), f"{name}: impulses after the position sweeps"
    assert same(r["lam_n"], c["lam_n"]), f"{name}: lam_n"
    assert same(r["vel_end"], c["vel_end"]), f"{name}: velocities after the velocity sweeps"
    assert same(r["imp_end"], c["imp_end"]), f"{name}: impulses"
    for k in ("lam_vel", "lam_t1", "lam_t2"):
        assert same(r["lam"][k], c[k]), f"{name}: {k}"
    assert same(r["wrench"], c["wrench"]), f"{name}: body wrenches"


def test_solver_golden_covers_cold_branches():
    """The fixtures exercise every branch of the sweep: clamped normal impulses,
    the friction cone, restitution above the threshold, k = 0 rows, mu = 0 rows."""
    allc = [case(n) for n in CASES]
    assert any((c["restitution_target"] > 0).any() for c in allc if int(c["m"]))
    assert any((c["kn"] == 0).any() for c in allc if int(c["m"]))
    assert any((c["mu"] == 0).any() for c in allc if int(c["m"]))
    assert any(((c["lam_n"] == 0) & (c["kn"] > 0)).any() for c in allc if int(c["m"]))
    lim = [np.hypot(c["lam_t1"], c["lam_t2"]) >= c["mu"] * c["lam_n"] * (1 - 1e-12) for c in allc if int(c["m"])]
    assert any((x & (np.hypot(c["lam_t1"], c["lam_t2"]) > 0)).any() for x, c in zip(lim, [c for c in allc if int(c["m"])]))
