"""Contact solver, the consumer of the reduced contacts.

Mirrors contactsim/dynamics/solver.py: SolverParams (:24-43), SolverState
(:46-77), ContactConstraints (:80-163) with build / position_sweeps /
velocity_sweeps / body_wrenches, and solve_contact_sweep (:174-176). Same names,
fields, argument meaning and errors; the arithmetic runs on the GPU
(csrc/cs_solver.cu) and is bit-identical to the reference. Arrays stay numpy on
the host like the reference's, so existing callers work unchanged.

The batched path for many scenes at once is `Plan.solve` (collide.py): one
system per env, rows straight from the device-resident reduced contacts.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .. import _native

RESTITUTION_THRESHOLD = 0.5  # m/s; impacts slower than this take e = 0 (solver.py:21)


@dataclass
class SolverParams:
    dt: float = 1.0 / 60.0
    substeps: int = 1
    pos_iterations: int = 16
    vel_iterations: int = 1
    penetration_slop: float | None = None  # None: 0.5 * voxel of the pair's grid
    bias_factor: float = 0.2
    contact_distance: float | None = None  # None: 2 * voxel of the pair's grid

    def __post_init__(self):
        if self.dt <= 0.0:
            raise ValueError("dt must be positive")
        if self.substeps < 1:
            raise ValueError("substeps must be at least 1")
        if self.pos_iterations < 1:
            raise ValueError("pos_iterations must be at least 1")
        if self.vel_iterations < 0:
            raise ValueError("vel_iterations must be non-negative")

    def to_c(self) -> _native.SolverParamsC:
        return _native.SolverParamsC(self.dt / self.substeps, self.bias_factor, self.pos_iterations,
                                     self.vel_iterations)


SOLVER_MAX_BODIES = 1 << 20  # cs_solver.cuh SOLVER_MAX_BODIES


def check_solver_bodies(nb: int) -> None:
    """Systems up to 8 bodies keep their state on chip; larger ones (any size the
    reference takes) run the sweeps with the state in global memory. The bound only
    keeps the device's element indices in 32 bits."""
    if not 1 <= int(nb) <= SOLVER_MAX_BODIES:
        raise ValueError(f"the device contact solver handles systems of 1..{SOLVER_MAX_BODIES} bodies per call "
                         f"(got {int(nb)})")


class SolverState:
    """Twist (at a reference point) + 6x6 inverse mobility per body (solver.py:46-77)."""

    def __init__(self, n_bodies: int):
        self.ref = np.zeros((n_bodies, 3))
        self.w_mat = np.zeros((n_bodies, 6, 6))
        self.vel = np.zeros((n_bodies, 6))
        self.impulse = np.zeros((n_bodies, 6))

    @classmethod
    def from_bodies(cls, bodies) -> "SolverState":
        """Duck-typed over the reference's RigidBody (dynamics/body.py)."""
        state = cls(len(bodies))
        for i, body in enumerate(bodies):
            if body.is_static or body.driven_by_chain:
                continue
            state.ref[i] = body.com_world()
            inv_m = body.inv_mass()
            state.w_mat[i, 0, 0] = state.w_mat[i, 1, 1] = state.w_mat[i, 2, 2] = inv_m
            state.w_mat[i, 3:, 3:] = body.inv_inertia_world()
            state.vel[i, :3] = body.linear_velocity
            state.vel[i, 3:] = body.angular_velocity
        return state

    def write_back(self, bodies) -> None:
        for i, body in enumerate(bodies):
            if body.is_static or body.driven_by_chain:
                continue
            body.linear_velocity = self.vel[i, :3].copy()
            body.angular_velocity = self.vel[i, 3:].copy()


def _t(a, dtype=None):
    import torch

    a = np.ascontiguousarray(a, dtype=dtype or np.float64)
    return torch.from_numpy(a).cuda()


class ContactConstraints:
    """Flattened contact rows for one substep, ready for the sweep (solver.py:80-163)."""

    _F3 = ("point", "ra", "rb", "normal", "tan1", "tan2")
    _F1 = ("depth", "kn", "kt1", "kt2", "mu", "restitution", "bias_target", "restitution_target", "lam_n", "lam_t1",
           "lam_t2", "lam_vel")

    def __init__(self, n: int):
        self.body_a = np.zeros(n, dtype=np.int64)
        self.body_b = np.zeros(n, dtype=np.int64)
        for k in self._F3:
            setattr(self, k, np.zeros((n, 3)))
        for k in self._F1:
            setattr(self, k, np.zeros(n))

    def __len__(self) -> int:
        return len(self.depth)

    @classmethod
    def build(cls, rows: list[dict], state: SolverState, h: float, bias_factor: float) -> "ContactConstraints":
        """rows: dicts with body_a, body_b, point, normal, depth, mu, restitution, slop.
        Order is preserved and defines the sweep order (solver.py:105-141)."""
        import torch

        con = cls(len(rows))
        m = len(rows)
        if m == 0:
            return con
        con.body_a[:] = [r["body_a"] for r in rows]
        con.body_b[:] = [r["body_b"] for r in rows]
        con.point[:] = [r["point"] for r in rows]
        con.normal[:] = [r["normal"] for r in rows]
        con.depth[:] = [r["depth"] for r in rows]
        con.mu[:] = [r["mu"] for r in rows]
        con.restitution[:] = [r["restitution"] for r in rows]
        slop = np.array([r["slop"] for r in rows], dtype=np.float64)
        nb = len(state.vel)
        check_solver_bodies(nb)
        d_in = [_t(con.body_a, np.int64), _t(con.body_b, np.int64), _t(con.point), _t(con.normal), _t(con.depth),
                _t(con.restitution), _t(slop), _t(state.ref), _t(state.w_mat), _t(state.vel)]
        names = ("ra", "rb", "tan1", "tan2", "kn", "kt1", "kt2", "bias_target", "restitution_target")
        d_out = {k: torch.zeros(getattr(con, k).shape, dtype=torch.float64, device="cuda") for k in names}
        off = torch.tensor([0, m], dtype=torch.int64, device="cuda")
        _native.call("cs_constraints_build", 1, nb, off.data_ptr(), *(t.data_ptr() for t in d_in[:7]),
                     *(t.data_ptr() for t in d_in[7:]), float(h), float(bias_factor),
                     *(d_out[k].data_ptr() for k in names), _native.stream_handle())
        for k in names:
            getattr(con, k)[...] = d_out[k].cpu().numpy()
        return con

    def _sweeps(self, state: SolverState, iterations: int, target: np.ndarray, lam_n: np.ndarray, friction: bool):
        from ._kernels import gauss_seidel_sweeps

        gauss_seidel_sweeps(iterations, state.w_mat, state.vel, state.impulse, self.body_a, self.body_b, self.ra,
                            self.rb, self.normal, self.tan1, self.tan2, self.kn, self.kt1, self.kt2, target, self.mu,
                            lam_n, self.lam_t1, self.lam_t2, friction)

    def position_sweeps(self, state: SolverState, iterations: int) -> None:
        if len(self) == 0 or iterations == 0:
            return
        self._sweeps(state, iterations, self.bias_target, self.lam_n, True)

    def velocity_sweeps(self, state: SolverState, iterations: int) -> None:
        if len(self) == 0 or iterations == 0:
            return
        self._sweeps(state, iterations, self.restitution_target, self.lam_vel, False)

    def body_wrenches(self, n_bodies: int, h: float) -> np.ndarray:
        """(nb, 6) net contact force/torque per body over this substep (solver.py:154-163)."""
        import torch

        m = len(self)
        if m == 0:
            return np.zeros((n_bodies, 6))
        check_solver_bodies(n_bodies)
        out = torch.zeros((n_bodies, 6), dtype=torch.float64, device="cuda")
        off = torch.tensor([0, m], dtype=torch.int64, device="cuda")
        d = [_t(self.body_a, np.int64), _t(self.body_b, np.int64)] + [
            _t(getattr(self, k)) for k in ("ra", "rb", "normal", "tan1", "tan2", "lam_n", "lam_vel", "lam_t1",
                                           "lam_t2")]
        _native.call("cs_body_wrenches", 1, int(n_bodies), off.data_ptr(), *(t.data_ptr() for t in d), float(h),
                     out.data_ptr(), _native.stream_handle())
        return out.cpu().numpy()


def solve_contact_sweep(constraints: ContactConstraints, state: SolverState) -> None:
    """One in-order position-phase sweep; exposed for unit-level verification (solver.py:174-176)."""
    constraints.position_sweeps(state, 1)


class BatchedSolverState:
    """Device SolverState of E systems of n_bodies each (float64 CUDA tensors:
    ref (E,nb,3), w_mat (E,nb,6,6), vel (E,nb,6), impulse (E,nb,6)). For Plan.solve
    nb = 2: body 0 is each env's SDF body, body 1 its mesh body (scene.py:228-243);
    for MultiPairScenes.solve the scene's bodies in order."""

    def __init__(self, n_envs: int, n_bodies: int = 2):
        import torch

        z = lambda *s: torch.zeros(s, dtype=torch.float64, device="cuda")  # noqa: E731
        self.ref = z(n_envs, n_bodies, 3)
        self.w_mat = z(n_envs, n_bodies, 6, 6)
        self.vel = z(n_envs, n_bodies, 6)
        self.impulse = z(n_envs, n_bodies, 6)

    @classmethod
    def from_numpy(cls, ref, w_mat, vel, impulse=None) -> "BatchedSolverState":
        import torch

        st = cls(len(ref), np.asarray(ref).shape[1])
        st.ref.copy_(torch.from_numpy(np.ascontiguousarray(ref, np.float64)))
        st.w_mat.copy_(torch.from_numpy(np.ascontiguousarray(w_mat, np.float64)))
        st.vel.copy_(torch.from_numpy(np.ascontiguousarray(vel, np.float64)))
        if impulse is not None:
            st.impulse.copy_(torch.from_numpy(np.ascontiguousarray(impulse, np.float64)))
        return st
