"""B200-native SDF contact generation + contact reduction (Factory, arXiv 2205.03532).

Drop-in for the hot path of the reference package `contactsim`:
SDF asset registration, per-pair `generate_contacts` / `reduce_contacts`, and the
batched `collide` over thousands of envs, and the contact solver that consumes
the reduced contacts (`dynamics`: ContactConstraints / gauss_seidel_sweeps and
the batched `Plan.solve`). All compute runs in hand-written
sm_100a CUDA (libcontactsim_b200.so, C ABI in include/contactsim_b200.h); there
is no CPU fallback.
"""

from .collide import Plan, ReducedContacts, collide, pin_sdf_in_l2, register_mesh, register_sdf
from .contacts import (
    BodyShape,
    CollisionPairing,
    Contact,
    ContactPatch,
    ContactSet,
    ReductionParams,
    assign_roles,
    generate_contacts,
    reduce_contacts,
)
from .dynamics import BatchedSolverState, ContactConstraints, SolverParams, SolverState
from .errors import ContactSimError, MeshValidationError, NonFiniteStateError
from .geometry import TriMesh
from .math3d import Transform
from .sdf import SdfResolutionSpec, SignedDistanceGrid, cached_sdf, generate_sdf

__all__ = [
    "Plan", "ReducedContacts", "collide", "pin_sdf_in_l2", "register_mesh", "register_sdf",
    "BodyShape", "CollisionPairing", "Contact", "ContactPatch", "ContactSet", "ReductionParams",
    "assign_roles", "generate_contacts", "reduce_contacts",
    "SolverParams", "SolverState", "ContactConstraints", "BatchedSolverState",
    "ContactSimError", "MeshValidationError", "NonFiniteStateError",
    "TriMesh", "Transform", "SdfResolutionSpec", "SignedDistanceGrid", "cached_sdf", "generate_sdf",
]
