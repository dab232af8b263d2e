from .fasteners import (
    ThreadSpec,
    bolt_thread_base_z,
    generate_iso_thread,
    generate_peg_hole,
    make_box,
)
from .broadphase import aabb_of_points, aabb_overlap, broadphase_batched, broadphase_pairs, world_aabbs
from .mesh import TriMesh

__all__ = ["TriMesh", "broadphase_pairs", "broadphase_batched", "world_aabbs", "aabb_of_points", "aabb_overlap", "ThreadSpec", "bolt_thread_base_z", "generate_iso_thread", "generate_peg_hole", "make_box"]
