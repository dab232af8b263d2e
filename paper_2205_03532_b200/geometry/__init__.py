from .fasteners import (
    ThreadSpec,
    bolt_thread_base_z,
    generate_iso_thread,
    generate_peg_hole,
    make_box,
)
from .mesh import TriMesh

__all__ = ["TriMesh", "ThreadSpec", "bolt_thread_base_z", "generate_iso_thread", "generate_peg_hole", "make_box"]
