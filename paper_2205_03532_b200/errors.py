"""Exception classes, name- and hierarchy-compatible with contactsim.errors
(/root/reference/pkg/src/contactsim/errors.py:4-27), so `except` clauses written
against the reference keep working. The C ABI reports failures as cs_status
codes; `_native.check` raises the matching class below.
"""


class ContactSimError(Exception):
    """Base class; every error raised by this package derives from it."""


class MeshValidationError(ContactSimError, ValueError):
    """Mesh rejected at registration (bad indices, non-finite vertices, not
    watertight for SDF generation, grid above the voxel guard)."""


class ObjParseError(MeshValidationError):
    """OBJ text could not be parsed; `lineno` is 1-based (0 = whole file)."""

    def __init__(self, message: str, lineno: int):
        self.lineno = lineno
        super().__init__(message if not lineno else f"line {lineno}: {message}")


class SceneConfigError(ContactSimError, ValueError):
    """Invalid scene / collide configuration (the message names the key)."""


class NonFiniteStateError(ContactSimError, RuntimeError):
    """A pose handed to contact generation is NaN/inf (flagged per env on device)."""


class SingularOrientationError(ContactSimError, ValueError):
    """Orientation parametrisation evaluated at its singularity."""
