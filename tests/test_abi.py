"""CPU checks of the C-ABI library: it loads without a GPU and exports every
symbol include/contactsim_b200.h declares (no compute calls here)."""

import os
import re

from conftest import ROOT


def _declared():
    text = open(os.path.join(ROOT, "include", "contactsim_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(cs_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = _declared()
    for required in ("cs_face_contacts", "cs_sdf_register", "cs_mesh_register", "cs_plan_create", "cs_collide",
                     "cs_reduce", "cs_sdf_generate", "cs_last_error"):
        assert required in names


def test_library_exports_every_declared_symbol():
    from paper_2205_03532_b200 import _native

    so = _native.load_symbols_only()
    missing = [n for n in _declared() if not hasattr(so, n)]
    assert not missing, missing
    assert set(_declared()) == set(_native.EXPORTED)
    assert so.cs_abi_version() == 1


def test_library_is_sm100a():
    from paper_2205_03532_b200 import _native
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True,
                         text=True)
    assert out.returncode == 0, out.stderr
    assert "sm_100a" in out.stdout


def test_error_string_roundtrip():
    from paper_2205_03532_b200 import _native
    import ctypes

    so = _native.load_symbols_only()
    h = ctypes.c_int32(-1)
    # argument validation happens before any CUDA call
    st = so.cs_sdf_register(None, 0, 1, 1, 1, None, 1.0, None, None, ctypes.byref(h))
    assert st == _native.CS_ERR_VALUE
    assert b"dims" in so.cs_last_error()
