"""The C-ABI library loads and exports every symbol include/glu_b200.h declares
(no compute calls: this runs without a GPU)."""

from __future__ import annotations

import ctypes
import re

from conftest import ROOT


def declared_functions():
    text = (ROOT / "include" / "glu_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(glu_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("glu_symbolic_fillin", "glu_detect_relaxed", "glu_levelize", "glu_plan_build",
                 "glu_create", "glu_factor_device", "glu_factor_host", "glu_solve_device",
                 "glu_solve_host", "glu_destroy", "glu_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_1908_00204_b200 import _lib

    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert missing == []


def test_python_binding_covers_the_header():
    from paper_1908_00204_b200 import _lib

    assert set(declared_functions()) <= set(_lib.SIGNATURES)


def test_library_is_sm100a():
    import subprocess

    from paper_1908_00204_b200 import _lib

    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_version_string():
    from paper_1908_00204_b200 import _lib

    assert b"sm_100a" in _lib.lib.glu_version()
