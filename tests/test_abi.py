"""The drop-in boundary: every entry point include/splbcu.h declares is
exported by the B200 library (and by both CPU oracles, which implement the
same C-ABI).  Loading only — no compute calls needed."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "splbcu.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = set(re.findall(r"\b(splbcu_[a-z0-9_]+)\s*\(", src))
    return sorted(names)


def test_header_parses():
    names = declared()
    assert "splbcu_sim_create" in names and "splbcu_sim_run" in names
    assert len(names) >= 50


@pytest.mark.parametrize("lib", ["paper_2202_11770_b200/libsplbcu.so", "oracle/liboracle.so",
                                 "oracle/_ref/libsplbref.so"])
def test_exports_every_symbol(lib):
    path = os.path.join(ROOT, lib)
    if not os.path.exists(path):
        if "_ref" in lib:
            pytest.skip("reference shim not built")
        pytest.fail(f"{lib} missing — run __graft_entry__.build()")
    so = ctypes.CDLL(path)
    missing = [n for n in declared() if not hasattr(so, n)]
    assert not missing, missing


def test_python_signatures_cover_header():
    from paper_2202_11770_b200 import _lib
    assert sorted(n for n, _, _ in _lib.SIGNATURES) == declared()


def test_product_is_sm100a():
    """The fatbin inside libsplbcu.so carries sm_100a SASS for the kernels."""
    import shutil
    import subprocess
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cuobjdump):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([cuobjdump, "--list-elf", os.path.join(ROOT, "paper_2202_11770_b200/libsplbcu.so")],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
