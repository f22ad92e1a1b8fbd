"""The C++ surface (include/splbcu.hpp over the C-ABI): a restatement of the
reference's engine tests compiled with g++ against libsplbcu.so.  The build is
checked on CPU; the run needs a GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_engine_cpp.cpp")
LIBDIR = os.path.join(ROOT, "paper_2202_11770_b200")


def _build(tmp_path):
    exe = str(tmp_path / "test_engine_cpp")
    cmd = ["g++", "-std=c++17", "-O2", "-ffp-contract=off", f"-I{ROOT}/include", SRC, "-o", exe,
           f"-L{LIBDIR}", "-lsplbcu", f"-Wl,-rpath,{LIBDIR}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_cpp_header_builds(tmp_path):
    _build(tmp_path)


@pytest.mark.gpu
def test_cpp_engine_tests_pass(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 check(s) failed" in r.stdout
