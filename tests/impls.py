"""TEST INFRASTRUCTURE: one Python mirror API (paper_2202_11770_b200/splb.py)
bound to each implementation of the include/splbcu.h C-ABI:

  product   paper_2202_11770_b200/libsplbcu.so   (B200 engine)
  port      oracle/liboracle.so                  (plain-C restatement)
  reference oracle/_ref/libsplbref.so            (unmodified reference headers)

Only tests/, __graft_entry__.smoke() and bench.py's CPU arm import this.
"""
from __future__ import annotations

import ctypes
import os
import sys
import types

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PORT_LIB = os.path.join(ROOT, "oracle", "liboracle.so")
REF_LIB = os.path.join(ROOT, "oracle", "_ref", "libsplbref.so")
PKG = os.path.join(ROOT, "paper_2202_11770_b200")

_cache = {}


def _load_file(path: str, name: str):
    """Imports a module by file path (no package __init__, so nothing that
    dlopens libsplbcu.so runs)."""
    import importlib.util
    spec = importlib.util.spec_from_file_location(name, path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def _bind(path: str, name: str):
    """The product's Python mirror (splb.py) executed over another library
    implementing the same C-ABI.  Only `_abi.py` (pure ctypes declarations)
    and the mirror's source are read from the package: the product library
    is never mapped into a process that only uses the oracles."""
    A = _load_file(os.path.join(PKG, "_abi.py"), name + "_abi")
    lib = ctypes.CDLL(path)
    for fn, res, args in A.SIGNATURES:
        f = getattr(lib, fn)
        f.restype = res
        f.argtypes = args
    shim = types.SimpleNamespace(lib=lib, Iolet=A.Iolet, BC=A.BC, Params=A.Params)
    spath = os.path.join(PKG, "splb.py")
    src = open(spath).read().replace("from . import _lib as L\n", "")
    mod = types.ModuleType(name)
    mod.__dict__["L"] = shim
    mod.__dict__["__name__"] = name
    sys.modules[name] = mod
    exec(compile(src, spath, "exec"), mod.__dict__)
    return mod


def product():
    from paper_2202_11770_b200 import splb
    return splb


def port():
    if "port" not in _cache:
        if not os.path.exists(PORT_LIB):
            raise RuntimeError("oracle/liboracle.so not built (make -C oracle)")
        _cache["port"] = _bind(PORT_LIB, "splb_port")
    return _cache["port"]


def have_reference() -> bool:
    return os.path.exists(REF_LIB)


def reference():
    if "ref" not in _cache:
        _cache["ref"] = _bind(REF_LIB, "splb_ref")
    return _cache["ref"]
