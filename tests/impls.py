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

_cache = {}


def _bind(path: str, name: str):
    from paper_2202_11770_b200 import _lib as L
    from paper_2202_11770_b200 import splb as S
    lib = ctypes.CDLL(path)
    for fn, res, args in L.SIGNATURES:
        f = getattr(lib, fn)
        f.restype = res
        f.argtypes = args
    shim = types.SimpleNamespace(lib=lib, Iolet=L.Iolet, BC=L.BC, Params=L.Params)
    src = open(S.__file__).read().replace("from . import _lib as L\n", "")
    mod = types.ModuleType(name)
    mod.__dict__["L"] = shim
    mod.__dict__["__name__"] = name
    sys.modules[name] = mod
    exec(compile(src, S.__file__, "exec"), mod.__dict__)
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
