"""ctypes binding of libsplbcu.so (include/splbcu.h).

The shared library is built in-tree (``python -m paper_2202_11770_b200.build``
or ``__graft_entry__.build()``).  There is no fallback: if the library is
missing, importing the package raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# SPLBCU_LIB: another build of the same library (e.g. libsplbcu_tuning.so,
# `make -C csrc tuning`, which adds the tuning-sweep kernel variants)
LIB_PATH = os.environ.get("SPLBCU_LIB") or os.path.join(_HERE, "libsplbcu.so")

from ._abi import *  # noqa: F401,F403  (structs, SIGNATURES)
from ._abi import SIGNATURES


def _point_at_torch_nccl() -> None:
    """libsplbcu binds NCCL at run time (csrc/nccl_dyn.hpp).  Point it at the
    libnccl.so.2 PyTorch ships so both share one NCCL whatever the import
    order (two NCCL builds cannot coexist under one soname)."""
    if "SPLBCU_NCCL_LIB" in os.environ:
        return
    try:
        import importlib.util
        spec = importlib.util.find_spec("nvidia.nccl")
        for base in (spec.submodule_search_locations or []) if spec else []:
            cand = os.path.join(base, "lib", "libnccl.so.2")
            if os.path.exists(cand):
                os.environ["SPLBCU_NCCL_LIB"] = cand
                return
    except Exception:
        pass


def load(path: str = LIB_PATH) -> C.CDLL:
    _point_at_torch_nccl()
    if not os.path.exists(path):
        raise ImportError(
            f"libsplbcu.so not built at {path}; run __graft_entry__.build() "
            "(there is no CPU fallback for the engine)")
    lib = C.CDLL(path)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = load()
