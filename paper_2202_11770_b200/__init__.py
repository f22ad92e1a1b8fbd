"""B200-native sparse D3Q19 lattice Boltzmann step (HemeLB / splb hot path).

The engine lives in libsplbcu.so (C-ABI: include/splbcu.h); this package is
the host-side mirror of the reference's `splb` C++ API.
"""
from .splb import *  # noqa: F401,F403
from .splb import Simulation, SparseDomain, partition  # noqa: F401
