"""Python mirror of the reference's `splb` C++ API, over the C-ABI.

Names, argument meaning and error types follow /root/reference/proj/include/
splb (geometry.hpp, decomp.hpp, boundary.hpp, engine.hpp), so tests read like
the reference's own doctest suites.  Everything here is host plumbing; the
time step runs in libsplbcu.so's sm_100a kernels.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _lib as L

lib = L.lib

# ---- constants (lattice.hpp:20-65) -----------------------------------------
Q = 19
VELOCITIES = np.array([
    [0, 0, 0], [1, 0, 0], [-1, 0, 0], [0, 1, 0], [0, -1, 0], [0, 0, 1], [0, 0, -1],
    [1, 1, 0], [-1, -1, 0], [1, -1, 0], [-1, 1, 0], [1, 0, 1], [-1, 0, -1], [1, 0, -1],
    [-1, 0, 1], [0, 1, 1], [0, -1, -1], [0, 1, -1], [0, -1, 1]], dtype=np.int32)
INVERSE = [0, 2, 1, 4, 3, 6, 5, 8, 7, 10, 9, 12, 11, 14, 13, 16, 15, 18, 17]
CS2 = 1.0 / 3.0
K_AXIS_OFFSET_X = 0.375
K_AXIS_OFFSET_Y = 0.5

AOS, SOA = 0, 1
PUSH, PULL = 0, 1
CLASSIC, REORDERED = 0, 1
PRESSURE, VELOCITY = 0, 1
INLET, OUTLET = 0, 1


# ---- errors (common.hpp:11-28) ------------------------------------------------
class Error(RuntimeError):
    pass


class DegenerateState(Error):
    pass


class GeometryError(Error):
    pass


class ConfigError(Error):
    pass


_ERR = {1: ConfigError, 2: Error, 3: Error, 4: GeometryError, 5: DegenerateState, 6: Error}


def _check(rc: int) -> None:
    if rc != 0:
        raise _ERR.get(rc, Error)(lib.splbcu_last_error().decode())


def _ptr(a: np.ndarray, ct):
    return a.ctypes.data_as(C.POINTER(ct))


# ---- lattice helpers ------------------------------------------------------------
def equilibrium(rho: float, u: Sequence[float]) -> np.ndarray:
    """equilibrium (lattice.hpp:152-158)."""
    out = np.zeros(Q)
    uu = np.asarray(u, dtype=np.float64)
    lib.splbcu_equilibrium(rho, _ptr(uu, C.c_double), _ptr(out, C.c_double))
    return out


def moments(f: Sequence[float]):
    """moments (lattice.hpp:162-170): (rho, u) or DegenerateState."""
    ff = np.ascontiguousarray(f, dtype=np.float64)
    rho = C.c_double()
    u = np.zeros(3)
    _check(lib.splbcu_moments(_ptr(ff, C.c_double), C.byref(rho), _ptr(u, C.c_double)))
    return rho.value, u


def bgk_collide(f: Sequence[float], tau: float) -> np.ndarray:
    """bgk_collide (lattice.hpp:173-185)."""
    ff = np.ascontiguousarray(f, dtype=np.float64)
    out = np.zeros(Q)
    _check(lib.splbcu_bgk_collide(_ptr(ff, C.c_double), tau, _ptr(out, C.c_double)))
    return out


@dataclass
class Iolet:
    """geometry.hpp:44-52."""
    kind: int
    center: Sequence[float]
    normal: Sequence[float]
    radius: float

    def to_c(self) -> L.Iolet:
        x = L.Iolet()
        x.kind = self.kind
        x.center[:] = list(self.center)
        x.normal[:] = list(self.normal)
        x.radius = self.radius
        return x


def iolet_weight(io: Iolet, coords: Sequence[int]) -> float:
    """iolet_weight (boundary.hpp:107-113)."""
    c = np.asarray(coords, dtype=np.int32)
    x = io.to_c()
    return lib.splbcu_iolet_weight(C.byref(x), _ptr(c, C.c_int32))


@dataclass
class TimeTable:
    """boundary.hpp:18-74: piecewise-linear (time, value) nodes."""
    nodes: List[tuple] = field(default_factory=list)
    period: float = 0.0

    @staticmethod
    def constant(v: float) -> "TimeTable":
        return TimeTable([(0.0, v)], 0.0)

    def at(self, t: float) -> float:
        ts = np.array([n[0] for n in self.nodes], dtype=np.float64)
        vs = np.array([n[1] for n in self.nodes], dtype=np.float64)
        out = C.c_double()
        _check(lib.splbcu_timetable_at(_ptr(ts, C.c_double), _ptr(vs, C.c_double), len(ts),
                                       self.period, t, C.byref(out)))
        return out.value


@dataclass
class BCEntry:
    kind: int = PRESSURE
    table: TimeTable = field(default_factory=lambda: TimeTable.constant(CS2))


@dataclass
class BCSet:
    """engine.hpp:37-44."""
    entries: List[BCEntry] = field(default_factory=list)


@dataclass
class EngineParams:
    """engine.hpp:46-57 (+ B200 device placement)."""
    tau: float = 0.9
    rho0: float = 1.0
    dt_s: float = 1.0
    layout: int = AOS
    scheme: int = PUSH
    sequence: int = CLASSIC
    workers: int = 1
    capture_period: int = 0
    observe_iolets: bool = False
    exchange_timeout_s: float = 30.0
    devices: Optional[List[int]] = None
    halo_mode: int = 0  # B200: 0 NCCL / peer copies + PostReceive, 1 fused NVLink P2P stores
    storage: int = 0  # B200: 0 two buffers (push), 1 single buffer (AA pattern, in place)


# ---- domain -----------------------------------------------------------------------
class SparseDomain:
    """geometry.hpp:64-73, owned by libsplbcu.  Field arrays are exported on
    demand as numpy arrays in domain order."""

    def __init__(self, handle):
        self._h = C.c_void_p(handle) if not isinstance(handle, C.c_void_p) else handle

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and h.value:
            lib.splbcu_domain_free(h)
            self._h = C.c_void_p(None)

    @property
    def handle(self):
        return self._h

    def n_sites(self) -> int:
        return int(lib.splbcu_domain_n_sites(self._h))

    @property
    def voxel_size(self) -> float:
        return float(lib.splbcu_domain_voxel_size(self._h))

    def export(self):
        n = self.n_sites()
        nio = int(lib.splbcu_domain_n_iolets(self._h))
        coords = np.zeros((n, 3), np.int32)
        types = np.zeros(n, np.uint8)
        kinds = np.zeros((n, 18), np.uint8)
        iol = np.zeros((n, 18), np.uint16)
        ios = (L.Iolet * max(nio, 1))()
        tr = np.zeros(12, np.uint64)
        _check(lib.splbcu_domain_export(self._h, _ptr(coords, C.c_int32), _ptr(types, C.c_uint8),
                                        _ptr(kinds, C.c_uint8), _ptr(iol, C.c_uint16), ios,
                                        _ptr(tr, C.c_uint64)))
        iolets = [Iolet(ios[k].kind, list(ios[k].center), list(ios[k].normal), ios[k].radius)
                  for k in range(nio)]
        return dict(coords=coords, types=types, link_kind=kinds, link_iolet=iol, iolets=iolets,
                    type_ranges=tr.reshape(6, 2).astype(np.int64), voxel_size=self.voxel_size)

    @property
    def iolets(self) -> List[Iolet]:
        nio = int(lib.splbcu_domain_n_iolets(self._h))
        ios = (L.Iolet * max(nio, 1))()
        _check(lib.splbcu_domain_export(self._h, None, None, None, None, ios, None))
        return [Iolet(ios[k].kind, list(ios[k].center), list(ios[k].normal), ios[k].radius) for k in range(nio)]

    @property
    def type_ranges(self) -> np.ndarray:
        """[begin, end) of each CollisionType in site order (SparseDomain::type_ranges)."""
        tr = np.zeros(12, np.uint64)
        _check(lib.splbcu_domain_export(self._h, None, None, None, None, None, _ptr(tr, C.c_uint64)))
        return tr.reshape(6, 2).astype(np.int64)

    def validate(self) -> None:
        _check(lib.splbcu_domain_validate(self._h))

    def write(self, path: str) -> None:
        _check(lib.splbcu_domain_write(self._h, path.encode()))

    @staticmethod
    def read(path: str) -> "SparseDomain":
        h = C.c_void_p()
        _check(lib.splbcu_domain_read(path.encode(), C.byref(h)))
        return SparseDomain(h)

    @staticmethod
    def from_arrays(coords, types, link_kind, link_iolet, iolets, type_ranges, voxel_size=1.0):
        coords = np.ascontiguousarray(coords, np.int32)
        types = np.ascontiguousarray(types, np.uint8)
        link_kind = np.ascontiguousarray(link_kind, np.uint8)
        link_iolet = np.ascontiguousarray(link_iolet, np.uint16)
        tr = np.ascontiguousarray(np.asarray(type_ranges).reshape(-1), np.uint64)
        ios = (L.Iolet * max(len(iolets), 1))(*[i.to_c() for i in iolets])
        h = C.c_void_p()
        _check(lib.splbcu_domain_from_arrays(len(types), _ptr(coords, C.c_int32), _ptr(types, C.c_uint8),
                                             _ptr(link_kind, C.c_uint8), _ptr(link_iolet, C.c_uint16), ios,
                                             len(iolets), _ptr(tr, C.c_uint64), voxel_size, C.byref(h)))
        return SparseDomain(h)


def classify_sites(voxels, iolets: Sequence[Iolet] = (), voxel_size: float = 1.0) -> SparseDomain:
    """classify_sites (geometry.hpp:139-208)."""
    v = np.ascontiguousarray(np.asarray(voxels, dtype=np.int32).reshape(-1, 3))
    ios = (L.Iolet * max(len(iolets), 1))(*[i.to_c() for i in iolets])
    h = C.c_void_p()
    _check(lib.splbcu_domain_classify(_ptr(v, C.c_int32), len(v), ios, len(iolets), voxel_size, C.byref(h)))
    return SparseDomain(h)


def build_pipe(radius: int, length: int, voxel_size: float = 1.0) -> SparseDomain:
    h = C.c_void_p()
    _check(lib.splbcu_domain_build_pipe(radius, length, voxel_size, C.byref(h)))
    return SparseDomain(h)


def build_bifurcation(trunk_radius, branch_radius, trunk_length, branch_length, voxel_size=1.0):
    h = C.c_void_p()
    _check(lib.splbcu_domain_build_bifurcation(trunk_radius, branch_radius, trunk_length, branch_length,
                                               voxel_size, C.byref(h)))
    return SparseDomain(h)


def build_tree(root_radius, root_length, levels, radius_ratio=0.8, length_ratio=0.8, voxel_size=1.0):
    h = C.c_void_p()
    _check(lib.splbcu_domain_build_tree(root_radius, root_length, levels, radius_ratio, length_ratio,
                                        voxel_size, C.byref(h)))
    return SparseDomain(h)


def build_channel(nx, ny, nz, voxel_size=1.0):
    h = C.c_void_p()
    _check(lib.splbcu_domain_build_channel(nx, ny, nz, voxel_size, C.byref(h)))
    return SparseDomain(h)


class Source:
    """A geometry generator evaluated slice by slice (include/splbcu.h,
    "geometry sources").  ``build()`` is the whole domain, identical to the
    matching ``build_*``; ``Simulation.distributed(source, ...)`` builds only
    each rank's slab."""

    def __init__(self, handle):
        self._h = C.c_void_p(handle) if not isinstance(handle, C.c_void_p) else handle

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and h.value:
            lib.splbcu_source_free(h)
            self._h = C.c_void_p(None)

    @property
    def handle(self):
        return self._h

    @staticmethod
    def _make(fn, *args) -> "Source":
        h = C.c_void_p()
        _check(fn(*args, C.byref(h)))
        return Source(h)

    @staticmethod
    def pipe(radius, length, voxel_size=1.0) -> "Source":
        return Source._make(lib.splbcu_source_pipe, radius, length, voxel_size)

    @staticmethod
    def bifurcation(trunk_radius, branch_radius, trunk_length, branch_length, voxel_size=1.0) -> "Source":
        return Source._make(lib.splbcu_source_bifurcation, trunk_radius, branch_radius, trunk_length,
                            branch_length, voxel_size)

    @staticmethod
    def tree(root_radius, root_length, levels, radius_ratio=0.8, length_ratio=0.8, voxel_size=1.0) -> "Source":
        return Source._make(lib.splbcu_source_tree, root_radius, root_length, levels, radius_ratio, length_ratio,
                            voxel_size)

    @staticmethod
    def channel(nx, ny, nz, voxel_size=1.0) -> "Source":
        return Source._make(lib.splbcu_source_channel, nx, ny, nz, voxel_size)

    def build(self) -> "SparseDomain":
        h = C.c_void_p()
        _check(lib.splbcu_source_build(self._h, C.byref(h)))
        return SparseDomain(h)

    def window(self, n_workers: int, worker: int):
        """What rank `worker` builds in slab-local mode: None when the
        partition is not a z-slab split, else a dict with the window domain,
        its global indices, own slice range, global site count and the
        worker's part (site lists index the window)."""
        slab = C.c_int32()
        hd, hp = C.c_void_p(), C.c_void_p()
        _check(lib.splbcu_source_window(self._h, n_workers, worker, C.byref(slab), C.byref(hd), C.byref(hp)))
        if not slab.value:
            return None
        dom = SparseDomain(hd)
        n = dom.n_sites()
        gi = np.zeros(max(n, 1), np.uint64)
        ng, lo, hi = C.c_uint64(), C.c_int32(), C.c_int32()
        _check(lib.splbcu_window_info(hd, C.byref(ng), C.byref(lo), C.byref(hi), _ptr(gi, C.c_uint64)))
        part = PartitionAssignment(hp, n, n_workers)
        return dict(domain=dom, global_index=gi[:n], own=(lo.value, hi.value), n_global=ng.value, part=part)


# ---- decomposition ----------------------------------------------------------------
@dataclass
class WorkerPart:
    sites: np.ndarray
    n_edge: int
    edge_ranges: np.ndarray
    mid_ranges: np.ndarray
    neighbors: List[int]


class PartitionAssignment:
    """decomp.hpp:16-39, copied out of a C handle."""

    def __init__(self, handle, n_sites: int, n_workers: int, owned=True):
        self.n_workers = n_workers
        self.owner = np.zeros(n_sites, np.int32)
        self.local_index = np.zeros(n_sites, np.uint32)
        _check(lib.splbcu_partition_global(handle, _ptr(self.owner, C.c_int32), _ptr(self.local_index, C.c_uint32)))
        self.parts: List[WorkerPart] = []
        for w in range(n_workers):
            ns, ne, nn = C.c_uint32(), C.c_uint32(), C.c_uint32()
            _check(lib.splbcu_partition_part_shape(handle, w, C.byref(ns), C.byref(ne), C.byref(nn)))
            sites = np.zeros(ns.value, np.uint32)
            er = np.zeros(12, np.uint64)
            mr = np.zeros(12, np.uint64)
            nb = np.zeros(max(nn.value, 1), np.int32)
            _check(lib.splbcu_partition_part(handle, w, _ptr(sites, C.c_uint32), _ptr(er, C.c_uint64),
                                             _ptr(mr, C.c_uint64), _ptr(nb, C.c_int32)))
            self.parts.append(WorkerPart(sites, ne.value, er.reshape(6, 2).astype(np.int64),
                                         mr.reshape(6, 2).astype(np.int64), [int(x) for x in nb[:nn.value]]))
        self._imb = float(lib.splbcu_partition_imbalance(handle))
        if owned:
            lib.splbcu_partition_free(handle)

    def load_imbalance_ratio(self) -> float:
        return self._imb


def partition(domain: SparseDomain, n_workers: int) -> PartitionAssignment:
    """partition (decomp.hpp:65-188)."""
    h = C.c_void_p()
    _check(lib.splbcu_partition_create(domain.handle, n_workers, C.byref(h)))
    return PartitionAssignment(h, domain.n_sites(), n_workers)


# ---- simulation ---------------------------------------------------------------------
@dataclass
class StreamingMap:
    """layout.hpp:113-140 in the reference encoding (exported from the device table)."""
    n_local: int
    shared_size: int
    dest: np.ndarray
    op: np.ndarray
    iolet: np.ndarray
    recv_dest: np.ndarray
    send_src_site: np.ndarray
    send_src_dir: np.ndarray
    segments: List[tuple]
    # pull side (GatherSource, layout.hpp:104-108): per slot [site*18 + j-1]
    src_site: np.ndarray = None
    src_op: np.ndarray = None
    src_iolet: np.ndarray = None


@dataclass
class Capture:
    step: int
    fields: np.ndarray


class DistributionStore:
    """Host view of store(w) (layout.hpp:19-62): f_old()/f_new() download,
    set_f_old()/set_f_new() upload, in the reference layout and local order."""

    def __init__(self, sim: "Simulation", w: int):
        self._sim, self._w = sim, w
        n, sh = C.c_uint32(), C.c_uint32()
        _check(lib.splbcu_sim_store_shape(sim._h, w, C.byref(n), C.byref(sh)))
        self.n_sites, self.shared_size = n.value, sh.value
        self.layout = sim.params.layout

    def shared_base(self) -> int:
        return Q * self.n_sites

    def total_size(self) -> int:
        return Q * self.n_sites + self.shared_size

    def idx(self, s: int, i: int) -> int:
        return Q * s + i if self.layout == AOS else i * self.n_sites + s

    def _get(self, which):
        out = np.zeros(self.total_size())
        _check(lib.splbcu_sim_get_f(self._sim._h, self._w, which, _ptr(out, C.c_double)))
        return out

    def _set(self, which, arr):
        a = np.ascontiguousarray(arr, np.float64)
        assert a.size == self.total_size()
        _check(lib.splbcu_sim_set_f(self._sim._h, self._w, which, _ptr(a, C.c_double)))

    def f_old(self) -> np.ndarray:
        return self._get(0)

    def f_new(self) -> np.ndarray:
        return self._get(1)

    def set_f_old(self, a) -> None:
        self._set(0, a)

    def set_f_new(self, a) -> None:
        self._set(1, a)


def _bc_array(bcs: BCSet):
    keep = []
    arr = (L.BC * max(len(bcs.entries), 1))()
    for k, e in enumerate(bcs.entries):
        ts = np.array([n[0] for n in e.table.nodes], np.float64)
        vs = np.array([n[1] for n in e.table.nodes], np.float64)
        keep += [ts, vs]
        arr[k].kind = e.kind
        arr[k].times = _ptr(ts, C.c_double)
        arr[k].values = _ptr(vs, C.c_double)
        arr[k].n_nodes = len(ts)
        arr[k].period = e.table.period
    return arr, keep


def _params_c(p: EngineParams):
    c = L.Params()
    lib.splbcu_params_default(C.byref(c))
    c.tau, c.rho0, c.dt_s = p.tau, p.rho0, p.dt_s
    c.layout, c.scheme, c.sequence, c.workers = p.layout, p.scheme, p.sequence, p.workers
    c.capture_period = p.capture_period
    c.observe_iolets = 1 if p.observe_iolets else 0
    c.exchange_timeout_s = p.exchange_timeout_s
    c.halo_mode = p.halo_mode
    c.storage = p.storage
    devs = None
    if p.devices:
        devs = np.array(p.devices, np.int32)
        c.n_devices = len(devs)
        c.device_ids = _ptr(devs, C.c_int32)
    return c, devs


class Simulation:
    """splb::Simulation (engine.hpp:121-205) on B200 workers.

    ``Simulation(domain, bcs, params)`` places params.workers workers on
    params.devices (round robin).  ``Simulation.distributed(...)`` builds the
    one-process-per-GPU variant whose halo exchange is NCCL send/recv.
    """

    def __init__(self, domain: SparseDomain, bcs: BCSet, params: EngineParams, _dist=None):
        self.domain_ = domain
        self.params = params
        self._n_io = len(bcs.entries)
        arr, keep = _bc_array(bcs)
        pc, devs = _params_c(params)
        h = C.c_void_p()
        if _dist is None:
            _check(lib.splbcu_sim_create(domain.handle, arr, len(bcs.entries), C.byref(pc), C.byref(h)))
        else:
            rank, nranks, uid = _dist
            idb = (C.c_uint8 * 128).from_buffer_copy(bytes(uid))
            create = lib.splbcu_sim_create_dist_source if isinstance(domain, Source) else lib.splbcu_sim_create_dist
            _check(create(domain.handle, arr, len(bcs.entries), C.byref(pc), rank, nranks, idb, C.byref(h)))
        self._h = h
        del keep, devs
        self._part = None

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        _check(lib.splbcu_nccl_unique_id(buf))
        return bytes(buf)

    @classmethod
    def distributed(cls, domain, bcs, params, rank: int, nranks: int, uid: bytes) -> "Simulation":
        """One process per GPU.  `domain` may be a SparseDomain (every rank
        holds all of it) or a Source (slab-local construction)."""
        return cls(domain, bcs, params, _dist=(rank, nranks, uid))

    def slab_local(self) -> bool:
        return bool(lib.splbcu_sim_slab_local(self._h))

    def n_sites(self) -> int:
        """Sites of the whole domain."""
        return int(lib.splbcu_sim_n_sites(self._h))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and h.value:
            lib.splbcu_sim_destroy(h)
            self._h = C.c_void_p(None)

    def close(self):
        self.__del__()

    def domain(self) -> SparseDomain:
        return self.domain_

    def run(self, n_steps: int) -> None:
        _check(lib.splbcu_sim_run(self._h, n_steps))

    def steps_run(self) -> int:
        return int(lib.splbcu_sim_steps_run(self._h))

    def step_loop_seconds(self) -> float:
        return float(lib.splbcu_sim_step_loop_seconds(self._h))

    def device_loop_seconds(self) -> float:
        return float(lib.splbcu_sim_device_loop_seconds(self._h))

    def set_kernel_timing(self, on: bool) -> None:
        _check(lib.splbcu_sim_set_kernel_timing(self._h, 1 if on else 0))

    def kernel_stats(self):
        s, n, sites = C.c_double(), C.c_uint64(), C.c_uint64()
        _check(lib.splbcu_sim_kernel_stats(self._h, C.byref(s), C.byref(n), C.byref(sites)))
        return s.value, n.value, sites.value

    def write_snapshots(self, path: str) -> None:
        """write_snapshots (snapshot.hpp:15-29): snapshots.bin."""
        _check(lib.splbcu_sim_write_snapshots(self._h, path.encode()))

    def series_csv(self, dt_s: float) -> str:
        """series_csv (snapshot.hpp:59-82): timeseries.csv text."""
        n = C.c_size_t()
        _check(lib.splbcu_sim_series_csv(self._h, dt_s, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        _check(lib.splbcu_sim_series_csv(self._h, dt_s, buf, n.value + 1, C.byref(n)))
        return buf.value.decode()

    def launch_count(self) -> int:
        return int(lib.splbcu_sim_launch_count(self._h))

    def bulk_kernel(self) -> int:
        """0: just-in-time table kernel, 1: prefetch kernel, -1: other."""
        return int(lib.splbcu_sim_bulk_kernel(self._h))

    def series_d2h_bytes(self) -> int:
        return int(lib.splbcu_sim_series_d2h_bytes(self._h))

    def snapshot_fields(self) -> np.ndarray:
        out = np.zeros(4 * self.n_sites())
        _check(lib.splbcu_sim_snapshot(self._h, _ptr(out, C.c_double)))
        return out

    def store(self, w: int) -> DistributionStore:
        return DistributionStore(self, w)

    def is_local(self, w: int) -> bool:
        return bool(lib.splbcu_sim_worker_is_local(self._h, w))

    def assignment(self) -> PartitionAssignment:
        if self._part is None:
            h = lib.splbcu_sim_partition(self._h)
            if not h:
                raise Error("assignment(): not held by a slab-local simulation")
            self._part = PartitionAssignment(C.c_void_p(h), self.n_sites(), self.params.workers, owned=False)
        return self._part

    def map(self, w: int) -> StreamingMap:
        n, sh, ns = C.c_uint32(), C.c_uint32(), C.c_uint32()
        _check(lib.splbcu_sim_map_shape(self._h, w, C.byref(n), C.byref(sh), C.byref(ns)))
        n, sh, ns = n.value, sh.value, ns.value
        dest = np.zeros(18 * n, np.uint32)
        op = np.zeros(18 * n, np.uint8)
        io = np.zeros(18 * n, np.uint16)
        rd = np.zeros(max(sh, 1), np.uint32)
        ss = np.zeros(max(sh, 1), np.uint32)
        sd = np.zeros(max(sh, 1), np.uint8)
        sn = np.zeros(max(ns, 1), np.int32)
        sb = np.zeros(max(ns, 1), np.uint32)
        sc = np.zeros(max(ns, 1), np.uint32)
        _check(lib.splbcu_sim_export_map(self._h, w, _ptr(dest, C.c_uint32), _ptr(op, C.c_uint8),
                                         _ptr(io, C.c_uint16), _ptr(rd, C.c_uint32), _ptr(ss, C.c_uint32),
                                         _ptr(sd, C.c_uint8), _ptr(sn, C.c_int32), _ptr(sb, C.c_uint32),
                                         _ptr(sc, C.c_uint32)))
        gs = np.zeros(18 * n, np.uint32)
        go = np.zeros(18 * n, np.uint8)
        gi = np.zeros(18 * n, np.uint16)
        _check(lib.splbcu_sim_export_sources(self._h, w, _ptr(gs, C.c_uint32), _ptr(go, C.c_uint8),
                                             _ptr(gi, C.c_uint16)))
        return StreamingMap(n, sh, dest, op, io, rd[:sh], ss[:sh], sd[:sh],
                            [(int(sn[k]), int(sb[k]), int(sc[k])) for k in range(ns)], gs, go, gi)

    def cache(self) -> List[Capture]:
        out = []
        n = self.n_sites()
        for k in range(int(lib.splbcu_sim_n_captures(self._h))):
            st = C.c_uint64()
            f = np.zeros(4 * n)
            _check(lib.splbcu_sim_capture(self._h, k, C.byref(st), _ptr(f, C.c_double)))
            out.append(Capture(int(st.value), f))
        return out

    def series(self):
        rows = int(lib.splbcu_sim_series_rows(self._h))
        nio = self._n_io  # one BC entry per iolet (validated at construction)
        res = dict(rows=rows, max_speed=[], pressure=[], flow=[])
        if rows == 0:
            return res
        for k in range(nio):
            a, b, c = np.zeros(rows), np.zeros(rows), np.zeros(rows)
            _check(lib.splbcu_sim_series(self._h, k, _ptr(a, C.c_double), _ptr(b, C.c_double),
                                         _ptr(c, C.c_double)))
            res["max_speed"].append(a)
            res["pressure"].append(b)
            res["flow"].append(c)
        return res


def compute_metrics(n_fluid_sites: int, n_time_steps: int, sim_time_s: float, n_workers: int) -> dict:
    """compute_metrics (bench.hpp:170-188): MLUPS = n*steps/(T*1e6)."""
    if not sim_time_s > 0.0:
        raise Error(f"compute_metrics: SimTime must be positive, got {sim_time_s}")
    mlups = float(n_fluid_sites) * float(n_time_steps) / (sim_time_s * 1e6)
    return dict(mlups=mlups, mlups_pc=mlups / n_workers, mlups_pn=mlups / n_workers)
