"""Parity cases shared by tests/golden/make_golden.py and the tests.

Each helper takes a mirror module M (tests/impls.py: product, port or
reference) so the same case runs identically on every implementation.
Cases follow the reference's own tests (proj/tests/*.cpp) and configs.
"""
from __future__ import annotations

import numpy as np

CS2 = 1.0 / 3.0

# BC tables: bifurcation inlet (test_engine.cpp:30-38), 60-bpm beat
# (proj/configs/pipe_beat.cfg:15), smoke inlet (bifurcation_smoke.cfg:14).
TABLES = {
    "bif_inlet": ([(0.0, 0.01), (0.25, 0.04), (0.5, 0.02), (0.75, 0.015)], 1.0),
    "beat": ([(0.0, 0.008), (0.05, 0.012), (0.1, 0.024), (0.15, 0.036), (0.2, 0.04), (0.25, 0.036),
              (0.3, 0.026), (0.35, 0.016), (0.4, 0.01), (0.5, 0.007), (0.6, 0.006), (0.75, 0.0055),
              (0.9, 0.006)], 1.0),
    "smoke_inlet": ([(0.0, 0.01), (0.25, 0.04), (0.5, 0.02), (0.75, 0.012)], 1.0),
    "ramp": ([(0.0, 0.0), (1.0, 0.05)], 0.0),
}
WEIGHT_COORDS = [(0, 0, 0), (0, 1, 0), (5, 0, 3), (8, 0, 0), (-8, 0, 1), (3, 4, 0), (9, 9, 9)]

# dt from proj/configs/pipe_beat.cfg via config.hpp:42-46
DT_BEAT = CS2 * (0.8 - 0.5) * 0.001 * 0.001 / 0.0002


def closed_box(n):
    """test_engine.cpp:15-21"""
    z, y, x = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    return np.stack([x.ravel(), y.ravel(), z.ravel()], 1).astype(np.int32)


def random_blob(seed, size=180):
    """Connected voxel blob grown by a random walk (test_engine.cpp:317-332),
    emitted in std::set order (lexicographic (x,y,z))."""
    rng = np.random.default_rng(seed)
    vel = [(1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1)]
    pos = (0, 0, 0)
    blob = {pos}
    while len(blob) < size:
        c = vel[int(rng.integers(0, 6))]
        pos = (pos[0] + c[0], pos[1] + c[1], pos[2] + c[2])
        blob.add(pos)
    return np.array(sorted(blob), dtype=np.int32)


DOMAINS = {
    "box6": ("voxels", "box", 6),
    "box8": ("voxels", "box", 8),
    "box9": ("voxels", "box", 9),
    "pipe_2_4": ("pipe", 2, 4),
    "pipe_3_8": ("pipe", 3, 8),
    "pipe_3_12": ("pipe", 3, 12),
    "pipe_4_20": ("pipe", 4, 20),
    "pipe_8_64": ("pipe", 8, 64),
    "pipe_16_128": ("pipe", 16, 128),
    "bif_3_2_6_8": ("bif", 3, 2, 6, 8),
    "bif_4_3_12_12": ("bif", 4, 3, 12, 12),
    "blob0": ("voxels", "blob", 20240808),
    "blob1": ("voxels", "blob", 20240809),
}

PARTITION_WORKERS = {
    "box8": [1, 2, 3, 8],
    "pipe_3_8": [1, 2, 3],
    "pipe_3_12": [1, 3],
    "pipe_4_20": [1, 4, 7],
    "pipe_16_128": [1, 2, 4, 8],
    "bif_3_2_6_8": [1, 2, 3, 4, 5, 23],
    "bif_4_3_12_12": [1, 2, 3, 8],
    "blob0": [1, 5, 23, 180],
    "blob1": [1, 5, 23],
}


def make_domain(M, spec):
    kind = spec[0]
    if kind == "pipe":
        return M.build_pipe(spec[1], spec[2])
    if kind == "bif":
        return M.build_bifurcation(*spec[1:])
    if spec[1] == "box":
        return M.classify_sites(closed_box(spec[2]), [])
    return M.classify_sites(random_blob(spec[2]), [])


def make_bcs(M, name):
    if name is None:
        return M.BCSet([])
    kind, args = name[0], name[1:]
    if kind == "pressure":
        return M.BCSet([M.BCEntry(M.PRESSURE, M.TimeTable.constant(v)) for v in args])
    if kind == "bif":
        t, p = TABLES[args[0]]
        return M.BCSet([M.BCEntry(M.VELOCITY, M.TimeTable(t, p)),
                        M.BCEntry(M.PRESSURE, M.TimeTable.constant(CS2)),
                        M.BCEntry(M.PRESSURE, M.TimeTable.constant(CS2))])
    if kind == "beat":
        t, p = TABLES["beat"]
        return M.BCSet([M.BCEntry(M.VELOCITY, M.TimeTable(t, p)), M.BCEntry(M.PRESSURE, M.TimeTable.constant(CS2))])
    if kind == "velocity_const":
        return M.BCSet([M.BCEntry(M.VELOCITY, M.TimeTable.constant(args[0])),
                        M.BCEntry(M.PRESSURE, M.TimeTable.constant(CS2))])
    raise ValueError(name)


def _c1_dp():
    # acceptance.cpp:196-205, k = 1 (R=16, Len=128)
    tau = 0.9
    eta = CS2 * (tau - 0.5)
    R, Len, umax = 16, 128, 0.04 / 2
    return umax * 4.0 * eta * Len / (float(R) * R)


C1_DP = _c1_dp()

MAP_CASES = {
    "pipe_3_8/W1/aos": dict(domain="pipe_3_8", bcs=("pressure", CS2, CS2), W=1, layout=0),
    "pipe_3_8/W2/soa": dict(domain="pipe_3_8", bcs=("pressure", CS2, CS2), W=2, layout=1),
    "pipe_3_12/W3/aos": dict(domain="pipe_3_12", bcs=("pressure", CS2, CS2), W=3, layout=0),
    "bif_3_2_6_8/W1/aos": dict(domain="bif_3_2_6_8", bcs=("bif", "bif_inlet"), W=1, layout=0),
    "bif_3_2_6_8/W3/aos": dict(domain="bif_3_2_6_8", bcs=("bif", "bif_inlet"), W=3, layout=0),
    "bif_3_2_6_8/W3/soa": dict(domain="bif_3_2_6_8", bcs=("bif", "bif_inlet"), W=3, layout=1),
    "blob0/W5/soa": dict(domain="blob0", bcs=None, W=5, layout=1),
    "blob1/W23/aos": dict(domain="blob1", bcs=None, W=23, layout=0),
    "pipe_16_128/W4/soa": dict(domain="pipe_16_128", bcs=("pressure", CS2, CS2), W=4, layout=1),
}

# Runs: perturbation = ("noise", seed, amplitude) added to every f_old entry
# in (global site, direction) order before the first step.
RUNS = {
    "box8_noise_W2_1000": dict(domain="box8", bcs=None, tau=0.8, W=2, steps=1000, noise=(99, 0.05)),
    "bif_W1_aos": dict(domain="bif_3_2_6_8", bcs=("bif", "bif_inlet"), tau=0.8, dt=1e-3, W=1, steps=24,
                       capture=8, observe=True),
    "bif_W3_soa_reordered": dict(domain="bif_3_2_6_8", bcs=("bif", "bif_inlet"), tau=0.8, dt=1e-3, W=3,
                                 layout=1, sequence=1, steps=24, capture=8, observe=True),
    "bif_W4_noise": dict(domain="bif_3_2_6_8", bcs=("bif", "bif_inlet"), tau=0.8, dt=1e-3, W=4, steps=12,
                         noise=(4242, 0.02), capture=4),
    "bif4_cross_engine": dict(domain="bif_4_3_12_12", bcs=("bif", "smoke_inlet"), tau=0.8, dt=1e-3, W=1,
                              steps=120, capture=10),
    "pipe_4_20_W4": dict(domain="pipe_4_20", bcs=("pressure", 0.3383333333333333, CS2), tau=0.8, dt=1e-3,
                         W=4, steps=100, capture=50),
    "pipe_3_8_obs_W2": dict(domain="pipe_3_8", bcs=("pressure", 0.34, CS2), tau=0.8, dt=1e-3, W=2, steps=25,
                            observe=True),
    "blob0_noise_W5": dict(domain="blob0", bcs=None, tau=0.8, W=5, layout=1, steps=12, noise=(1000, 0.03)),
    "blob1_noise_W23": dict(domain="blob1", bcs=None, tau=0.8, W=23, steps=12, noise=(1001, 0.03)),
    "pipe_beat_6_30": dict(domain="pipe_6_30", bcs=("beat",), tau=0.8, dt=DT_BEAT, W=2, steps=400, capture=200,
                           observe=True),
    "C1_pipe_16_128": dict(domain="pipe_16_128", bcs=("pressure", CS2 + C1_DP / 2, CS2 - C1_DP / 2), tau=0.9,
                           W=1, steps=1000),
}
DOMAINS["pipe_6_30"] = ("pipe", 6, 30)


def noise_for(n_sites, seed, amp):
    rng = np.random.default_rng(seed)
    return rng.uniform(0.0, amp, size=(n_sites, 19))


def apply_noise(M, sim, noise, pa=None):
    """Adds noise[g, i] to f_old of global site g, direction i, on every
    worker the simulation holds (reference layout / local order).  `pa`
    (parts[w].sites = global indices) defaults to sim.assignment()."""
    pa = pa or sim.assignment()
    for w in range(pa.n_workers):
        if not sim.is_local(w):
            continue
        st = sim.store(w)
        f = st.f_old()
        sites = pa.parts[w].sites.astype(np.int64)
        n = len(sites)
        if st.layout == M.AOS:
            f[:19 * n].reshape(n, 19)[:] += noise[sites]
        else:
            f[:19 * n].reshape(19, n)[:] += noise[sites].T
        st.set_f_old(f)


def total_mass(M, sim):
    m = 0.0
    pa = sim.assignment()
    for w in range(pa.n_workers):
        st = sim.store(w)
        f = st.f_old()
        n = st.n_sites
        # the reference sums site-major then direction (test_engine.cpp:40-45)
        arr = f[:19 * n].reshape(n, 19) if st.layout == M.AOS else f[:19 * n].reshape(19, n).T
        for v in arr.ravel():
            m += float(v)
    return m


def execute_run(M, run, devices=None, halo_mode=None, storage=None):
    d = make_domain(M, DOMAINS[run["domain"]])
    p = M.EngineParams(tau=run.get("tau", 0.9), dt_s=run.get("dt", 1.0), workers=run["W"],
                       layout=run.get("layout", 0), sequence=run.get("sequence", 0), scheme=run.get("scheme", 0),
                       capture_period=run.get("capture", 0), observe_iolets=run.get("observe", False))
    if devices is not None:
        p.devices = devices
    if halo_mode is not None:
        p.halo_mode = halo_mode
    if storage is not None:
        p.storage = storage
    sim = M.Simulation(d, make_bcs(M, run["bcs"]), p)
    if "noise" in run:
        apply_noise(M, sim, noise_for(d.n_sites(), *run["noise"]))
    m0 = total_mass(M, sim) if run["domain"].startswith("box") else None
    sim.run(run["steps"])
    m1 = total_mass(M, sim) if m0 is not None else None
    return dict(snapshot=sim.snapshot_fields(), captures=sim.cache(), series=sim.series(),
                mass=[m0, m1], sim=sim, domain=d)


def h(a) -> str:
    """sha256 of an array; floats canonicalised with `a + 0.0` (-0 == +0)."""
    import hashlib
    a = np.ascontiguousarray(a)
    if a.dtype.kind == "f":
        a = a + 0.0
    return hashlib.sha256(a.tobytes()).hexdigest()


def domain_digest(d):
    e = d.export()
    return dict(n=int(d.n_sites()), coords=h(e["coords"]), types=h(e["types"]), link_kind=h(e["link_kind"]),
                link_iolet=h(np.where(e["link_kind"] >= 2, e["link_iolet"], 0).astype(np.uint16)),
                type_ranges=e["type_ranges"].ravel().tolist())


def partition_digest(p):
    return dict(owner=h(p.owner), local_index=h(p.local_index),
                parts=[dict(sites=h(w.sites), n_edge=int(w.n_edge), edge=w.edge_ranges.ravel().tolist(),
                            mid=w.mid_ranges.ravel().tolist(), nb=list(w.neighbors)) for w in p.parts],
                imbalance=p.load_imbalance_ratio())


def map_digest(m):
    return dict(n_local=m.n_local, shared=m.shared_size, dest=h(m.dest), op=h(m.op),
                iolet=h(np.where(m.op == 3, m.iolet, 0).astype(np.uint16)), recv_dest=h(m.recv_dest),
                send_site=h(m.send_src_site), send_dir=h(m.send_src_dir), segments=[list(s) for s in m.segments],
                sources=dict(site=h(m.src_site), op=h(m.src_op),
                             iolet=h(np.where(m.src_op == 3, m.src_iolet, 0).astype(np.uint16))))


def run_digest(res):
    return dict(snapshot=h(res["snapshot"]), captures=[[c.step, h(c.fields)] for c in res["captures"]],
                series={k: [h(a) for a in v] for k, v in res["series"].items() if k != "rows"},
                rows=res["series"].get("rows", 0), mass=res["mass"])
