"""BASELINE's full sizes, through size-independent properties (GPU).

The CPU oracle cannot run C2/C3 at full size in test time (and C3 does not
fit its memory), so at full size the checks are the reference's
own invariances (test_engine.cpp:218-267, 302-368): results are bitwise
independent of the kernel variant that computes them and of the number of
workers the domain is split into.  The kernels themselves are pinned to the
reference bit for bit on the golden runs (test_gpu_parity.py).
"""
import os

import numpy as np
import pytest

import cases

pytestmark = pytest.mark.gpu

CS2 = 1.0 / 3.0
BEAT = ([(0.0, 0.008), (0.05, 0.012), (0.1, 0.024), (0.15, 0.036), (0.2, 0.04), (0.25, 0.036), (0.3, 0.026),
         (0.35, 0.016), (0.4, 0.01), (0.5, 0.007), (0.6, 0.006), (0.75, 0.0055), (0.9, 0.006)], 1.0)


def _run(P, d, bcs, prm, steps, variant=None, noise=None):
    old = os.environ.get("SPLBCU_PLAIN_VARIANT")
    if variant is not None:
        os.environ["SPLBCU_PLAIN_VARIANT"] = variant
    try:
        sim = P.Simulation(d, bcs, prm)
    finally:
        if variant is not None:
            if old is None:
                del os.environ["SPLBCU_PLAIN_VARIANT"]
            else:
                os.environ["SPLBCU_PLAIN_VARIANT"] = old
    if noise is not None:
        cases.apply_noise(P, sim, noise)
    sim.run(steps // 2)
    sim.run(steps - steps // 2)
    snap = sim.snapshot_fields()
    ser = sim.series() if prm.observe_iolets else {}
    out = (cases.h(snap), {k: [cases.h(a) for a in v] for k, v in ser.items() if k != "rows"})
    rho = snap[0::4]
    stats = (float(rho.min()), float(rho.max()), bool(np.isfinite(snap).all()))
    sim.close()
    return out, stats


def test_c2_full_size_kernels_and_workers_agree(product):
    """C2 (build_pipe(48, 1400), 10,130,400 sites, 60-bpm velocity inlet) with
    a perturbed start: the default kernel, the prefetch and u32-table kernels
    and a 3-worker split give the same bits after 200 steps, series included."""
    P = product
    d = P.build_pipe(48, 1400)
    assert d.n_sites() == 10130400
    bcs = P.BCSet([P.BCEntry(P.VELOCITY, P.TimeTable(*BEAT)), P.BCEntry(P.PRESSURE, P.TimeTable.constant(CS2))])
    noise = cases.noise_for(d.n_sites(), 20240808, 0.01)
    runs = {}
    for name, variant, workers in (("default", None, 1), ("prefetch", "59", 1), ("u32", "24", 1),
                                   ("runs", "71", 1), ("w3", None, 3)):
        prm = P.EngineParams(tau=0.8, dt_s=5e-4, workers=workers, devices=[0], observe_iolets=True)
        runs[name] = _run(P, d, bcs, prm, 200, variant, noise)
    want = runs["default"][0]
    for name, (got, stats) in runs.items():
        assert got == want, name
        assert stats[2] and 0.9 < stats[0] <= stats[1] < 1.2, (name, stats)


def test_c3_full_size_kernels_and_workers_agree(product):
    """C3 (1.07e8-site tree, 65 pressure iolets): the default (online choice),
    the just-in-time and prefetch compressed-table kernels, the u32-table
    kernel and a 2-worker split give the same bits after 40 steps (the
    compressed table is pinned to the reference on C3-shaped samples in
    test_bench_geometries.py)."""
    P = product
    d = P.build_tree(80, 800, 6, 0.8, 0.8)
    assert d.n_sites() == 107037564
    ents = [P.BCEntry(P.PRESSURE, P.TimeTable.constant(CS2 * 1.001))]
    ents += [P.BCEntry(P.PRESSURE, P.TimeTable.constant(CS2 * 0.999)) for _ in range(64)]
    bcs = P.BCSet(ents)
    runs = {}
    for name, variant, workers in (("default", None, 1), ("jit", "43", 1), ("prefetch", "59", 1), ("u32", "24", 1),
                                   ("runs", "71", 1), ("w2", None, 2)):
        prm = P.EngineParams(tau=0.8, dt_s=1.0, workers=workers, devices=[0])
        runs[name] = _run(P, d, bcs, prm, 40, variant)
    want = runs["default"][0]
    for name, (got, stats) in runs.items():
        assert got == want, name
        assert stats[2] and 0.99 < stats[0] <= stats[1] < 1.01, (name, stats)
