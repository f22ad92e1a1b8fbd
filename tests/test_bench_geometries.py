"""The bench's own geometries against the live reference engine (GPU).

bench.py reports MSUPS on C3 (bifurcating tree, 65 pressure iolets), C2 (the
1e7-site pulsatile pipe), C4 (dense channel) and C5 (7-level tree, 129
iolets).  Here the same generators run through the product and through the
unmodified reference (oracle/_ref: its own classify_sites on the voxels of
oracle/geometry_gen.py, its own Simulation), from a perturbed start, with
captures and the iolet series on, and every field is compared bit for bit —
the reference's own cross-engine check (proj/tools/splb.cpp:142-203) and its
variant suite (proj/tests/test_engine.cpp:218-267).

C3/C4/C5 run at reduced size (the oracle holds ~830 B/site); C2 runs at full
size (build_pipe(48, 1400), 10,130,400 sites).  The product runs the bench
configuration (one worker, two buffers) plus the multi-slab, fused-P2P and
AA single-buffer modes on the same inputs.
"""
import os

import numpy as np
import pytest

import cases
import geometry_gen as G

pytestmark = pytest.mark.gpu

CS2 = cases.CS2


def _tree_bcs(M, n_iolets):
    ents = [M.BCEntry(M.PRESSURE, M.TimeTable.constant(CS2 * 1.001))]
    ents += [M.BCEntry(M.PRESSURE, M.TimeTable.constant(CS2 * 0.999)) for _ in range(n_iolets - 1)]
    return M.BCSet(ents)


def _digest(M, d, bcs, prm, steps, noise):
    sim = M.Simulation(d, bcs, prm)
    cases.apply_noise(M, sim, noise)
    sim.run(steps // 3)
    sim.run(steps - steps // 3)
    out = dict(snapshot=cases.h(sim.snapshot_fields()),
               captures=[(c.step, cases.h(c.fields)) for c in sim.cache()],
               series={k: [cases.h(a) for a in v] for k, v in sim.series().items() if k != "rows"},
               rows=sim.series()["rows"])
    sim.close() if hasattr(sim, "close") else None
    return out


def _cores():
    return max(1, min(32, os.cpu_count() or 1))


def _compare(product, reference, kind, args, steps, tau=0.8, seed=20240808, amp=0.01, modes=None):
    vox, io = getattr(G, kind)(*args)
    dr = G.classify(reference, vox, io)
    dp = getattr(product, "build_" + kind)(*args)
    assert cases.domain_digest(dp) == cases.domain_digest(dr)
    noise = cases.noise_for(dp.n_sites(), seed, amp)
    kw = dict(tau=tau, dt_s=1.0, capture_period=steps // 2, observe_iolets=True)
    want = _digest(reference, dr, _tree_bcs(reference, len(io)),
                   reference.EngineParams(workers=_cores(), layout=reference.SOA, **kw), steps, noise)
    for name, extra in (modes or {"bench (1 worker)": {}}).items():
        got = _digest(product, dp, _tree_bcs(product, len(io)), product.EngineParams(devices=[0], **kw, **extra),
                      steps, noise)
        assert got == want, name
    return dp.n_sites(), len(io)


MODES = {"bench (1 worker)": {}, "4 slabs, NCCL-style tail": dict(workers=4),
         "4 slabs, fused P2P": dict(workers=4, halo_mode=1), "AA single buffer, 3 slabs": dict(workers=3, storage=1)}


def test_c3_tree_sample_vs_reference(product, reference):
    """C3-shaped: the bench tree generator with 6 levels (65 pressure
    iolets, u16 iolet ids, 65 staged values per step, series over 65
    iolets), 60 steps from a perturbed start."""
    n, nio = _compare(product, reference, "tree", (16, 80, 6, 0.8, 0.8), 60, modes=MODES)
    assert nio == 65 and n > 2e5


def test_c5_tree_sample_vs_reference(product, reference):
    """C5-shaped: 7 levels, 129 pressure iolets."""
    n, nio = _compare(product, reference, "tree", (10, 60, 7, 0.8, 0.8), 40,
                      modes={"bench (1 worker)": {}, "3 slabs, fused P2P": dict(workers=3, halo_mode=1)})
    assert nio == 129


def test_c4_channel_sample_vs_reference(product, reference):
    """C4-shaped: dense channel, iolet discs covering the cross-section
    (classifier margin, geometry.hpp:76-78, 102-113)."""
    _compare(product, reference, "channel", (48, 40, 120), 60, modes=MODES)


@pytest.mark.slow
def test_c2_full_size_vs_reference(product, reference):
    """C2 at full size: build_pipe(48, 1400) = 10,130,400 sites, 60-bpm
    velocity inlet (pipe_beat.cfg), outlet p = 1/3, tau 0.8, dt 5e-4 s; the
    reference on the host's cores.  60 steps with the series on, plus
    a mid-run capture."""
    beat = cases.TABLES["beat"]

    def run(M, prm):
        d = M.build_pipe(48, 1400)
        bcs = M.BCSet([M.BCEntry(M.VELOCITY, M.TimeTable(*beat)), M.BCEntry(M.PRESSURE, M.TimeTable.constant(CS2))])
        sim = M.Simulation(d, bcs, prm)
        sim.run(20)
        sim.run(40)
        return d.n_sites(), dict(snapshot=cases.h(sim.snapshot_fields()),
                                 captures=[(c.step, cases.h(c.fields)) for c in sim.cache()],
                                 series={k: [cases.h(a) for a in v] for k, v in sim.series().items() if k != "rows"})

    kw = dict(tau=0.8, dt_s=5e-4, capture_period=30, observe_iolets=True)
    n, want = run(reference, reference.EngineParams(workers=_cores(), layout=reference.SOA, **kw))
    assert n == 10130400
    _, got = run(product, product.EngineParams(devices=[0], **kw))
    assert got == want
