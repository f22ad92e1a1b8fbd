"""The CPU oracle (oracle/liboracle.so, a plain-C restatement) pinned
against the golden vectors produced by the unmodified reference, and —
when oracle/_ref is built — against the reference live."""
import numpy as np
import pytest

import cases

FAST_RUNS = [k for k in cases.RUNS if k not in ("C1_pipe_16_128",)]


def test_kat_equilibrium(port, golden):
    assert port.equilibrium(1.0, [0, 0, 0]).tolist() == golden["kat"]["eq_rest"]
    eq = port.equilibrium(1.0, [0.1, 0.0, 0.0])
    assert eq.tolist() == golden["kat"]["eq_01"]
    assert abs(eq[1] - 133.0 / 1800.0) <= 1e-14 * 133.0 / 1800.0  # test_lattice.cpp:95-102


def test_kat_collide_moments(port, golden_arrays):
    F = golden_arrays["kat_f"]
    got = np.stack([port.bgk_collide(f, 0.8) for f in F])
    assert np.array_equal(got, golden_arrays["kat_collide_08"])
    mom = np.stack([np.r_[port.moments(f)[0], port.moments(f)[1]] for f in F])
    assert np.array_equal(mom, golden_arrays["kat_moments"])
    eq = np.stack([port.equilibrium(r[0], r[1:]) for r in golden_arrays["kat_eq_in"]])
    assert np.array_equal(eq, golden_arrays["kat_eq"])


def test_kat_tables_weights(port, golden):
    for name, tab in cases.TABLES.items():
        ts = np.linspace(-0.3, 2.7, 61)
        assert [port.TimeTable(tab[0], tab[1]).at(float(t)) for t in ts] == golden["kat"]["tables"][name]
    io = port.Iolet(0, [0.375, 0.5, -0.5], [0.0, 0.0, 1.0], 8.0)
    assert [port.iolet_weight(io, c) for c in cases.WEIGHT_COORDS] == golden["kat"]["weights"]
    # test_boundary.cpp:27-41: axis weight 1, clamped 0 outside
    assert port.iolet_weight(io, (0, 0, 0)) <= 1.0


@pytest.mark.parametrize("name", sorted(cases.DOMAINS))
def test_domains(port, golden, name):
    d = cases.make_domain(port, cases.DOMAINS[name])
    assert cases.domain_digest(d) == golden["domains"][name]


@pytest.mark.parametrize("key", sorted(k for k in cases.PARTITION_WORKERS for _ in [0]))
def test_partitions(port, golden, key):
    d = cases.make_domain(port, cases.DOMAINS[key])
    for W in cases.PARTITION_WORKERS[key]:
        assert cases.partition_digest(port.partition(d, W)) == golden["partitions"][f"{key}/W{W}"]


@pytest.mark.parametrize("key", sorted(cases.MAP_CASES))
def test_maps(port, golden, key):
    run = cases.MAP_CASES[key]
    d = cases.make_domain(port, cases.DOMAINS[run["domain"]])
    s = port.Simulation(d, cases.make_bcs(port, run["bcs"]), port.EngineParams(workers=run["W"], layout=run["layout"]))
    assert [cases.map_digest(s.map(w)) for w in range(run["W"])] == golden["maps"][key]


@pytest.mark.parametrize("key", FAST_RUNS)
def test_runs(port, golden, key):
    res = cases.execute_run(port, cases.RUNS[key])
    assert cases.run_digest(res) == golden["runs"][key]


def test_closed_box_mass(port, golden):
    m0, m1 = golden["runs"]["box8_noise_W2_1000"]["mass"]
    assert abs(m1 - m0) <= 1e-12 * m0  # test_engine.cpp:121-138


def test_live_reference_agrees(port, reference):
    """Oracle vs the reference itself on a fresh seeded case not in the
    golden set (bifurcation, 3 workers, SoA, perturbed)."""
    run = dict(domain="bif_3_2_6_8", bcs=("bif", "bif_inlet"), tau=0.7, dt=2e-3, W=3, layout=1, steps=30,
               capture=10, observe=True, noise=(7, 0.01))
    a = cases.execute_run(port, run)
    b = cases.execute_run(reference, run)
    assert cases.run_digest(a) == cases.run_digest(b)


def test_errors_match_reference(port, reference):
    for M in (port, reference):
        with pytest.raises(M.GeometryError, match="empty voxel set"):
            M.classify_sites(np.zeros((0, 3), np.int32), [])
        with pytest.raises(M.GeometryError, match="duplicate voxel"):
            M.classify_sites([[0, 0, 0], [1, 0, 0], [0, 0, 0]], [])
        d = M.build_pipe(3, 8)
        with pytest.raises(M.ConfigError, match="configured for 1 iolets"):
            M.Simulation(d, M.BCSet([M.BCEntry(M.PRESSURE, M.TimeTable.constant(cases.CS2))]), M.EngineParams())
        with pytest.raises(M.Error, match="exceeds site count"):
            M.partition(M.classify_sites(cases.closed_box(2), []), 9)


def test_output_files_match_reference(port, reference, tmp_path):
    """snapshots.bin and timeseries.csv (snapshot.hpp:15-82) byte-identical."""
    outs = []
    for M in (port, reference):
        run = dict(domain="pipe_3_8", bcs=("pressure", 0.34, cases.CS2), tau=0.8, dt=1e-3, W=2, steps=25,
                   capture=10, observe=True)
        res = cases.execute_run(M, run)
        p = str(tmp_path / f"{M.__name__}.bin")
        res["sim"].write_snapshots(p)
        outs.append((open(p, "rb").read(), res["sim"].series_csv(1e-3)))
    assert outs[0] == outs[1]
    assert outs[0][1].count("\n") == 27 and "iolet1_flow" in outs[0][1]
