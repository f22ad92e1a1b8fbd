"""Parity of the B200 engine (sm_100a kernels, device-built tables) with the
reference, through the C-ABI.  Bar: bit-exact tables/decomposition and
bit-exact f/rho/u (== semantics: -0.0 == +0.0) — the engine compiles with
--fmad=false and restates the reference's expression trees, so the FP64
tolerance stated in BASELINE (1e-12 relative) is not needed; the tests
assert equality and would report the max deviation if it ever appeared."""
import numpy as np
import pytest

import cases

pytestmark = pytest.mark.gpu

FAST_RUNS = [k for k in cases.RUNS]


def _skip_unbuilt(P):
    """Tuning variants (measured slower than the defaults) are compiled only
    with `make TUNING=1`; the default build refuses them with a ConfigError."""
    try:
        P.Simulation(P.build_pipe(2, 4), P.BCSet([P.BCEntry(P.PRESSURE, P.TimeTable.constant(cases.CS2))] * 2),
                     P.EngineParams()).close()
    except P.ConfigError as e:
        if "not built" in str(e):
            pytest.skip(str(e))
        raise


@pytest.mark.parametrize("key", sorted(cases.MAP_CASES))
def test_device_table_bit_exact(product, golden, key):
    run = cases.MAP_CASES[key]
    d = cases.make_domain(product, cases.DOMAINS[run["domain"]])
    s = product.Simulation(d, cases.make_bcs(product, run["bcs"]),
                           product.EngineParams(workers=run["W"], layout=run["layout"]))
    assert [cases.map_digest(s.map(w)) for w in range(run["W"])] == golden["maps"][key]


def _writes_partition_store(m, layout):
    """Every f_new location of a worker is written exactly once per step:
    (s, 0) by s, each ToLocal / bounce-back / iolet link by its site, each
    received slot by the exchange (recv_dest) — and the shared links fill
    the tail exactly once (test_layout.cpp:173-191, injectivity and
    coverage).  This is what makes the fused P2P stores, the AA in-place
    update and the pull gather race-free."""
    n = m.n_local
    idx0 = np.arange(n, dtype=np.int64) * 19 if layout == 0 else np.arange(n, dtype=np.int64)
    local = m.dest[m.op != 1].astype(np.int64)
    writes = np.concatenate([idx0, local, m.recv_dest.astype(np.int64)])
    assert writes.size == 19 * n
    assert np.array_equal(np.sort(writes), np.arange(19 * n)), "f_new not partitioned by the step's writes"
    tail = np.sort(m.dest[m.op == 1].astype(np.int64))
    assert np.array_equal(tail, 19 * n + np.arange(m.shared_size))


@pytest.mark.parametrize("spec", [("tree", (12, 48, 6, 0.8, 0.8), 4, 1), ("tree", (8, 40, 7, 0.8, 0.8), 3, 0),
                                  ("blob", 20240808, 23, 0), ("pipe", (16, 128), 8, 1)])
def test_step_writes_partition_the_store(product, spec):
    """Write-disjointness of the device-built tables (the structural check
    standing in for a race detector: compute-sanitizer is closed on this
    GPU pool)."""
    kind, args, W, layout = spec
    if kind == "blob":
        d = product.classify_sites(cases.random_blob(args), [])
        bcs = product.BCSet([])
    else:
        d = getattr(product, "build_" + kind)(*args)
        bcs = product.BCSet([product.BCEntry(product.PRESSURE, product.TimeTable.constant(cases.CS2))
                             for _ in d.iolets])
    s = product.Simulation(d, bcs, product.EngineParams(workers=W, layout=layout))
    for w in range(W):
        _writes_partition_store(s.map(w), layout)


@pytest.mark.parametrize("key", FAST_RUNS)
def test_runs_bit_exact(product, golden, golden_arrays, key):
    res = cases.execute_run(product, cases.RUNS[key])
    want = golden["runs"][key]
    got = cases.run_digest(res)
    arr = golden_arrays.get(f"run_{key}_snapshot")
    if got["snapshot"] != want["snapshot"] and arr is not None:
        dev = np.max(np.abs(res["snapshot"] - arr) / np.maximum(np.abs(arr), 1e-300))
        pytest.fail(f"snapshot differs from the reference, max rel deviation {dev:.3e}")
    assert got == want


@pytest.mark.parametrize("variant", ["1", "3", "5", "10", "11", "12", "13", "14", "15", "16", "17", "18", "19",
                                     "20", "21", "22", "23", "24", "25", "26", "27", "28", "29", "30", "31", "32", "33", "34", "35", "36", "40", "41", "43", "44", "45", "46", "47", "48",
                                     "42", "49", "52", "53", "54", "55", "56", "57", "58", "59", "67", "68", "69",
                                     "70", "71", "74", "75", "76", "77"])
def test_kernel_variants_bit_exact(product, golden, variant, monkeypatch):
    """Every launch shape of the plain kernel (register-resident and
    TMA-pipelined persistent) gives the reference's bits."""
    monkeypatch.setenv("SPLBCU_PLAIN_VARIANT", variant)
    _skip_unbuilt(product)
    for key in ("bif_W3_soa_reordered", "pipe_4_20_W4", "blob1_noise_W23"):
        res = cases.execute_run(product, cases.RUNS[key])
        assert cases.run_digest(res) == golden["runs"][key], key


@pytest.mark.parametrize("key", sorted(cases.RUNS))
@pytest.mark.parametrize("halo", [0, 1])
def test_pull_scheme_bit_exact(product, golden, key, halo):
    """scheme=pull (update_pull + fill_send_slots, engine.hpp:435-502): every
    population gathered from its source with the source's collision
    recomputed; cut links through the send tail + PostReceive (halo 0) or
    stored straight into the neighbour (halo 1).  The reference's bits
    (its push/pull contract, test_engine.cpp:269-300)."""
    res = cases.execute_run(product, dict(cases.RUNS[key], scheme=1), halo_mode=halo)
    assert cases.run_digest(res) == golden["runs"][key]


@pytest.mark.parametrize("key", ["bif_W3_soa_reordered", "bif_W4_noise", "pipe_4_20_W4", "pipe_3_8_obs_W2",
                                 "blob0_noise_W5", "pipe_beat_6_30", "box8_noise_W2_1000"])
def test_fused_p2p_halo_bit_exact(product, golden, key):
    """halo_mode=1: edge kernels store cut-crossing links straight into the
    neighbour's f_new (no shared tail, no PostReceive), flag-synchronised.
    Same bits as the reference."""
    res = cases.execute_run(product, cases.RUNS[key], halo_mode=1)
    assert cases.run_digest(res) == golden["runs"][key]


@pytest.mark.parametrize("key", sorted(cases.RUNS))
def test_aa_single_buffer_bit_exact(product, golden, key):
    """storage=1: one buffer updated in place with the AA pattern (even steps
    local, odd steps gather/scatter, cut links read/written in the
    neighbour's buffer).  Same bits as the reference for every golden run —
    captures and series are taken in both AA states."""
    res = cases.execute_run(product, cases.RUNS[key], storage=1)
    assert cases.run_digest(res) == golden["runs"][key]


@pytest.mark.parametrize("variant", ["0", "60", "61", "62", "63", "64", "65", "66", "72", "79", "81", "88", "89", "90", "91", "92", "93", "94", "95", "96"])
def test_aa_odd_kernel_variants(product, golden, variant, monkeypatch):
    """Odd-step kernels: the default warp-autonomous cp.async pipeline, its
    128-register shape (72), the round-1 register gather over the compressed
    table (64) and over the u32 table (60), and the tuning shapes (61-63, 65,
    66 = CTA-wide cp.async pipeline; built with TUNING=1) give the reference's
    bits."""
    monkeypatch.setenv("SPLBCU_PLAIN_VARIANT", variant)
    _skip_unbuilt(product)
    for key in ("bif_W3_soa_reordered", "pipe_beat_6_30", "C1_pipe_16_128"):
        res = cases.execute_run(product, cases.RUNS[key], storage=1)
        assert cases.run_digest(res) == golden["runs"][key], key


def test_aa_store_views_odd_and_even(product):
    """store(w).f_old() in the AA scheme equals the push engine's after odd
    and even step counts (the state-S gather), for several workers."""
    d = product.build_bifurcation(3, 2, 6, 8)
    bcs = cases.make_bcs(product, ("bif", "bif_inlet"))
    for W in (1, 3):
        a = product.Simulation(d, bcs, product.EngineParams(tau=0.8, dt_s=1e-3, workers=W, layout=product.SOA))
        b = product.Simulation(d, bcs, product.EngineParams(tau=0.8, dt_s=1e-3, workers=W, layout=product.SOA,
                                                            storage=1))
        for n in (7, 6):
            a.run(n)
            b.run(n)
            for w in range(W):
                fa, fb = a.store(w).f_old(), b.store(w).f_old()
                n19 = 19 * a.store(w).n_sites
                assert np.array_equal(fa[:n19], fb[:n19]), (W, n, w)
            assert np.array_equal(a.snapshot_fields(), b.snapshot_fields())


def test_fused_p2p_multi_gpu_in_process(product, golden):
    import torch
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    for key in ("bif_W4_noise", "pipe_4_20_W4"):
        for mode in (0, 1):
            res = cases.execute_run(product, cases.RUNS[key], devices=list(range(n)), halo_mode=mode)
            assert cases.run_digest(res) == golden["runs"][key], (key, mode)
        res = cases.execute_run(product, cases.RUNS[key], devices=list(range(n)), storage=1)
        assert cases.run_digest(res) == golden["runs"][key], (key, "aa")


@pytest.mark.parametrize("mode", ["peer copies", "fused P2P", "AA", "pull"])
def test_eight_slabs_over_all_devices(product, golden, mode):
    """8 workers (8 z-slabs, the 8-GPU decomposition) spread over every
    visible device — 2 per GPU on a 4-GPU box, 8 on one GPU — give the
    single-worker reference bits on C1 (1000 steps) and on the 60-bpm pipe
    with the series (test_engine.cpp:302-368: invariance to worker count)."""
    import torch
    n = torch.cuda.device_count()
    kw = {"peer copies": dict(halo_mode=0), "fused P2P": dict(halo_mode=1), "AA": dict(storage=1),
          "pull": dict(halo_mode=1)}[mode]
    for key in ("C1_pipe_16_128", "pipe_beat_6_30"):
        run = dict(cases.RUNS[key], W=8)
        if mode == "pull":
            run["scheme"] = 1
        res = cases.execute_run(product, run, devices=list(range(n)), **kw)
        assert cases.run_digest(res) == golden["runs"][key], (key, mode)


def test_live_reference_random_case(product, reference):
    """A case outside the golden set, against the reference run live."""
    run = dict(domain="bif_3_2_6_8", bcs=("bif", "bif_inlet"), tau=0.7, dt=2e-3, W=3, layout=1, steps=30,
               capture=10, observe=True, noise=(7, 0.01))
    a = cases.execute_run(product, run)
    b = cases.execute_run(reference, run)
    assert cases.run_digest(a) == cases.run_digest(b)


def test_partition_invariance_many_workers(product):
    """1 vs 2/4/7 workers bitwise (test_engine.cpp:302-315)."""
    d = product.build_pipe(5, 40)
    bcs = cases.make_bcs(product, ("pressure", 0.34, cases.CS2))
    snaps = []
    for W in (1, 2, 4, 7):
        s = product.Simulation(d, bcs, product.EngineParams(tau=0.8, workers=W, capture_period=25))
        s.run(50)
        snaps.append(s.snapshot_fields())
    for x in snaps[1:]:
        assert np.array_equal(x, snaps[0])


def test_fixed_point_closed_box(product):
    """test_engine.cpp:69-78"""
    d = product.classify_sites(cases.closed_box(6), [])
    s = product.Simulation(d, product.BCSet([]), product.EngineParams(tau=0.8))
    before = s.snapshot_fields()
    s.run(50)
    assert np.max(np.abs(s.snapshot_fields() - before)) <= 1e-13


def test_locality_one_link_per_step(product):
    """test_engine.cpp:80-119"""
    d = product.classify_sites(cases.closed_box(9), [])
    e = d.export()
    ref = product.Simulation(d, product.BCSet([]), product.EngineParams(tau=0.8))
    poke = product.Simulation(d, product.BCSet([]), product.EngineParams(tau=0.8))
    center = int(np.where((e["coords"] == [4, 4, 4]).all(1))[0][0])
    lc = poke.assignment().local_index[center]
    st = poke.store(0)
    f = st.f_old()
    f[st.idx(lc, 3)] += 0.01
    st.set_f_old(f)
    ref.run(1)
    poke.run(1)
    a, b = ref.snapshot_fields().reshape(-1, 4), poke.snapshot_fields().reshape(-1, 4)
    changed = np.where((a != b).any(1))[0]
    assert 1 < len(changed) <= 19
    dc = np.abs(e["coords"][changed] - 4)
    assert (dc <= 1).all() and (dc.sum(1) <= 2).all()


def test_capture_schedule_and_rest(product):
    """test_engine.cpp:140-192"""
    d = product.build_pipe(3, 8)
    bcs = cases.make_bcs(product, ("pressure", cases.CS2, cases.CS2))
    s = product.Simulation(d, bcs, product.EngineParams(tau=0.8, capture_period=100))
    f = s.snapshot_fields().reshape(-1, 4)
    assert np.all(np.abs(f[:, 0] - 1.0) <= 1e-15) and np.all(f[:, 1:] == 0.0)
    s.run(0)
    c = s.cache()
    assert len(c) == 1 and c[0].step == 0 and np.array_equal(c[0].fields, f.ravel())
    s.run(201)
    assert np.max(np.abs(s.snapshot_fields().reshape(-1, 4)[:, 1:])) <= 1e-10
    s2 = product.Simulation(product.build_pipe(2, 4), bcs, product.EngineParams(tau=0.8, capture_period=100))
    s2.run(250)
    assert [c.step for c in s2.cache()] == [0, 100, 200]


def test_repeated_runs_continue(product, reference):
    """run() may be called repeatedly; captures/series continue (engine.hpp:155-197)."""
    outs = []
    for M in (product, reference):
        d = M.build_pipe(3, 8)
        s = M.Simulation(d, cases.make_bcs(M, ("pressure", 0.34, cases.CS2)),
                         M.EngineParams(tau=0.8, workers=2, capture_period=7, observe_iolets=True))
        for n in (5, 0, 9, 11):
            s.run(n)
        outs.append((s.snapshot_fields(), [(c.step, cases.h(c.fields)) for c in s.cache()],
                     {k: [cases.h(a) for a in v] for k, v in s.series().items() if k != "rows"}, s.steps_run()))
    assert cases.h(outs[0][0]) == cases.h(outs[1][0])
    assert outs[0][1:] == outs[1][1:]


def test_store_roundtrip_layouts(product):
    d = product.build_bifurcation(3, 2, 6, 8)
    for lay in (product.AOS, product.SOA):
        s = product.Simulation(d, cases.make_bcs(product, ("bif", "bif_inlet")),
                               product.EngineParams(tau=0.8, workers=3, layout=lay))
        for w in range(3):
            st = s.store(w)
            x = np.random.default_rng(w).uniform(0, 1, st.total_size())
            st.set_f_old(x)
            assert np.array_equal(st.f_old(), x)


@pytest.mark.parametrize("storage", [0, 1])
def test_store_set_then_step_large(product, storage):
    """set_f of large stores is ordered before the next kernels (a legacy
    pageable cudaMemcpy can return before its DMA lands, and the engine's
    streams do not wait for it): 3 workers, 2.3e5 sites, a perturbed store
    written and read back, then stepped — equal to one worker, every time."""
    d = product.build_channel(48, 40, 120)
    bcs = product.BCSet([product.BCEntry(product.PRESSURE, product.TimeTable.constant(cases.CS2 * 1.001)),
                         product.BCEntry(product.PRESSURE, product.TimeTable.constant(cases.CS2 * 0.999))])
    noise = cases.noise_for(d.n_sites(), 20240808, 0.01)
    ref = product.Simulation(d, bcs, product.EngineParams(tau=0.8))
    cases.apply_noise(product, ref, noise)
    ref.run(1)
    want = ref.snapshot_fields()
    for rep in range(3):
        s = product.Simulation(d, bcs, product.EngineParams(tau=0.8, workers=3, storage=storage))
        cases.apply_noise(product, s, noise)
        pa = s.assignment()
        for w in range(3):
            got = s.store(w).f_old()
            n = len(pa.parts[w].sites)
            assert np.all(got[:19 * n].reshape(n, 19) >= 0.0)
        s.run(1)
        assert np.array_equal(s.snapshot_fields(), want), (storage, rep)
        s.close()


def test_multi_device_placement_single_gpu(product):
    """Workers placed round-robin on the device list; with one device all
    share it and exchange by device-to-device copies."""
    d = product.build_pipe(4, 20)
    bcs = cases.make_bcs(product, ("pressure", 0.3383333333333333, cases.CS2))
    a = product.Simulation(d, bcs, product.EngineParams(tau=0.8, workers=4, devices=[0, 0]))
    b = product.Simulation(d, bcs, product.EngineParams(tau=0.8, workers=1))
    a.run(30)
    b.run(30)
    assert np.array_equal(a.snapshot_fields(), b.snapshot_fields())


def test_velocity_pipe_centerline(product):
    """test_engine.cpp:370-401: velocity-driven pipe reaches the imposed
    centreline speed within 3% (R=8)."""
    R, Len, u0 = 8, 64, 0.04
    d = product.build_pipe(R, Len)
    bcs = cases.make_bcs(product, ("velocity_const", u0))
    s = product.Simulation(d, bcs, product.EngineParams(tau=0.9, workers=2))
    e = d.export()
    mid = np.where(e["coords"][:, 2] == Len // 2)[0]
    r2 = (e["coords"][mid, 0] - 0.375) ** 2 + (e["coords"][mid, 1] - 0.5) ** 2
    cidx = mid[np.argmin(r2)]
    q_prev = 0.0
    for _ in range(60):
        s.run(250)
        f = s.snapshot_fields().reshape(-1, 4)
        q = f[mid, 3].sum()
        if abs(q - q_prev) < 1e-7 * abs(q):
            break
        q_prev = q
    assert abs(f[cidx, 3] - u0) / u0 <= 0.03


def test_engine_rejects_bad_setup(product):
    d = product.build_pipe(3, 8)
    with pytest.raises(product.ConfigError, match="configured for 1 iolets"):
        product.Simulation(d, product.BCSet([product.BCEntry(product.PRESSURE, product.TimeTable.constant(0.3))]),
                           product.EngineParams())
    with pytest.raises(product.ConfigError, match="tau must exceed 0.5"):
        product.Simulation(d, cases.make_bcs(product, ("pressure", 0.3, 0.3)), product.EngineParams(tau=0.5))
    with pytest.raises(product.ConfigError, match="ghost density must stay positive"):
        product.Simulation(d, cases.make_bcs(product, ("pressure", -0.3, 0.3)), product.EngineParams())
    with pytest.raises(product.Error, match="exceeds site count"):
        product.Simulation(product.classify_sites(cases.closed_box(2), []), product.BCSet([]),
                           product.EngineParams(workers=9))


def test_kernel_timing_counts(product):
    d = product.build_pipe(8, 64)
    s = product.Simulation(d, cases.make_bcs(product, ("pressure", cases.CS2, cases.CS2)), product.EngineParams())
    s.set_kernel_timing(True)
    s.run(10)
    secs, launches, sites = s.kernel_stats()
    assert launches == 10 and secs > 0.0
    e = d.export()["type_ranges"]
    assert sites == 10 * int(e[1][1])  # Inner + Wall sites per step


def test_output_files_match_reference(product, reference, tmp_path):
    """snapshots.bin and timeseries.csv written from the B200 engine are
    byte-identical to the reference's writers (snapshot.hpp:15-82)."""
    outs = []
    for M in (product, reference):
        run = dict(domain="bif_3_2_6_8", bcs=("bif", "bif_inlet"), tau=0.8, dt=1e-3, W=3, steps=40, capture=10,
                   observe=True)
        res = cases.execute_run(M, run)
        p = str(tmp_path / f"{M.__name__}.bin")
        res["sim"].write_snapshots(p)
        outs.append((open(p, "rb").read(), res["sim"].series_csv(1e-3)))
    assert outs[0][0] == outs[1][0]
    assert outs[0][1] == outs[1][1]


def test_online_bulk_kernel_choice(product, monkeypatch):
    """The engine times the bulk kernels online (every 500 launches: delta
    table with a dynamic tile order / prefetch, run-length table) and keeps
    the fastest; switching between them mid-run leaves the bits alone,
    and splbcu_sim_bulk_kernel reports the choice (forced variants included)."""
    d = product.build_pipe(16, 128)
    bcs = cases.make_bcs(product, ("pressure", cases.CS2 * 1.001, cases.CS2 * 0.999))

    def run(variant, steps=1010):
        if variant is None:
            monkeypatch.delenv("SPLBCU_PLAIN_VARIANT", raising=False)
        else:
            monkeypatch.setenv("SPLBCU_PLAIN_VARIANT", variant)
        s = product.Simulation(d, bcs, product.EngineParams())
        s.run(steps)
        return s.bulk_kernel(), s.snapshot_fields()

    k_auto, f_auto = run(None)
    k76, f76 = run("76")
    k43, f43 = run("43")
    k59, f59 = run("59")
    k71, f71 = run("71")
    k1, _ = run("24", 2)  # the u32-table kernel everywhere
    assert k_auto in (0, 1, 2) and (k76, k59, k71, k43, k1) == (0, 1, 2, 3, -1)
    for f in (f76, f43, f59, f71):
        assert np.array_equal(f_auto, f)


@pytest.mark.parametrize("variant", ["43", "59", "71", "76"])
def test_chunked_bulk_range_bit_exact(product, golden, variant, monkeypatch):
    """SPLBCU_BULK_CHUNK (tuning knob) cuts the bulk range into several
    launches at 256-site boundaries; the bits do not change."""
    monkeypatch.setenv("SPLBCU_PLAIN_VARIANT", variant)
    monkeypatch.setenv("SPLBCU_BULK_CHUNK", "700")
    for key in ("bif_W3_soa_reordered", "pipe_4_20_W4", "blob1_noise_W23"):
        res = cases.execute_run(product, cases.RUNS[key])
        assert cases.run_digest(res) == golden["runs"][key], key
