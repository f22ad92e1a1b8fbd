"""Host-side logic of the B200 engine (libsplbcu.so, no GPU needed):
classification, validation, decomposition, time tables, geometry files and
the lattice helpers, all checked bit-exactly against the reference's golden
vectors (tests/golden) and, when built, the reference itself."""
import os

import numpy as np
import pytest

import cases


def test_kat(product, golden, golden_arrays):
    assert product.equilibrium(1.0, [0, 0, 0]).tolist() == golden["kat"]["eq_rest"]
    assert product.equilibrium(1.0, [0.1, 0.0, 0.0]).tolist() == golden["kat"]["eq_01"]
    F = golden_arrays["kat_f"]
    # folded device arithmetic (lattice.hpp of the product) == reference
    assert np.array_equal(np.stack([product.bgk_collide(f, 0.8) for f in F]), golden_arrays["kat_collide_08"])
    mom = np.stack([np.r_[product.moments(f)[0], product.moments(f)[1]] for f in F])
    assert np.array_equal(mom, golden_arrays["kat_moments"])
    eq = np.stack([product.equilibrium(r[0], r[1:]) for r in golden_arrays["kat_eq_in"]])
    assert np.array_equal(eq, golden_arrays["kat_eq"])
    with pytest.raises(product.DegenerateState):
        product.moments(np.zeros(19))


def test_tables_and_weights(product, golden):
    for name, tab in cases.TABLES.items():
        ts = np.linspace(-0.3, 2.7, 61)
        assert [product.TimeTable(tab[0], tab[1]).at(float(t)) for t in ts] == golden["kat"]["tables"][name]
    io = product.Iolet(0, [0.375, 0.5, -0.5], [0.0, 0.0, 1.0], 8.0)
    assert [product.iolet_weight(io, c) for c in cases.WEIGHT_COORDS] == golden["kat"]["weights"]
    for bad, msg in [(([], 0.0), "empty table"), (([(0.0, 1.0), (0.0, 2.0)], 0.0), "strictly ascending"),
                     (([(0.0, 1.0)], -1.0), "period must be > 0"), (([(0.0, 1.0), (1.5, 1)], 1.0), "inside one period"),
                     (([(-0.1, 1.0)], 1.0), "starts before t=0")]:
        with pytest.raises(product.ConfigError, match=msg):
            product.TimeTable(*bad).at(0.0)


@pytest.mark.parametrize("name", sorted(cases.DOMAINS))
def test_domains_bit_exact(product, golden, name):
    d = cases.make_domain(product, cases.DOMAINS[name])
    assert cases.domain_digest(d) == golden["domains"][name]


@pytest.mark.parametrize("key", sorted(cases.PARTITION_WORKERS))
def test_partitions_bit_exact(product, golden, key):
    d = cases.make_domain(product, cases.DOMAINS[key])
    for W in cases.PARTITION_WORKERS[key]:
        assert cases.partition_digest(product.partition(d, W)) == golden["partitions"][f"{key}/W{W}"]


def test_classify_shuffled_input(product, golden):
    """classify_sites sorts any input order (geometry.hpp:189-195)."""
    v = cases.closed_box(8)
    rng = np.random.default_rng(3)
    d = product.classify_sites(v[rng.permutation(len(v))], [])
    assert cases.domain_digest(d) == golden["domains"]["box8"]


def test_classify_errors(product, port):
    for M in (product, port):
        with pytest.raises(M.GeometryError, match="empty voxel set"):
            M.classify_sites(np.zeros((0, 3), np.int32), [])
        with pytest.raises(M.GeometryError, match="duplicate voxel"):
            M.classify_sites([[0, 0, 0], [1, 0, 0], [0, 0, 0]], [])
        with pytest.raises(M.GeometryError, match="normal is not unit length"):
            M.classify_sites(cases.closed_box(3), [M.Iolet(0, [0, 0, -0.5], [0, 0, 2.0], 1.0)])
        with pytest.raises(M.GeometryError, match="intersects no boundary links"):
            M.classify_sites(cases.closed_box(3), [M.Iolet(0, [50, 50, -0.5], [0, 0, 1.0], 1.0)])
        # inlet and outlet planes both cut a 1-plane slab
        with pytest.raises(M.GeometryError, match=r"site \(0,0,0\) carries both inlet and outlet"):
            M.classify_sites([[0, 0, 0]], [M.Iolet(0, [0, 0, -0.5], [0, 0, 1.0], 3.0),
                                          M.Iolet(1, [0, 0, 0.5], [0, 0, -1.0], 3.0)])
        with pytest.raises(M.GeometryError, match="need radius >= 2"):
            M.build_pipe(1, 8)
        with pytest.raises(M.GeometryError, match="need radii >= 2"):
            M.build_bifurcation(3, 1, 6, 8)


def test_validate_domain_errors(product, port):
    for M in (product, port):
        e = M.build_pipe(3, 8).export()
        args = lambda **kw: {**dict(coords=e["coords"], types=e["types"], link_kind=e["link_kind"],  # noqa: E731
                                    link_iolet=e["link_iolet"], iolets=e["iolets"], type_ranges=e["type_ranges"]), **kw}
        M.SparseDomain.from_arrays(**args()).validate()
        lk = e["link_kind"].copy()
        lk[0, 0] = 1 - lk[0, 0] if lk[0, 0] <= 1 else 0
        with pytest.raises(M.GeometryError, match="inconsistent link closure"):
            M.SparseDomain.from_arrays(**args(link_kind=lk))
        tr = e["type_ranges"].copy()
        tr[0, 1] -= 1
        with pytest.raises(M.GeometryError, match="type_ranges do not partition"):
            M.SparseDomain.from_arrays(**args(type_ranges=tr))
        ty = e["types"].copy()
        ty[0] = 1
        with pytest.raises(M.GeometryError, match="site type outside its range"):
            M.SparseDomain.from_arrays(**args(types=ty))
        li = e["link_iolet"].copy()
        li[e["link_kind"] >= 2] = 7
        with pytest.raises(M.GeometryError, match="unknown iolet"):
            M.SparseDomain.from_arrays(**args(link_iolet=li))


def test_partition_errors(product):
    d = product.classify_sites(cases.closed_box(2), [])
    with pytest.raises(product.Error, match="nWorkers must be >= 1"):
        product.partition(d, 0)
    with pytest.raises(product.Error, match=r"nWorkers \(9\) exceeds site count \(8\)"):
        product.partition(d, 9)
    p = product.partition(d, 8)  # nWorkers == nSites (test_decomp.cpp:118-131)
    assert all(len(w.sites) == 1 for w in p.parts)


def test_geometry_file_roundtrip(product, tmp_path, reference):
    d = product.build_bifurcation(3, 2, 6, 8)
    path = str(tmp_path / "bif.splb")
    d.write(path)
    back = product.SparseDomain.read(path)
    assert cases.domain_digest(back) == cases.domain_digest(d)
    # the file is byte-identical to the reference writer's
    rp = str(tmp_path / "bif_ref.splb")
    reference.build_bifurcation(3, 2, 6, 8).write(rp)
    assert open(path, "rb").read() == open(rp, "rb").read()
    with open(path, "r+b") as f:
        f.write(b"XXXX")
    with pytest.raises(product.GeometryError, match="not a SPLB file"):
        product.SparseDomain.read(path)


def test_generators_validate(product, reference):
    """Tree (C3) and channel (C4) generators produce domains the reference's
    own validate_domain accepts, and the product partitions them like the
    reference."""
    for d in (product.build_tree(6, 24, 3, 0.8, 0.8), product.build_channel(6, 5, 12)):
        e = d.export()
        r = reference.SparseDomain.from_arrays(e["coords"], e["types"], e["link_kind"], e["link_iolet"],
                                               [reference.Iolet(i.kind, i.center, i.normal, i.radius) for i in e["iolets"]],
                                               e["type_ranges"])
        r.validate()
        for W in (1, 3, 8):
            assert cases.partition_digest(product.partition(d, W)) == cases.partition_digest(reference.partition(r, W))


@pytest.mark.parametrize("spec", [("tree", 6, 24, 3, 0.8, 0.8), ("tree", 8, 40, 5, 0.8, 0.8),
                                  ("tree", 5, 20, 6, 0.8, 0.8), ("tree", 12, 30, 2, 0.7, 0.6),
                                  ("channel", 10, 12, 30), ("channel", 7, 5, 9)])
def test_generators_match_reference_classifier(product, reference, spec):
    """The bench geometries (C3/C5 trees with up to 65 iolets, the C4
    channel) from the product's generator + classifier are bit-identical to
    the reference's classify_sites (geometry.hpp:139-208) run on the same
    voxels (oracle/geometry_gen.py restates the voxelisation): coordinates,
    types, every link's kind and iolet id, type ranges and iolet discs."""
    import geometry_gen as G
    kind, args = spec[0], spec[1:]
    vox, io = getattr(G, kind)(*args)
    r = G.classify(reference, vox, io)
    d = getattr(product, "build_" + kind)(*args)
    assert cases.domain_digest(d) == cases.domain_digest(r)
    got = [(i.kind, tuple(i.center), tuple(i.normal), i.radius) for i in d.export()["iolets"]]
    want = [(i.kind, tuple(i.center), tuple(i.normal), i.radius) for i in r.export()["iolets"]]
    assert got == want


def test_tree_size_model(product):
    d = product.build_tree(8, 40, 4, 0.8, 0.8)
    e = d.export()
    assert d.n_sites() > 10000
    assert len(e["iolets"]) == 1 + 2 ** 4


# ---- slab-local construction ---------------------------------
SOURCES = {
    "pipe": (("pipe", 6, 40), "build_pipe", (6, 40)),
    "bifurcation": (("bifurcation", 5, 3, 12, 16), "build_bifurcation", (5, 3, 12, 16)),
    "tree": (("tree", 6, 24, 3, 0.8, 0.8), "build_tree", (6, 24, 3, 0.8, 0.8)),
    "channel": (("channel", 6, 5, 30), "build_channel", (6, 5, 30)),
}


def _source(P, spec):
    kind, *args = spec
    return getattr(P.Source, kind)(*args)


@pytest.mark.parametrize("name", sorted(SOURCES))
def test_source_build_matches_builder(product, name):
    spec, builder, args = SOURCES[name]
    a = _source(product, spec).build().export()
    b = getattr(product, builder)(*args).export()
    for k in ("coords", "types", "link_kind", "link_iolet", "type_ranges"):
        assert np.array_equal(a[k], b[k]), k


@pytest.mark.parametrize("name", sorted(SOURCES))
@pytest.mark.parametrize("W", [1, 2, 3, 5])
def test_source_window_matches_whole_domain(product, name, W):
    """Each rank's window (own slices + one halo slice per side) holds exactly
    the whole domain's sites there, at their global indices, classified the
    same; its part equals partition() of the whole domain."""
    spec, builder, args = SOURCES[name]
    src = _source(product, spec)
    full = getattr(product, builder)(*args)
    e = full.export()
    part = product.partition(full, W)
    z = e["coords"][:, 2]
    for w in range(W):
        win = src.window(W, w)
        assert win is not None
        assert win["n_global"] == full.n_sites()
        lo, hi = win["own"]
        gi = win["global_index"].astype(np.int64)
        want = np.flatnonzero((z >= lo - 1) & (z <= hi + 1))
        assert np.array_equal(np.sort(gi), want)  # the window is exactly those slices
        assert np.all(np.diff(gi[np.argsort(gi)]) > 0)
        we = win["domain"].export()
        for k in ("coords", "types", "link_kind", "link_iolet"):
            assert np.array_equal(we[k], e[k][gi]), k
        mine = win["part"].parts[w]
        ref = part.parts[w]
        assert np.array_equal(gi[mine.sites], ref.sites.astype(np.int64))
        assert mine.n_edge == ref.n_edge
        assert np.array_equal(mine.edge_ranges, ref.edge_ranges)
        assert np.array_equal(mine.mid_ranges, ref.mid_ranges)
        assert mine.neighbors == ref.neighbors
        assert np.array_equal(win["part"].owner, part.owner[gi])


def test_source_window_not_slab(product):
    """Longest axis x (a wide, short channel) or more workers than slices:
    the partition is not a z-slab split, so ranks build the whole domain."""
    assert product.Source.channel(40, 6, 12).window(2, 0) is None
    assert product.Source.pipe(4, 6).window(7, 0) is None
    with pytest.raises(product.GeometryError, match="build_pipe"):
        product.Source.pipe(1, 6)
