// The reference's engine tests (proj/tests/test_engine.cpp), restated against
// the B200 engine through include/splbcu.hpp.  A tiny CHECK harness stands in
// for doctest; exit code = number of failed checks.
#include <cmath>
#include <cstdio>
#include <random>

#include "splbcu.hpp"

using namespace splb;

static int g_fail = 0;
#define CHECK(c)                                                          \
    do {                                                                  \
        if (!(c)) {                                                       \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);      \
            ++g_fail;                                                     \
        }                                                                 \
    } while (0)

static SparseDomain closed_box(int n) {
    std::vector<Vec3i> v;
    for (int z = 0; z < n; ++z)
        for (int y = 0; y < n; ++y)
            for (int x = 0; x < n; ++x) v.push_back({x, y, z});
    return classify_sites(v, {});
}

static BCSet pipe_bcs(double pin, double pout) {
    BCSet b;
    b.entries = {{BCSet::Kind::Pressure, TimeTable::constant(pin)}, {BCSet::Kind::Pressure, TimeTable::constant(pout)}};
    return b;
}

static EngineParams params(int workers, uint64_t capture = 0) {
    EngineParams p;
    p.tau = 0.8;
    p.workers = workers;
    p.capture_period = capture;
    p.dt_s = 1e-3;
    return p;
}

int main() {
    const double cs2 = 1.0 / 3.0;
    {  // uniform equilibrium in a closed box is a fixed point (test_engine.cpp:69-78)
        Simulation sim(closed_box(6), BCSet{}, params(1));
        const auto before = sim.snapshot_fields();
        sim.run(50);
        const auto after = sim.snapshot_fields();
        for (size_t k = 0; k < before.size(); ++k) CHECK(std::abs(after[k] - before[k]) <= 1e-13);
    }
    {  // closed all-wall box conserves mass to 1e-12 over 1000 steps (121-138)
        Simulation sim(closed_box(8), BCSet{}, params(2));
        std::mt19937_64 rng(99);
        std::uniform_real_distribution<double> noise(0.0, 0.05);
        double m0 = 0.0;
        for (int w = 0; w < 2; ++w) {
            DistributionStore& s = sim.store(w);  // mutable, as the reference's store(w)
            for (uint32_t site = 0; site < s.n_sites; ++site)
                for (int i = 0; i < 19; ++i) s.f_old()[s.idx(site, i)] += noise(rng);
            for (uint32_t site = 0; site < s.n_sites; ++site)
                for (int i = 0; i < 19; ++i) m0 += s.f_old()[s.idx(site, i)];
        }
        sim.run(1000);
        double m1 = 0.0;
        for (int w = 0; w < 2; ++w) {
            const DistributionStore& s = sim.store(w);
            for (uint32_t site = 0; site < s.n_sites; ++site)
                for (int i = 0; i < 19; ++i) m1 += s.f_old()[s.idx(site, i)];
        }
        CHECK(std::abs(m1 - m0) <= 1e-12 * m0);
    }
    {  // pipe partition invariance: 1 vs 4 workers over 100 steps (302-315)
        const SparseDomain d = build_pipe(4, 20);
        Simulation a(d, pipe_bcs(0.3383333333333333, cs2), params(1, 50));
        Simulation b(d, pipe_bcs(0.3383333333333333, cs2), params(4, 50));
        a.run(100);
        b.run(100);
        const auto ca = a.cache().captures, cb = b.cache().captures;
        CHECK(ca.size() == cb.size());
        for (size_t c = 0; c < ca.size() && c < cb.size(); ++c) CHECK(ca[c].fields == cb[c].fields);
    }
    {  // capture schedule (182-192)
        Simulation sim(build_pipe(2, 4), pipe_bcs(cs2, cs2), params(1, 100));
        sim.run(250);
        const auto c = sim.cache().captures;
        CHECK(c.size() == 3);
        if (c.size() == 3) CHECK(c[0].step == 0 && c[1].step == 100 && c[2].step == 200);
    }
    {  // iolet series rows cover init plus every step (444-459)
        auto p = params(2);
        p.observe_iolets = true;
        Simulation sim(build_pipe(3, 8), pipe_bcs(0.34, cs2), p);
        sim.run(25);
        const IoletSeries s = sim.series();
        CHECK(s.rows == 26);
        CHECK(s.flow.size() == 2);
        if (s.flow.size() == 2) CHECK(s.flow[0][25] > 0.0);
    }
    {  // engine rejects inconsistent BC sets (418-426)
        bool threw = false;
        try {
            BCSet few;
            few.entries = {{BCSet::Kind::Pressure, TimeTable::constant(cs2)}};
            Simulation sim(build_pipe(3, 8), few, params(1));
        } catch (const ConfigError&) {
            threw = true;
        }
        CHECK(threw);
    }
    {  // B200 extension: one-rank distributed engine over a geometry source
       // (slab-local construction) == the in-process engine on the built domain
        auto p = params(1);
        p.observe_iolets = true;
        const Source src = Source::pipe(3, 12);
        uint8_t id[128];
        Simulation::nccl_unique_id(id);
        Simulation a = Simulation::distributed(src, pipe_bcs(0.34, cs2), p, 0, 1, id);
        Simulation b(src.build(), pipe_bcs(0.34, cs2), p);
        a.run(30);
        b.run(30);
        CHECK(a.slab_local() && !b.slab_local());
        CHECK(a.n_sites() == b.domain().n_sites());
        CHECK(a.snapshot_fields() == b.snapshot_fields());
        CHECK(a.series().flow == b.series().flow);
    }
    {  // store(w) is a live, mutable view (engine.hpp:149): a write through it
       // reaches the next step, and the same reference reads the new state
        Simulation a(closed_box(5), BCSet{}, params(2)), b(closed_box(5), BCSet{}, params(2));
        DistributionStore& sb = b.store(1);
        const size_t k = sb.idx(3, 3);
        const double v0 = sb.f_old()[k];
        sb.f_old()[k] += 0.01;
        a.run(1);
        b.run(1);
        CHECK(a.snapshot_fields() != b.snapshot_fields());
        CHECK(sb.f_old()[k] != v0 + 0.01);  // refetched after the step
        const DistributionStore copy = b.store(1);  // detached snapshot of the same state
        bool same = true;
        for (size_t q = 0; q < copy.total_size(); ++q) same &= copy.f_old()[q] == sb.f_old()[q];
        CHECK(same);
        double ma = 0.0, mb = 0.0;
        for (int w = 0; w < 2; ++w)
            for (size_t q = 0; q < a.store(w).shared_base(); ++q) ma += a.store(w).f_old()[q], mb += b.store(w).f_old()[q];
        CHECK(std::abs((mb - ma) - 0.01) <= 1e-12);  // the poke is conserved
    }
    std::printf("%d check(s) failed\n", g_fail);
    return g_fail;
}
