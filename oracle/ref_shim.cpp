// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// Exposes the UNMODIFIED reference engine (header-only splb, compiled from
// /root/reference/proj/include by oracle/Makefile with the reference's own
// -ffp-contract=off) behind the same C-ABI names and struct layouts as
// include/splbcu.h, so tests and bench.py's CPU arm can drive both engines
// through one Python mirror.  Output: oracle/_ref/libsplbref.so.
//
// Every function forwards to the reference symbol named in include/splbcu.h.
#include <cstring>
#include <memory>
#include <sstream>
#include <string>

#include "splb/engine.hpp"
#include "splb/geometry_io.hpp"
#include "splb/snapshot.hpp"
#include "splbcu.h"

using namespace splb;

struct splbcu_domain {
    SparseDomain d;
};
struct splbcu_partition {
    PartitionAssignment p;
    bool borrowed = false;
};
struct splbcu_sim {
    std::unique_ptr<Simulation> s;
    splbcu_partition view;
    uint64_t dom_n = 0;
};

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const ConfigError& e) {
        g_err = e.what();
        return SPLBCU_ERR_CONFIG;
    } catch (const GeometryError& e) {
        g_err = e.what();
        return SPLBCU_ERR_GEOMETRY;
    } catch (const DegenerateState& e) {
        g_err = e.what();
        return SPLBCU_ERR_DEGENERATE;
    } catch (const Error& e) {
        g_err = e.what();
        return std::string(e.what()).find("exchange failure") != std::string::npos ? SPLBCU_ERR_COMM
                                                                                     : SPLBCU_ERR_RUNTIME;
    } catch (const std::exception& e) {
        g_err = e.what();
        return SPLBCU_ERR_RUNTIME;
    }
}

std::vector<Iolet> to_iolets(const splbcu_iolet* io, uint32_t n) {
    std::vector<Iolet> v(n);
    for (uint32_t k = 0; k < n; ++k) {
        v[k].kind = io[k].kind == 0 ? Iolet::Kind::Inlet : Iolet::Kind::Outlet;
        for (int a = 0; a < 3; ++a) v[k].center[a] = io[k].center[a], v[k].normal[a] = io[k].normal[a];
        v[k].radius = io[k].radius;
    }
    return v;
}

TimeTable to_table(const double* t, const double* v, uint32_t n, double period) {
    TimeTable tt;
    for (uint32_t k = 0; k < n; ++k) tt.nodes.push_back({t[k], v[k]});
    tt.period = period;
    return tt;
}
}  // namespace

extern "C" {

const char* splbcu_last_error(void) { return g_err.c_str(); }
const char* splbcu_version(void) { return "splb reference (CPU, /root/reference/proj/include)"; }
void splbcu_params_default(splbcu_params* p) {
    std::memset(p, 0, sizeof(*p));
    EngineParams d;
    p->tau = d.tau;
    p->rho0 = d.rho0;
    p->dt_s = d.dt_s;
    p->workers = d.workers;
    p->exchange_timeout_s = d.exchange_timeout_s;
}

void splbcu_equilibrium(double rho, const double u[3], double out[19]) {
    const Populations p = equilibrium(rho, {u[0], u[1], u[2]});
    std::memcpy(out, p.data(), sizeof(double) * 19);
}
int splbcu_moments(const double f[19], double* rho, double u[3]) {
    return guard([&] {
        Populations p;
        std::memcpy(p.data(), f, sizeof(double) * 19);
        const SiteMacro m = moments(p);
        *rho = m.rho;
        for (int a = 0; a < 3; ++a) u[a] = m.u[a];
    });
}
int splbcu_bgk_collide(const double f[19], double tau, double out[19]) {
    return guard([&] {
        Populations p;
        std::memcpy(p.data(), f, sizeof(double) * 19);
        const Populations o = bgk_collide(p, RelaxationParams(tau));
        std::memcpy(out, o.data(), sizeof(double) * 19);
    });
}
int splbcu_timetable_at(const double* t, const double* v, uint32_t n, double period, double tq, double* out) {
    return guard([&] {
        TimeTable tt = to_table(t, v, n, period);
        tt.validate();
        *out = tt.at(tq);
    });
}
double splbcu_iolet_weight(const splbcu_iolet* io, const int32_t c[3]) {
    return iolet_weight(to_iolets(io, 1)[0], {c[0], c[1], c[2]});
}

int splbcu_domain_classify(const int32_t* vox, uint64_t n, const splbcu_iolet* io, uint32_t nio, double vs,
                           splbcu_domain** out) {
    return guard([&] {
        std::vector<Vec3i> v(n);
        for (uint64_t s = 0; s < n; ++s) v[s] = {vox[3 * s], vox[3 * s + 1], vox[3 * s + 2]};
        auto d = std::make_unique<splbcu_domain>();
        d->d = classify_sites(v, to_iolets(io, nio), vs);
        *out = d.release();
    });
}
int splbcu_domain_build_pipe(int32_t r, int32_t l, double vs, splbcu_domain** out) {
    return guard([&] {
        auto d = std::make_unique<splbcu_domain>();
        d->d = build_pipe(r, l, vs);
        *out = d.release();
    });
}
int splbcu_domain_build_bifurcation(int32_t tr, int32_t br, int32_t tl, int32_t bl, double vs,
                                    splbcu_domain** out) {
    return guard([&] {
        auto d = std::make_unique<splbcu_domain>();
        d->d = build_bifurcation(tr, br, tl, bl, vs);
        *out = d.release();
    });
}
int splbcu_domain_build_tree(int32_t, int32_t, int32_t, double, double, double, splbcu_domain**) {
    g_err = "reference has no tree generator";
    return SPLBCU_ERR_CONFIG;
}
int splbcu_domain_build_channel(int32_t, int32_t, int32_t, double, splbcu_domain**) {
    g_err = "reference has no channel generator";
    return SPLBCU_ERR_CONFIG;
}
int splbcu_domain_from_arrays(uint64_t n, const int32_t* coords, const uint8_t* types, const uint8_t* kind,
                              const uint16_t* iol, const splbcu_iolet* io, uint32_t nio, const uint64_t* tr,
                              double vs, splbcu_domain** out) {
    return guard([&] {
        auto dd = std::make_unique<splbcu_domain>();
        SparseDomain& d = dd->d;
        d.voxel_size = vs;
        d.sites.resize(n);
        for (uint64_t s = 0; s < n; ++s) {
            SiteRecord& r = d.sites[s];
            r.coords = {coords[3 * s], coords[3 * s + 1], coords[3 * s + 2]};
            r.type = CollisionType(types[s]);
            for (int i = 0; i < 18; ++i) {
                r.links[i].kind = LinkKind(kind[18 * s + i]);
                r.links[i].iolet = kind[18 * s + i] >= 2 && iol ? iol[18 * s + i] : 0;
            }
        }
        d.iolets = to_iolets(io, nio);
        for (int t = 0; t < 6; ++t) d.type_ranges[t] = {tr[2 * t], tr[2 * t + 1]};
        validate_domain(d);
        *out = dd.release();
    });
}
int splbcu_domain_validate(const splbcu_domain* d) {
    return guard([&] { validate_domain(d->d); });
}
int splbcu_domain_read(const char* path, splbcu_domain** out) {
    return guard([&] {
        auto d = std::make_unique<splbcu_domain>();
        d->d = read_domain(std::string(path));
        *out = d.release();
    });
}
int splbcu_domain_write(const splbcu_domain* d, const char* path) {
    return guard([&] { write_domain(d->d, std::string(path)); });
}
uint64_t splbcu_domain_n_sites(const splbcu_domain* d) { return d->d.n_sites(); }
uint32_t splbcu_domain_n_iolets(const splbcu_domain* d) { return uint32_t(d->d.iolets.size()); }
double splbcu_domain_voxel_size(const splbcu_domain* d) { return d->d.voxel_size; }
int splbcu_domain_export(const splbcu_domain* dd, int32_t* coords, uint8_t* types, uint8_t* kind, uint16_t* iol,
                         splbcu_iolet* io, uint64_t* tr) {
    return guard([&] {
        const SparseDomain& d = dd->d;
        for (uint64_t s = 0; s < d.n_sites(); ++s) {
            const SiteRecord& r = d.sites[s];
            if (coords)
                for (int a = 0; a < 3; ++a) coords[3 * s + a] = r.coords[a];
            if (types) types[s] = uint8_t(r.type);
            for (int i = 0; i < 18; ++i) {
                if (kind) kind[18 * s + i] = uint8_t(r.links[i].kind);
                if (iol) iol[18 * s + i] = r.links[i].iolet;
            }
        }
        if (io)
            for (size_t k = 0; k < d.iolets.size(); ++k) {
                io[k].kind = int32_t(d.iolets[k].kind);
                for (int a = 0; a < 3; ++a) io[k].center[a] = d.iolets[k].center[a], io[k].normal[a] = d.iolets[k].normal[a];
                io[k].radius = d.iolets[k].radius;
            }
        if (tr)
            for (int t = 0; t < 6; ++t) tr[2 * t] = d.type_ranges[t].begin, tr[2 * t + 1] = d.type_ranges[t].end;
    });
}
void splbcu_domain_free(splbcu_domain* d) { delete d; }

int splbcu_partition_create(const splbcu_domain* d, int32_t w, splbcu_partition** out) {
    return guard([&] {
        auto p = std::make_unique<splbcu_partition>();
        p->p = partition(d->d, w);
        *out = p.release();
    });
}
int splbcu_partition_global(const splbcu_partition* p, int32_t* owner, uint32_t* li) {
    return guard([&] {
        for (size_t s = 0; s < p->p.owner.size(); ++s) {
            if (owner) owner[s] = p->p.owner[s];
            if (li) li[s] = p->p.local_index[s];
        }
    });
}
int splbcu_partition_part_shape(const splbcu_partition* p, int32_t w, uint32_t* ns, uint32_t* ne, uint32_t* nn) {
    return guard([&] {
        const auto& wp = p->p.parts.at(size_t(w));
        if (ns) *ns = uint32_t(wp.sites.size());
        if (ne) *ne = wp.n_edge;
        if (nn) *nn = uint32_t(wp.neighbors.size());
    });
}
int splbcu_partition_part(const splbcu_partition* p, int32_t w, uint32_t* sites, uint64_t* er, uint64_t* mr,
                          int32_t* nb) {
    return guard([&] {
        const auto& wp = p->p.parts.at(size_t(w));
        if (sites) std::memcpy(sites, wp.sites.data(), wp.sites.size() * 4);
        for (int t = 0; t < 6; ++t) {
            if (er) er[2 * t] = wp.edge_ranges[t].begin, er[2 * t + 1] = wp.edge_ranges[t].end;
            if (mr) mr[2 * t] = wp.mid_ranges[t].begin, mr[2 * t + 1] = wp.mid_ranges[t].end;
        }
        if (nb)
            for (size_t k = 0; k < wp.neighbors.size(); ++k) nb[k] = wp.neighbors[k];
    });
}
double splbcu_partition_imbalance(const splbcu_partition* p) { return p->p.load_imbalance_ratio(); }
void splbcu_partition_free(splbcu_partition* p) {
    if (p && !p->borrowed) delete p;
}

int splbcu_sim_create(const splbcu_domain* d, const splbcu_bc* bcs, uint32_t nb, const splbcu_params* pr,
                      splbcu_sim** out) {
    return guard([&] {
        BCSet b;
        for (uint32_t k = 0; k < nb; ++k)
            b.entries.push_back({bcs[k].kind == 0 ? BCSet::Kind::Pressure : BCSet::Kind::Velocity,
                                 to_table(bcs[k].times, bcs[k].values, bcs[k].n_nodes, bcs[k].period)});
        EngineParams p;
        p.tau = pr->tau;
        p.rho0 = pr->rho0;
        p.dt_s = pr->dt_s;
        p.layout = pr->layout == 0 ? Layout::AoS : Layout::SoA;
        p.scheme = pr->scheme == 0 ? Scheme::Push : Scheme::Pull;
        p.sequence = pr->sequence == 0 ? StepSequence::Classic : StepSequence::Reordered;
        p.workers = pr->workers;
        p.capture_period = pr->capture_period;
        p.observe_iolets = pr->observe_iolets != 0;
        p.exchange_timeout_s = pr->exchange_timeout_s;
        auto s = std::make_unique<splbcu_sim>();
        s->s = std::make_unique<Simulation>(d->d, b, p);
        s->dom_n = d->d.n_sites();
        *out = s.release();
    });
}
int splbcu_nccl_unique_id(uint8_t*) {
    g_err = "reference has no NCCL path";
    return SPLBCU_ERR_CONFIG;
}
int splbcu_sim_create_dist(const splbcu_domain*, const splbcu_bc*, uint32_t, const splbcu_params*, int32_t,
                           int32_t, const uint8_t*, splbcu_sim**) {
    g_err = "reference has no NCCL path";
    return SPLBCU_ERR_CONFIG;
}
int splbcu_sim_run(splbcu_sim* s, uint64_t n) {
    return guard([&] { s->s->run(n); });
}
uint64_t splbcu_sim_steps_run(const splbcu_sim* s) { return s->s->steps_run(); }
double splbcu_sim_step_loop_seconds(const splbcu_sim* s) { return s->s->step_loop_seconds(); }
double splbcu_sim_device_loop_seconds(const splbcu_sim* s) { return s->s->step_loop_seconds(); }
int splbcu_sim_snapshot(splbcu_sim* s, double* out) {
    return guard([&] {
        const auto v = s->s->snapshot_fields();
        std::memcpy(out, v.data(), v.size() * 8);
    });
}
int32_t splbcu_sim_n_workers(const splbcu_sim* s) { return int32_t(s->s->assignment().n_workers); }
int32_t splbcu_sim_worker_is_local(const splbcu_sim*, int32_t) { return 1; }
int splbcu_sim_store_shape(const splbcu_sim* s, int32_t w, uint32_t* n, uint32_t* sh) {
    return guard([&] {
        auto& st = const_cast<splbcu_sim*>(s)->s->store(w);
        if (n) *n = st.n_sites;
        if (sh) *sh = st.shared_size;
    });
}
int splbcu_sim_get_f(splbcu_sim* s, int32_t w, int32_t which, double* host) {
    return guard([&] {
        auto& st = s->s->store(w);
        std::memcpy(host, which == 0 ? st.f_old() : st.f_new(), st.total_size() * 8);
    });
}
int splbcu_sim_set_f(splbcu_sim* s, int32_t w, int32_t which, const double* host) {
    return guard([&] {
        auto& st = s->s->store(w);
        std::memcpy(which == 0 ? st.f_old() : st.f_new(), host, st.total_size() * 8);
    });
}
int splbcu_sim_map_shape(const splbcu_sim* s, int32_t w, uint32_t* n, uint32_t* sh, uint32_t* ns) {
    return guard([&] {
        const StreamingMap& m = s->s->map(w);
        if (n) *n = m.n_local;
        if (sh) *sh = m.shared_size;
        if (ns) *ns = uint32_t(m.segments.size());
    });
}
int splbcu_sim_export_map(splbcu_sim* s, int32_t w, uint32_t* dest, uint8_t* op, uint16_t* iol, uint32_t* rd,
                          uint32_t* ss, uint8_t* sd, int32_t* sn, uint32_t* sb, uint32_t* sc) {
    return guard([&] {
        const StreamingMap& m = s->s->map(w);
        for (size_t q = 0; q < m.targets.size(); ++q) {
            if (dest) dest[q] = m.targets[q].dest;
            if (op) op[q] = uint8_t(m.targets[q].op);
            if (iol) iol[q] = m.targets[q].iolet;
        }
        for (size_t k = 0; k < m.recv_dest.size(); ++k) {
            if (rd) rd[k] = m.recv_dest[k];
            if (ss) ss[k] = m.send_src[k].first;
            if (sd) sd[k] = m.send_src[k].second;
        }
        for (size_t k = 0; k < m.segments.size(); ++k) {
            if (sn) sn[k] = m.segments[k].neighbor;
            if (sb) sb[k] = m.segments[k].base;
            if (sc) sc[k] = m.segments[k].count;
        }
    });
}
int splbcu_sim_export_sources(splbcu_sim* s, int32_t w, uint32_t* src, uint8_t* op, uint16_t* iol) {
    return guard([&] {
        const StreamingMap& m = s->s->map(w);
        for (size_t q = 0; q < m.sources.size(); ++q) {
            if (src) src[q] = m.sources[q].src_site;
            if (op) op[q] = uint8_t(m.sources[q].op);
            if (iol) iol[q] = m.sources[q].iolet;
        }
    });
}
const splbcu_partition* splbcu_sim_partition(const splbcu_sim* s) {
    auto* ss = const_cast<splbcu_sim*>(s);
    ss->view.p = s->s->assignment();
    ss->view.borrowed = true;
    return &ss->view;
}
uint64_t splbcu_sim_n_captures(const splbcu_sim* s) { return s->s->cache().captures.size(); }
int splbcu_sim_capture(const splbcu_sim* s, uint64_t k, uint64_t* step, double* f) {
    return guard([&] {
        const Capture& c = s->s->cache().captures.at(k);
        if (step) *step = c.step;
        if (f) std::memcpy(f, c.fields.data(), c.fields.size() * 8);
    });
}
uint64_t splbcu_sim_series_rows(const splbcu_sim* s) { return s->s->series().rows; }
int splbcu_sim_series(const splbcu_sim* s, uint32_t k, double* a, double* b, double* c) {
    return guard([&] {
        const IoletSeries& sr = s->s->series();
        if (a) std::memcpy(a, sr.max_speed.at(k).data(), sr.rows * 8);
        if (b) std::memcpy(b, sr.pressure.at(k).data(), sr.rows * 8);
        if (c) std::memcpy(c, sr.flow.at(k).data(), sr.rows * 8);
    });
}
int splbcu_sim_write_snapshots(const splbcu_sim* s, const char* path) {
    return guard([&] { write_snapshots(s->s->cache(), std::string(path)); });
}
int splbcu_sim_series_csv(const splbcu_sim* s, double dt_s, char* buf, size_t cap, size_t* len) {
    return guard([&] {
        const std::string out = series_csv(s->s->series(), dt_s);
        if (len) *len = out.size();
        if (buf && cap) {
            const size_t n = std::min(cap - 1, out.size());
            std::memcpy(buf, out.data(), n);
            buf[n] = '\0';
        }
    });
}
int splbcu_sim_set_kernel_timing(splbcu_sim*, int32_t) { return 0; }
int splbcu_sim_kernel_stats(const splbcu_sim*, double* a, uint64_t* b, uint64_t* c) {
    if (a) *a = 0;
    if (b) *b = 0;
    if (c) *c = 0;
    return 0;
}
// ---- geometry sources: the reference builds whole domains only ----------------
struct splbcu_source {
    int kind;  // 0 pipe, 1 bifurcation
    int32_t a, b, c, d;
    double vs;
};
int splbcu_source_pipe(int32_t r, int32_t l, double vs, splbcu_source** out) {
    return guard([&] {
        if (r < 2 || l < 4) (void)build_pipe(r, l, vs);  // the reference's own argument check throws
        *out = new splbcu_source{0, r, l, 0, 0, vs};
    });
}
int splbcu_source_bifurcation(int32_t tr, int32_t br, int32_t tl, int32_t bl, double vs, splbcu_source** out) {
    return guard([&] {
        if (tr < 2 || br < 2 || tl < 4 || bl < 4) (void)build_bifurcation(tr, br, tl, bl, vs);
        *out = new splbcu_source{1, tr, br, tl, bl, vs};
    });
}
int splbcu_source_tree(int32_t, int32_t, int32_t, double, double, double, splbcu_source**) {
    g_err = "reference has no tree generator";
    return SPLBCU_ERR_CONFIG;
}
int splbcu_source_channel(int32_t, int32_t, int32_t, double, splbcu_source**) {
    g_err = "reference has no channel generator";
    return SPLBCU_ERR_CONFIG;
}
int splbcu_source_build(const splbcu_source* s, splbcu_domain** out) {
    if (!s) {
        g_err = "null source";
        return SPLBCU_ERR_CONFIG;
    }
    return s->kind == 0 ? splbcu_domain_build_pipe(s->a, s->b, s->vs, out)
                        : splbcu_domain_build_bifurcation(s->a, s->b, s->c, s->d, s->vs, out);
}
int splbcu_source_window(const splbcu_source*, int32_t, int32_t, int32_t*, splbcu_domain**, splbcu_partition**) {
    g_err = "reference has no slab-local construction";
    return SPLBCU_ERR_CONFIG;
}
int splbcu_window_info(const splbcu_domain*, uint64_t*, int32_t*, int32_t*, uint64_t*) {
    g_err = "domain is not a source window";
    return SPLBCU_ERR_CONFIG;
}
void splbcu_source_free(splbcu_source* s) { delete s; }
int splbcu_sim_create_dist_source(const splbcu_source*, const splbcu_bc*, uint32_t, const splbcu_params*, int32_t,
                                  int32_t, const uint8_t*, splbcu_sim**) {
    g_err = "reference has no NCCL path";
    return SPLBCU_ERR_CONFIG;
}
int32_t splbcu_sim_slab_local(const splbcu_sim*) { return 0; }
uint64_t splbcu_sim_series_d2h_bytes(const splbcu_sim*) { return 0; }
uint64_t splbcu_sim_n_sites(const splbcu_sim* s) { return s->dom_n; }

uint64_t splbcu_sim_launch_count(const splbcu_sim*) { return 0; }
int32_t splbcu_sim_bulk_kernel(const splbcu_sim*) { return -1; }
void splbcu_sim_destroy(splbcu_sim* s) { delete s; }

}  // extern "C"
