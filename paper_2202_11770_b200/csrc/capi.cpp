// C-ABI of libsplbcu.so (include/splbcu.h).  Every entry point catches the
// engine's exceptions and maps them to the reference's taxonomy.
#include "splbcu.h"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <memory>
#include <string>

#include "engine.hpp"

using namespace splbcu;

struct splbcu_domain {
    Domain d;
    // set on windows from splbcu_source_window
    bool window = false;
    uint64_t n_global = 0;
    int32_t own_lo = 0, own_hi = -1;
    std::vector<uint64_t> global_index;
};
struct splbcu_source {
    Source s;
};
struct splbcu_partition {
    Partition p;
    bool borrowed = false;
};
struct splbcu_sim {
    std::unique_ptr<Simulation> s;
    splbcu_partition part_view;
};

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return SPLBCU_OK;
    } catch (const Error& e) {
        g_err = e.what();
        return int(e.kind);
    } catch (const std::bad_alloc&) {
        g_err = "out of host memory";
        return SPLBCU_ERR_RUNTIME;
    } catch (const std::exception& e) {
        g_err = e.what();
        return SPLBCU_ERR_RUNTIME;
    }
}

std::vector<IoletGeo> to_geo(const splbcu_iolet* io, uint32_t n) {
    std::vector<IoletGeo> v(n);
    for (uint32_t k = 0; k < n; ++k) {
        v[k].kind = io[k].kind;
        for (int a = 0; a < 3; ++a) v[k].center[a] = io[k].center[a], v[k].normal[a] = io[k].normal[a];
        v[k].radius = io[k].radius;
    }
    return v;
}

Params to_params(const splbcu_params* p) {
    Params q;
    q.tau = p->tau;
    q.rho0 = p->rho0;
    q.dt_s = p->dt_s;
    q.layout = p->layout;
    q.scheme = p->scheme;
    q.sequence = p->sequence;
    q.workers = p->workers;
    q.capture_period = p->capture_period;
    q.observe_iolets = p->observe_iolets != 0;
    q.exchange_timeout_s = p->exchange_timeout_s;
    for (int k = 0; k < p->n_devices; ++k) q.devices.push_back(p->device_ids[k]);
    q.halo_mode = p->halo_mode;
    q.storage = p->storage;
    return q;
}

std::vector<BCEntry> to_bcs(const splbcu_bc* b, uint32_t n) {
    std::vector<BCEntry> v(n);
    for (uint32_t k = 0; k < n; ++k) {
        v[k].kind = b[k].kind;
        v[k].table.t.assign(b[k].times, b[k].times + b[k].n_nodes);
        v[k].table.v.assign(b[k].values, b[k].values + b[k].n_nodes);
        v[k].table.period = b[k].period;
    }
    return v;
}

void check_ptr(const void* p, const char* what) {
    if (!p) config_error(std::string("null ") + what);
}
}  // namespace

extern "C" {

const char* splbcu_last_error(void) { return g_err.c_str(); }
const char* splbcu_version(void) { return "splbcu 0.1 (sm_100a, FP64 D3Q19 push, NCCL halo)"; }

void splbcu_params_default(splbcu_params* p) {
    std::memset(p, 0, sizeof(*p));
    p->tau = 0.9;
    p->rho0 = 1.0;
    p->dt_s = 1.0;
    p->workers = 1;
    p->exchange_timeout_s = 30.0;
}

// ---- lattice helpers -------------------------------------------------------
void splbcu_equilibrium(double rho, const double u[3], double out19[19]) {
    feq_all(rho, u[0], u[1], u[2], out19);
}

int splbcu_moments(const double f[19], double* rho, double u[3]) {
    return guard([&] {
        double r = f[0];
        for (int i = 1; i < kQ; ++i) r += f[i];
        if (!(r > 0.0)) fail(ErrKind::Degenerate, "moments: non-positive density rho=" + std::to_string(r));
        const Macro m = macro_of(f);
        *rho = m.rho;
        u[0] = m.ux;
        u[1] = m.uy;
        u[2] = m.uz;
    });
}

int splbcu_bgk_collide(const double f[19], double tau, double out[19]) {
    return guard([&] {
        if (!(tau > 1.0 / 2.0))
            runtime_error("RelaxationParams: tau must exceed dt/2, got tau=" + std::to_string(tau) +
                          " dt=" + std::to_string(1.0));
        double r = f[0];
        for (int i = 1; i < kQ; ++i) r += f[i];
        if (!(r > 0.0)) fail(ErrKind::Degenerate, "bgk_collide: non-positive density rho=" + std::to_string(r));
        const Macro m = macro_of(f);
        double feq[kQ];
        feq_all(m.rho, m.ux, m.uy, m.uz, feq);
        const double omega = 1.0 / tau;
        for (int i = 0; i < kQ; ++i) out[i] = relax(f[i], feq[i], omega);
    });
}

int splbcu_timetable_at(const double* times, const double* values, uint32_t n, double period, double t,
                        double* out) {
    return guard([&] {
        TimeTable tt;
        tt.t.assign(times, times + n);
        tt.v.assign(values, values + n);
        tt.period = period;
        tt.validate();
        *out = tt.at(t);
    });
}

double splbcu_iolet_weight(const splbcu_iolet* io, const int32_t c[3]) {
    return iolet_weight(io->center, io->normal, io->radius, c[0], c[1], c[2]);
}

// ---- domain ----------------------------------------------------------------
int splbcu_domain_classify(const int32_t* voxels, uint64_t n, const splbcu_iolet* iolets, uint32_t n_io,
                           double voxel_size, splbcu_domain** out) {
    return guard([&] {
        std::vector<int32_t> v(voxels, voxels + 3 * n);
        auto d = std::make_unique<splbcu_domain>();
        d->d = classify_sites(v, to_geo(iolets, n_io), voxel_size);
        *out = d.release();
    });
}

int splbcu_domain_build_pipe(int32_t radius, int32_t length, double vs, splbcu_domain** out) {
    return guard([&] {
        auto d = std::make_unique<splbcu_domain>();
        d->d = build_pipe(radius, length, vs);
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

int splbcu_domain_build_tree(int32_t rr, int32_t rl, int32_t levels, double radius_ratio, double length_ratio,
                             double vs, splbcu_domain** out) {
    return guard([&] {
        auto d = std::make_unique<splbcu_domain>();
        d->d = build_tree(rr, rl, levels, radius_ratio, length_ratio, vs);
        *out = d.release();
    });
}

int splbcu_domain_build_channel(int32_t nx, int32_t ny, int32_t nz, double vs, splbcu_domain** out) {
    return guard([&] {
        auto d = std::make_unique<splbcu_domain>();
        d->d = build_channel(nx, ny, nz, vs);
        *out = d.release();
    });
}

int splbcu_domain_from_arrays(uint64_t n, const int32_t* coords, const uint8_t* types, const uint8_t* link_kind,
                              const uint16_t* link_iolet, const splbcu_iolet* iolets, uint32_t n_io,
                              const uint64_t* type_ranges, double voxel_size, splbcu_domain** out) {
    return guard([&] {
        auto dd = std::make_unique<splbcu_domain>();
        Domain& d = dd->d;
        d.voxel_size = voxel_size;
        d.n = n;
        d.coords.assign(coords, coords + 3 * n);
        d.types.assign(types, types + n);
        d.link_kind.assign(link_kind, link_kind + 18 * n);
        for (uint64_t s = 0; s < n; ++s)
            if (d.types[s] >= 6) geometry_error("geometry load: bad collision type");
        for (uint64_t q = 0; q < 18 * n; ++q) {
            if (d.link_kind[q] > 3) geometry_error("geometry load: bad link tag");
            if (d.link_kind[q] >= 2) {
                d.iolet_link_pos.push_back(q);
                d.iolet_link_id.push_back(link_iolet ? link_iolet[q] : 0);
            }
        }
        d.iolets = to_geo(iolets, n_io);
        for (int t = 0; t < 6; ++t) d.type_ranges[t][0] = type_ranges[2 * t], d.type_ranges[t][1] = type_ranges[2 * t + 1];
        validate_domain(d);
        *out = dd.release();
    });
}

int splbcu_domain_validate(const splbcu_domain* d) {
    return guard([&] {
        check_ptr(d, "domain");
        validate_domain(d->d);
    });
}

int splbcu_domain_read(const char* path, splbcu_domain** out) {
    return guard([&] {
        auto d = std::make_unique<splbcu_domain>();
        d->d = read_domain(path);
        *out = d.release();
    });
}

int splbcu_domain_write(const splbcu_domain* d, const char* path) {
    return guard([&] { write_domain(d->d, path); });
}

uint64_t splbcu_domain_n_sites(const splbcu_domain* d) { return d ? d->d.n : 0; }
uint32_t splbcu_domain_n_iolets(const splbcu_domain* d) { return d ? uint32_t(d->d.iolets.size()) : 0; }
double splbcu_domain_voxel_size(const splbcu_domain* d) { return d ? d->d.voxel_size : 0.0; }

int splbcu_domain_export(const splbcu_domain* dd, int32_t* coords, uint8_t* types, uint8_t* link_kind,
                         uint16_t* link_iolet, splbcu_iolet* iolets, uint64_t* type_ranges) {
    return guard([&] {
        check_ptr(dd, "domain");
        const Domain& d = dd->d;
        if (coords) std::memcpy(coords, d.coords.data(), d.coords.size() * 4);
        if (types) std::memcpy(types, d.types.data(), d.n);
        if (link_kind) std::memcpy(link_kind, d.link_kind.data(), 18 * d.n);
        if (link_iolet) {
            std::memset(link_iolet, 0, 18 * d.n * 2);
            for (size_t q = 0; q < d.iolet_link_pos.size(); ++q) link_iolet[d.iolet_link_pos[q]] = d.iolet_link_id[q];
        }
        if (iolets)
            for (size_t k = 0; k < d.iolets.size(); ++k) {
                iolets[k].kind = d.iolets[k].kind;
                for (int a = 0; a < 3; ++a)
                    iolets[k].center[a] = d.iolets[k].center[a], iolets[k].normal[a] = d.iolets[k].normal[a];
                iolets[k].radius = d.iolets[k].radius;
            }
        if (type_ranges)
            for (int t = 0; t < 6; ++t) type_ranges[2 * t] = d.type_ranges[t][0], type_ranges[2 * t + 1] = d.type_ranges[t][1];
    });
}

void splbcu_domain_free(splbcu_domain* d) { delete d; }

// ---- sources -------------------------------------------------------------------
static int make_source(splbcu_source** out, const std::function<Source()>& f) {
    return guard([&] {
        auto p = std::make_unique<splbcu_source>();
        p->s = f();
        *out = p.release();
    });
}
int splbcu_source_pipe(int32_t radius, int32_t length, double voxel_size, splbcu_source** out) {
    return make_source(out, [&] { return source_pipe(radius, length, voxel_size); });
}
int splbcu_source_bifurcation(int32_t tr, int32_t br, int32_t tl, int32_t bl, double voxel_size,
                              splbcu_source** out) {
    return make_source(out, [&] { return source_bifurcation(tr, br, tl, bl, voxel_size); });
}
int splbcu_source_tree(int32_t root_radius, int32_t root_length, int32_t levels, double radius_ratio,
                       double length_ratio, double voxel_size, splbcu_source** out) {
    return make_source(out, [&] {
        return source_tree(root_radius, root_length, levels, radius_ratio, length_ratio, voxel_size);
    });
}
int splbcu_source_channel(int32_t nx, int32_t ny, int32_t nz, double voxel_size, splbcu_source** out) {
    return make_source(out, [&] { return source_channel(nx, ny, nz, voxel_size); });
}
int splbcu_source_build(const splbcu_source* s, splbcu_domain** out) {
    return guard([&] {
        check_ptr(s, "source");
        auto d = std::make_unique<splbcu_domain>();
        d->d = build_from_source(s->s);
        *out = d.release();
    });
}
int splbcu_source_window(const splbcu_source* s, int32_t n_workers, int32_t worker, int32_t* slab,
                         splbcu_domain** window, splbcu_partition** part) {
    return guard([&] {
        check_ptr(s, "source");
        if (worker < 0 || worker >= n_workers) config_error("source window: worker out of range");
        const SlabPlan plan = plan_slabs(plan_source(s->s), s->s.z0, n_workers);
        if (slab) *slab = plan.ok ? 1 : 0;
        if (!plan.ok) return;
        // every worker's own-slice counts, as the ranks' all-gather provides them
        std::vector<uint64_t> counts;
        Window mine;
        for (int v = 0; v < n_workers; ++v) {
            std::vector<uint64_t> own;
            Window w = classify_window(s->s, plan, v, &own, nullptr);
            counts.insert(counts.end(), own.begin(), own.end());
            if (v == worker) mine = std::move(w);
        }
        finish_window(mine, plan, counts);
        if (part) {
            auto p = std::make_unique<splbcu_partition>();
            p->p = partition_window(mine, plan, n_workers);
            *part = p.release();
        }
        if (window) {
            auto d = std::make_unique<splbcu_domain>();
            d->window = true;
            d->n_global = mine.n_global;
            d->own_lo = mine.own_lo;
            d->own_hi = mine.own_hi;
            d->global_index.resize(mine.dom.n);
            for (uint64_t q = 0; q < mine.dom.n; ++q) d->global_index[q] = mine.global_of(q);
            d->d = std::move(mine.dom);
            *window = d.release();
        }
    });
}
int splbcu_window_info(const splbcu_domain* w, uint64_t* n_global, int32_t* own_lo, int32_t* own_hi,
                       uint64_t* global_index) {
    return guard([&] {
        check_ptr(w, "domain");
        if (!w->window) config_error("domain is not a source window");
        if (n_global) *n_global = w->n_global;
        if (own_lo) *own_lo = w->own_lo;
        if (own_hi) *own_hi = w->own_hi;
        if (global_index) std::memcpy(global_index, w->global_index.data(), w->global_index.size() * 8);
    });
}
void splbcu_source_free(splbcu_source* s) { delete s; }

// ---- partition --------------------------------------------------------------
int splbcu_partition_create(const splbcu_domain* d, int32_t n_workers, splbcu_partition** out) {
    return guard([&] {
        check_ptr(d, "domain");
        auto p = std::make_unique<splbcu_partition>();
        p->p = partition(d->d, n_workers);
        *out = p.release();
    });
}

int splbcu_partition_global(const splbcu_partition* p, int32_t* owner, uint32_t* local_index) {
    return guard([&] {
        check_ptr(p, "partition");
        if (owner) std::memcpy(owner, p->p.owner.data(), p->p.owner.size() * 4);
        if (local_index) std::memcpy(local_index, p->p.local_index.data(), p->p.local_index.size() * 4);
    });
}

int splbcu_partition_part_shape(const splbcu_partition* p, int32_t w, uint32_t* n_sites, uint32_t* n_edge,
                                uint32_t* n_nb) {
    return guard([&] {
        check_ptr(p, "partition");
        if (w < 0 || w >= p->p.n_workers) config_error("partition: worker out of range");
        const WorkerPart& wp = p->p.parts[size_t(w)];
        if (n_sites) *n_sites = uint32_t(wp.sites.size());
        if (n_edge) *n_edge = wp.n_edge;
        if (n_nb) *n_nb = uint32_t(wp.neighbors.size());
    });
}

int splbcu_partition_part(const splbcu_partition* p, int32_t w, uint32_t* sites, uint64_t* edge_ranges,
                          uint64_t* mid_ranges, int32_t* neighbors) {
    return guard([&] {
        check_ptr(p, "partition");
        if (w < 0 || w >= p->p.n_workers) config_error("partition: worker out of range");
        const WorkerPart& wp = p->p.parts[size_t(w)];
        if (sites) std::memcpy(sites, wp.sites.data(), wp.sites.size() * 4);
        for (int t = 0; t < 6; ++t) {
            if (edge_ranges) edge_ranges[2 * t] = wp.edge_ranges[t][0], edge_ranges[2 * t + 1] = wp.edge_ranges[t][1];
            if (mid_ranges) mid_ranges[2 * t] = wp.mid_ranges[t][0], mid_ranges[2 * t + 1] = wp.mid_ranges[t][1];
        }
        if (neighbors)
            for (size_t k = 0; k < wp.neighbors.size(); ++k) neighbors[k] = wp.neighbors[k];
    });
}

double splbcu_partition_imbalance(const splbcu_partition* p) { return p ? p->p.imbalance() : 0.0; }
void splbcu_partition_free(splbcu_partition* p) {
    if (p && !p->borrowed) delete p;
}

// ---- simulation -------------------------------------------------------------
int splbcu_sim_create(const splbcu_domain* d, const splbcu_bc* bcs, uint32_t n_bcs, const splbcu_params* params,
                      splbcu_sim** out) {
    return guard([&] {
        check_ptr(d, "domain");
        check_ptr(params, "params");
        auto s = std::make_unique<splbcu_sim>();
        s->s = std::make_unique<Simulation>(d->d, to_bcs(bcs, n_bcs), to_params(params));
        *out = s.release();
    });
}

int splbcu_nccl_unique_id(uint8_t out[128]) {
    return guard([&] { nccl_unique_id(out); });
}

int splbcu_sim_create_dist(const splbcu_domain* d, const splbcu_bc* bcs, uint32_t n_bcs, const splbcu_params* params,
                           int32_t rank, int32_t nranks, const uint8_t id[128], splbcu_sim** out) {
    return guard([&] {
        check_ptr(d, "domain");
        check_ptr(params, "params");
        check_ptr(id, "nccl id");
        auto s = std::make_unique<splbcu_sim>();
        s->s = std::make_unique<Simulation>(d->d, to_bcs(bcs, n_bcs), to_params(params), rank, nranks, id);
        *out = s.release();
    });
}

int splbcu_sim_create_dist_source(const splbcu_source* src, const splbcu_bc* bcs, uint32_t n_bcs,
                                  const splbcu_params* params, int32_t rank, int32_t nranks, const uint8_t id[128],
                                  splbcu_sim** out) {
    return guard([&] {
        check_ptr(src, "source");
        check_ptr(params, "params");
        check_ptr(id, "nccl id");
        auto s = std::make_unique<splbcu_sim>();
        s->s = std::make_unique<Simulation>(src->s, to_bcs(bcs, n_bcs), to_params(params), rank, nranks, id);
        *out = s.release();
    });
}
uint64_t splbcu_sim_series_d2h_bytes(const splbcu_sim* s) { return s ? s->s->series_d2h_bytes() : 0; }
int32_t splbcu_sim_slab_local(const splbcu_sim* s) { return s && s->s->slab_local() ? 1 : 0; }
uint64_t splbcu_sim_n_sites(const splbcu_sim* s) { return s ? s->s->n_sites() : 0; }

int splbcu_sim_run(splbcu_sim* s, uint64_t n) {
    return guard([&] {
        check_ptr(s, "simulation");
        s->s->run(n);
    });
}
uint64_t splbcu_sim_steps_run(const splbcu_sim* s) { return s ? s->s->steps_run() : 0; }
double splbcu_sim_step_loop_seconds(const splbcu_sim* s) { return s ? s->s->step_loop_seconds() : 0.0; }
double splbcu_sim_device_loop_seconds(const splbcu_sim* s) { return s ? s->s->device_loop_seconds() : 0.0; }

int splbcu_sim_snapshot(splbcu_sim* s, double* out) {
    return guard([&] {
        check_ptr(s, "simulation");
        s->s->snapshot(out);
    });
}
int32_t splbcu_sim_n_workers(const splbcu_sim* s) { return s ? s->s->n_workers() : 0; }
int32_t splbcu_sim_worker_is_local(const splbcu_sim* s, int32_t w) { return s && s->s->is_local(w) ? 1 : 0; }

int splbcu_sim_store_shape(const splbcu_sim* s, int32_t w, uint32_t* n, uint32_t* shared) {
    return guard([&] {
        check_ptr(s, "simulation");
        s->s->store_shape(w, n, shared);
    });
}
int splbcu_sim_get_f(splbcu_sim* s, int32_t w, int32_t which, double* host) {
    return guard([&] {
        check_ptr(s, "simulation");
        s->s->get_f(w, which, host);
    });
}
int splbcu_sim_set_f(splbcu_sim* s, int32_t w, int32_t which, const double* host) {
    return guard([&] {
        check_ptr(s, "simulation");
        s->s->set_f(w, which, host);
    });
}

int splbcu_sim_map_shape(const splbcu_sim* s, int32_t w, uint32_t* n_local, uint32_t* shared, uint32_t* n_seg) {
    return guard([&] {
        check_ptr(s, "simulation");
        uint32_t n = 0, sh = 0;
        s->s->store_shape(w, &n, &sh);
        if (n_local) *n_local = n;
        if (shared) *shared = sh;
        if (n_seg) *n_seg = uint32_t(s->s->partition().parts[size_t(w)].neighbors.size());
    });
}

int splbcu_sim_export_map(splbcu_sim* s, int32_t w, uint32_t* dest, uint8_t* op, uint16_t* iolet,
                          uint32_t* recv_dest, uint32_t* send_site, uint8_t* send_dir, int32_t* seg_nb,
                          uint32_t* seg_base, uint32_t* seg_count) {
    return guard([&] {
        check_ptr(s, "simulation");
        const ExportedMap m = s->s->export_map(w);
        if (dest) std::memcpy(dest, m.dest.data(), m.dest.size() * 4);
        if (op) std::memcpy(op, m.op.data(), m.op.size());
        if (iolet) std::memcpy(iolet, m.iolet.data(), m.iolet.size() * 2);
        if (recv_dest) std::memcpy(recv_dest, m.recv_dest.data(), m.recv_dest.size() * 4);
        if (send_site) std::memcpy(send_site, m.send_site.data(), m.send_site.size() * 4);
        if (send_dir) std::memcpy(send_dir, m.send_dir.data(), m.send_dir.size());
        for (size_t k = 0; k < m.seg_neighbor.size(); ++k) {
            if (seg_nb) seg_nb[k] = m.seg_neighbor[k];
            if (seg_base) seg_base[k] = m.seg_base[k];
            if (seg_count) seg_count[k] = m.seg_count[k];
        }
    });
}

int splbcu_sim_export_sources(splbcu_sim* s, int32_t w, uint32_t* src_site, uint8_t* op, uint16_t* iolet) {
    return guard([&] {
        check_ptr(s, "simulation");
        const ExportedMap m = s->s->export_map(w);
        if (src_site) std::memcpy(src_site, m.src_site.data(), m.src_site.size() * 4);
        if (op) std::memcpy(op, m.src_op.data(), m.src_op.size());
        if (iolet) std::memcpy(iolet, m.src_iolet.data(), m.src_iolet.size() * 2);
    });
}

const splbcu_partition* splbcu_sim_partition(const splbcu_sim* s) {
    if (!s || s->s->slab_local()) return nullptr;
    auto* ss = const_cast<splbcu_sim*>(s);
    ss->part_view.p = s->s->partition();
    ss->part_view.borrowed = true;
    return &ss->part_view;
}

uint64_t splbcu_sim_n_captures(const splbcu_sim* s) { return s ? s->s->captures().size() : 0; }
int splbcu_sim_capture(const splbcu_sim* s, uint64_t k, uint64_t* step, double* fields) {
    return guard([&] {
        check_ptr(s, "simulation");
        const auto& c = s->s->captures();
        if (k >= c.size()) config_error("capture index out of range");
        if (step) *step = c[k].step;
        if (fields) std::memcpy(fields, c[k].fields.data(), c[k].fields.size() * 8);
    });
}

// The series accessor completes the pending host reduction (it can
// allocate): guarded like every other entry, 0 with the error recorded.
uint64_t splbcu_sim_series_rows(const splbcu_sim* s) {
    uint64_t rows = 0;
    if (guard([&] {
            check_ptr(s, "simulation");
            rows = s->s->series().rows;
        }) != SPLBCU_OK)
        return 0;
    return rows;
}
int splbcu_sim_series(const splbcu_sim* s, uint32_t k, double* max_speed, double* pressure, double* flow) {
    return guard([&] {
        check_ptr(s, "simulation");
        const Series& sr = s->s->series();
        if (k >= sr.max_speed.size()) config_error("series: iolet out of range");
        if (max_speed) std::memcpy(max_speed, sr.max_speed[k].data(), sr.max_speed[k].size() * 8);
        if (pressure) std::memcpy(pressure, sr.pressure[k].data(), sr.pressure[k].size() * 8);
        if (flow) std::memcpy(flow, sr.flow[k].data(), sr.flow[k].size() * 8);
    });
}

// write_snapshots (snapshot.hpp:15-29)
int splbcu_sim_write_snapshots(const splbcu_sim* s, const char* path) {
    return guard([&] {
        check_ptr(s, "simulation");
        std::FILE* f = std::fopen(path, "wb");
        if (!f) runtime_error(std::string("snapshot write: cannot open ") + path);
        bool ok = true;
        for (const Capture& c : s->s->captures()) {
            ok &= std::fwrite(&c.step, sizeof(uint64_t), 1, f) == 1;
            ok &= std::fwrite(c.fields.data(), sizeof(double), c.fields.size(), f) == c.fields.size();
        }
        ok &= std::fclose(f) == 0;
        if (!ok) runtime_error("snapshot write: stream failure");
    });
}

// series_csv (snapshot.hpp:59-82)
int splbcu_sim_series_csv(const splbcu_sim* s, double dt_s, char* buf, size_t cap, size_t* len) {
    return guard([&] {
        check_ptr(s, "simulation");
        const Series& sr = s->s->series();
        std::string out = "step,time_s";
        char b[256];
        for (size_t k = 0; k < sr.max_speed.size(); ++k) {
            std::snprintf(b, sizeof b, ",iolet%zu_max_speed,iolet%zu_pressure,iolet%zu_flow", k, k, k);
            out += b;
        }
        out += '\n';
        for (uint64_t row = 0; row < sr.rows; ++row) {
            std::snprintf(b, sizeof b, "%llu,%.17g", (unsigned long long)row, double(row) * dt_s);
            out += b;
            for (size_t k = 0; k < sr.max_speed.size(); ++k) {
                std::snprintf(b, sizeof b, ",%.17g,%.17g,%.17g", sr.max_speed[k][row], sr.pressure[k][row],
                              sr.flow[k][row]);
                out += b;
            }
            out += '\n';
        }
        if (len) *len = out.size();
        if (buf && cap) {
            const size_t n = std::min(cap - 1, out.size());
            std::memcpy(buf, out.data(), n);
            buf[n] = '\0';
        }
    });
}

int splbcu_sim_set_kernel_timing(splbcu_sim* s, int32_t on) {
    return guard([&] {
        check_ptr(s, "simulation");
        s->s->set_kernel_timing(on != 0);
    });
}

int splbcu_sim_kernel_stats(const splbcu_sim* s, double* secs, uint64_t* launches, uint64_t* sites) {
    return guard([&] {
        check_ptr(s, "simulation");
        if (secs) *secs = s->s->plain_kernel_seconds();
        if (launches) *launches = s->s->plain_kernel_launches();
        if (sites) *sites = s->s->plain_kernel_sites();
    });
}

uint64_t splbcu_sim_launch_count(const splbcu_sim* s) { return s ? s->s->launch_count() : 0; }

int32_t splbcu_sim_bulk_kernel(const splbcu_sim* s) { return s ? s->s->bulk_kernel() : -1; }

void splbcu_sim_destroy(splbcu_sim* s) { delete s; }

}  // extern "C"
