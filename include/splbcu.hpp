// splbcu.hpp — the reference's C++ surface (namespace splb, header-only)
// rebuilt over the C-ABI in splbcu.h.
//
// A C++ caller of the reference (proj/include/splb/engine.hpp:121-205) swaps
//   #include "splb/engine.hpp"   ->   #include "splbcu.hpp"
// and links libsplbcu.so.  Class names, argument meaning and exception types
// follow the reference (common.hpp:11-28, geometry.hpp:64-363,
// decomp.hpp:16-188, boundary.hpp:18-74, engine.hpp:37-205); the time step runs
// in the B200 kernels behind the C-ABI.  Differences: SparseDomain is an
// opaque owner of the site arrays (export() copies them out), and store(w)
// is a host mirror of the HBM-resident populations that the simulation keeps
// coherent (fetched on read, written back before its next operation).
#pragma once

#include <array>
#include <cstdint>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "splbcu.h"

namespace splb {

struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct DegenerateState : Error {
    using Error::Error;
};
struct GeometryError : Error {
    using Error::Error;
};
struct ConfigError : Error {
    using Error::Error;
};

namespace detail {
inline void check(int rc) {
    if (rc == SPLBCU_OK) return;
    const std::string m = splbcu_last_error();
    switch (rc) {
        case SPLBCU_ERR_CONFIG: throw ConfigError(m);
        case SPLBCU_ERR_GEOMETRY: throw GeometryError(m);
        case SPLBCU_ERR_DEGENERATE: throw DegenerateState(m);
        default: throw Error(m);
    }
}
}  // namespace detail

using Vec3 = std::array<double, 3>;
using Vec3i = std::array<int32_t, 3>;

enum class Layout : uint8_t { AoS = 0, SoA = 1 };
enum class Scheme : uint8_t { Push = 0, Pull = 1 };
enum class StepSequence : uint8_t { Classic = 0, Reordered = 1 };

struct Iolet {
    enum class Kind : uint8_t { Inlet = 0, Outlet = 1 };
    Kind kind;
    Vec3 center;
    Vec3 normal;
    double radius;
};

// boundary.hpp:18-74
struct TimeTable {
    std::vector<std::pair<double, double>> nodes;
    double period = 0.0;
    static TimeTable constant(double v) { return TimeTable{{{0.0, v}}, 0.0}; }
    double at(double t) const {
        std::vector<double> ts, vs;
        for (auto& n : nodes) ts.push_back(n.first), vs.push_back(n.second);
        double out = 0.0;
        detail::check(splbcu_timetable_at(ts.data(), vs.data(), uint32_t(ts.size()), period, t, &out));
        return out;
    }
};

// engine.hpp:37-44
struct BCSet {
    enum class Kind : uint8_t { Pressure = 0, Velocity = 1 };
    struct Entry {
        Kind kind = Kind::Pressure;
        TimeTable table;
    };
    std::vector<Entry> entries;
};

// engine.hpp:46-57 (+ device placement)
struct EngineParams {
    double tau = 0.9;
    double rho0 = 1.0;
    double dt_s = 1.0;
    Layout layout = Layout::AoS;
    Scheme scheme = Scheme::Push;
    StepSequence sequence = StepSequence::Classic;
    int workers = 1;
    uint64_t capture_period = 0;
    bool observe_iolets = false;
    double exchange_timeout_s = 30.0;
    std::vector<int32_t> devices;  // B200: workers placed round robin
    int32_t halo_mode = 0;         // B200: 0 NCCL/peer copies, 1 fused NVLink P2P stores
    int32_t storage = 0;           // B200: 0 two buffers (push), 1 single buffer (AA pattern)
};

// geometry.hpp:64-73 (opaque; site arrays on demand)
class SparseDomain {
  public:
    explicit SparseDomain(splbcu_domain* h) : h_(h, &splbcu_domain_free) {}
    uint64_t n_sites() const { return splbcu_domain_n_sites(h_.get()); }
    double voxel_size() const { return splbcu_domain_voxel_size(h_.get()); }
    splbcu_domain* handle() const { return h_.get(); }
    void validate() const { detail::check(splbcu_domain_validate(h_.get())); }
    void write(const std::string& path) const { detail::check(splbcu_domain_write(h_.get(), path.c_str())); }
    static SparseDomain read(const std::string& path) {
        splbcu_domain* d = nullptr;
        detail::check(splbcu_domain_read(path.c_str(), &d));
        return SparseDomain(d);
    }

  private:
    std::shared_ptr<splbcu_domain> h_;
};

inline splbcu_iolet to_c(const Iolet& io) {
    splbcu_iolet c{};
    c.kind = int32_t(io.kind);
    for (int a = 0; a < 3; ++a) c.center[a] = io.center[a], c.normal[a] = io.normal[a];
    c.radius = io.radius;
    return c;
}

// geometry.hpp:139-208
inline SparseDomain classify_sites(const std::vector<Vec3i>& voxels, const std::vector<Iolet>& iolets,
                                   double voxel_size = 1.0) {
    std::vector<splbcu_iolet> io;
    for (auto& i : iolets) io.push_back(to_c(i));
    splbcu_domain* d = nullptr;
    detail::check(splbcu_domain_classify(reinterpret_cast<const int32_t*>(voxels.data()), voxels.size(), io.data(),
                                         uint32_t(io.size()), voxel_size, &d));
    return SparseDomain(d);
}
// geometry.hpp:285-308
inline SparseDomain build_pipe(int radius, int length, double voxel_size = 1.0) {
    splbcu_domain* d = nullptr;
    detail::check(splbcu_domain_build_pipe(radius, length, voxel_size, &d));
    return SparseDomain(d);
}
// geometry.hpp:313-363
inline SparseDomain build_bifurcation(int tr, int br, int tl, int bl, double voxel_size = 1.0) {
    splbcu_domain* d = nullptr;
    detail::check(splbcu_domain_build_bifurcation(tr, br, tl, bl, voxel_size, &d));
    return SparseDomain(d);
}

// Geometry source (include/splbcu.h "geometry sources"): a generator evaluated
// slice by slice; build() is the whole domain, Simulation::distributed(source,
// ...) classifies only each rank's slab.
class Source {
  public:
    explicit Source(splbcu_source* h) : h_(h, &splbcu_source_free) {}
    static Source pipe(int radius, int length, double voxel_size = 1.0) {
        splbcu_source* s = nullptr;
        detail::check(splbcu_source_pipe(radius, length, voxel_size, &s));
        return Source(s);
    }
    static Source bifurcation(int tr, int br, int tl, int bl, double voxel_size = 1.0) {
        splbcu_source* s = nullptr;
        detail::check(splbcu_source_bifurcation(tr, br, tl, bl, voxel_size, &s));
        return Source(s);
    }
    static Source tree(int root_radius, int root_length, int levels, double radius_ratio = 0.8,
                       double length_ratio = 0.8, double voxel_size = 1.0) {
        splbcu_source* s = nullptr;
        detail::check(splbcu_source_tree(root_radius, root_length, levels, radius_ratio, length_ratio, voxel_size, &s));
        return Source(s);
    }
    static Source channel(int nx, int ny, int nz, double voxel_size = 1.0) {
        splbcu_source* s = nullptr;
        detail::check(splbcu_source_channel(nx, ny, nz, voxel_size, &s));
        return Source(s);
    }
    SparseDomain build() const {
        splbcu_domain* d = nullptr;
        detail::check(splbcu_source_build(h_.get(), &d));
        return SparseDomain(d);
    }
    splbcu_source* handle() const { return h_.get(); }

  private:
    std::shared_ptr<splbcu_source> h_;
};

struct Capture {
    uint64_t step = 0;
    std::vector<double> fields;  // 4 * nSites, (rho, ux, uy, uz) in domain order
};
struct PropertyCache {
    uint64_t capture_period = 0;
    std::vector<Capture> captures;
};
struct IoletSeries {
    uint64_t rows = 0;
    std::vector<std::vector<double>> max_speed, pressure, flow;
};

// store(w) (layout.hpp:19-62, engine.hpp:149): worker w's two f buffers in
// the reference layout.  The populations live in HBM, so the object the
// simulation hands out is a host mirror kept coherent with the device: it is
// fetched when first read after a step, and pointers taken through f_old() /
// f_new() may be written — the simulation writes the mirror back before its
// next operation (run, snapshot_fields, cache, series), as the reference's
// mutable DistributionStore& would be seen.  A copy (DistributionStore s =
// sim.store(w)) is a detached snapshot; set_f_old/set_f_new write it back.
class Simulation;
struct DistributionStore {
    Layout layout = Layout::AoS;
    uint32_t n_sites = 0, shared_size = 0;

    DistributionStore() = default;
    DistributionStore(const DistributionStore& o) { *this = o; }
    DistributionStore& operator=(const DistributionStore& o) {
        if (this == &o) return *this;
        o.sync_();
        layout = o.layout, n_sites = o.n_sites, shared_size = o.shared_size;
        old_ = o.old_, new_ = o.new_;
        h_ = nullptr, fresh_ = true, dirty_ = false;  // detached
        return *this;
    }
    size_t idx(uint32_t s, int i) const {
        return layout == Layout::AoS ? size_t(19) * s + size_t(i) : size_t(i) * n_sites + s;
    }
    size_t shared_base() const { return size_t(19) * n_sites; }
    size_t total_size() const { return shared_base() + shared_size; }
    double* f_old() {
        sync_();
        dirty_ = true;
        return old_.data();
    }
    double* f_new() {
        sync_();
        dirty_ = true;
        return new_.data();
    }
    const double* f_old() const {
        sync_();
        return old_.data();
    }
    const double* f_new() const {
        sync_();
        return new_.data();
    }

  private:
    friend class Simulation;
    mutable std::vector<double> old_, new_;
    splbcu_sim* h_ = nullptr;  // owning simulation (null: detached copy)
    int w_ = 0;
    mutable bool fresh_ = true;
    bool dirty_ = false;
    void sync_() const {
        if (h_ && !fresh_) {
            detail::check(splbcu_sim_get_f(h_, w_, 0, old_.data()));
            detail::check(splbcu_sim_get_f(h_, w_, 1, new_.data()));
            fresh_ = true;
        }
    }
    void write_back_() {
        if (h_ && dirty_) {
            detail::check(splbcu_sim_set_f(h_, w_, 0, old_.data()));
            detail::check(splbcu_sim_set_f(h_, w_, 1, new_.data()));
        }
        dirty_ = false;
    }
};

// engine.hpp:121-205
class Simulation {
    // BCSet + EngineParams in C form (the arrays stay alive for the create call)
    struct CArgs {
        std::vector<std::vector<double>> keep;
        std::vector<splbcu_bc> bc;
        splbcu_params c;
        CArgs(const BCSet& bcs, const EngineParams& p) {
            for (auto& e : bcs.entries) {
                std::vector<double> t, v;
                for (auto& n : e.table.nodes) t.push_back(n.first), v.push_back(n.second);
                keep.push_back(std::move(t));
                keep.push_back(std::move(v));
                bc.push_back({int32_t(e.kind), keep[keep.size() - 2].data(), keep.back().data(),
                              uint32_t(e.table.nodes.size()), e.table.period});
            }
            splbcu_params_default(&c);
            c.tau = p.tau, c.rho0 = p.rho0, c.dt_s = p.dt_s;
            c.layout = int32_t(p.layout), c.scheme = int32_t(p.scheme), c.sequence = int32_t(p.sequence);
            c.workers = p.workers, c.capture_period = p.capture_period, c.observe_iolets = p.observe_iolets;
            c.exchange_timeout_s = p.exchange_timeout_s;
            c.halo_mode = p.halo_mode;
            c.storage = p.storage;
            c.n_devices = int32_t(p.devices.size());
            c.device_ids = p.devices.data();
        }
    };
    Simulation(std::shared_ptr<SparseDomain> d, const EngineParams& p, uint32_t n_io, splbcu_sim* s)
        : domain_(std::move(d)), params_(p), n_io_(n_io), h_(s) {}

  public:
    Simulation(const SparseDomain& domain, const BCSet& bcs, const EngineParams& p)
        : domain_(std::make_shared<SparseDomain>(domain)), params_(p), n_io_(uint32_t(bcs.entries.size())) {
        CArgs a(bcs, p);
        splbcu_sim* s = nullptr;
        detail::check(splbcu_sim_create(domain.handle(), a.bc.data(), uint32_t(a.bc.size()), &a.c, &s));
        h_.reset(s);
    }

    // One process per GPU (B200; no reference equivalent): this process owns
    // worker `rank` of p.workers == nranks on p.devices[0]; nccl_id = 128
    // bytes from nccl_unique_id() on rank 0, broadcast by the caller.
    static void nccl_unique_id(uint8_t out[128]) { detail::check(splbcu_nccl_unique_id(out)); }
    static Simulation distributed(const SparseDomain& domain, const BCSet& bcs, const EngineParams& p, int rank,
                                  int nranks, const uint8_t nccl_id[128]) {
        CArgs a(bcs, p);
        splbcu_sim* s = nullptr;
        detail::check(splbcu_sim_create_dist(domain.handle(), a.bc.data(), uint32_t(a.bc.size()), &a.c, rank,
                                             nranks, nccl_id, &s));
        return Simulation(std::make_shared<SparseDomain>(domain), p, uint32_t(bcs.entries.size()), s);
    }
    // ... over a geometry source: each rank classifies only its own slab.
    static Simulation distributed(const Source& src, const BCSet& bcs, const EngineParams& p, int rank, int nranks,
                                  const uint8_t nccl_id[128]) {
        CArgs a(bcs, p);
        splbcu_sim* s = nullptr;
        detail::check(splbcu_sim_create_dist_source(src.handle(), a.bc.data(), uint32_t(a.bc.size()), &a.c, rank,
                                                    nranks, nccl_id, &s));
        return Simulation(nullptr, p, uint32_t(bcs.entries.size()), s);
    }

    void run(uint64_t n_steps) {
        flush_stores_();
        detail::check(splbcu_sim_run(h_.get(), n_steps));
        stale_stores_();
    }
    uint64_t steps_run() const { return splbcu_sim_steps_run(h_.get()); }
    double step_loop_seconds() const { return splbcu_sim_step_loop_seconds(h_.get()); }
    uint64_t n_sites() const { return splbcu_sim_n_sites(h_.get()); }
    bool slab_local() const { return splbcu_sim_slab_local(h_.get()) != 0; }
    const SparseDomain& domain() const {
        if (!domain_) throw Error("domain(): a slab-local simulation holds no whole domain");
        return *domain_;
    }

    std::vector<double> snapshot_fields() const {
        flush_stores_();
        std::vector<double> out(4 * n_sites());
        detail::check(splbcu_sim_snapshot(h_.get(), out.data()));
        return out;
    }

    // store(w) (engine.hpp:149): the mutable view described at DistributionStore.
    DistributionStore& store(int w) {
        std::unique_ptr<DistributionStore>& m = stores_[w];
        if (!m) {
            auto st = std::make_unique<DistributionStore>();
            st->layout = params_.layout;
            detail::check(splbcu_sim_store_shape(h_.get(), w, &st->n_sites, &st->shared_size));
            st->old_.resize(st->total_size());
            st->new_.resize(st->total_size());
            st->h_ = h_.get();
            st->w_ = w;
            st->fresh_ = false;
            m = std::move(st);
        }
        return *m;
    }
    void set_f_old(int w, const DistributionStore& st) {
        flush_stores_();
        detail::check(splbcu_sim_set_f(h_.get(), w, 0, st.f_old()));
        stale_stores_();
    }
    void set_f_new(int w, const DistributionStore& st) {
        flush_stores_();
        detail::check(splbcu_sim_set_f(h_.get(), w, 1, st.f_new()));
        stale_stores_();
    }

    PropertyCache cache() const {
        flush_stores_();
        PropertyCache c;
        c.capture_period = params_.capture_period;
        const uint64_t n = splbcu_sim_n_captures(h_.get());
        for (uint64_t k = 0; k < n; ++k) {
            Capture cap;
            cap.fields.resize(4 * n_sites());
            detail::check(splbcu_sim_capture(h_.get(), k, &cap.step, cap.fields.data()));
            c.captures.push_back(std::move(cap));
        }
        return c;
    }

    IoletSeries series() const {
        flush_stores_();
        IoletSeries s;
        s.rows = splbcu_sim_series_rows(h_.get());
        if (!s.rows) return s;
        for (uint32_t k = 0; k < n_io_; ++k) {
            std::vector<double> a(s.rows), b(s.rows), c(s.rows);
            detail::check(splbcu_sim_series(h_.get(), k, a.data(), b.data(), c.data()));
            s.max_speed.push_back(std::move(a));
            s.pressure.push_back(std::move(b));
            s.flow.push_back(std::move(c));
        }
        return s;
    }

  private:
    struct Del {
        void operator()(splbcu_sim* s) const { splbcu_sim_destroy(s); }
    };
    // user writes through store(w) reach the device before the next operation;
    // after a step the mirrors are refetched on their next read
    void flush_stores_() const {
        for (auto& kv : stores_) kv.second->write_back_();
    }
    void stale_stores_() const {
        for (auto& kv : stores_) kv.second->fresh_ = false;
    }
    std::shared_ptr<SparseDomain> domain_;  // null when slab-local
    mutable std::map<int, std::unique_ptr<DistributionStore>> stores_;
    EngineParams params_;
    uint32_t n_io_ = 0;
    std::unique_ptr<splbcu_sim, Del> h_;
};

}  // namespace splb
