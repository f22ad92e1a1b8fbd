// Host-side data model of the B200 engine: sparse domain, site lookup,
// partition.  Fresh C++ with the reference's semantics; the site order,
// link tags, decomposition and error texts are the parity contract.
#pragma once

#include <array>
#include <cstdint>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

#include "lattice.hpp"

namespace splbcu {

// ---- error taxonomy (reference common.hpp:11-28) -------------------------
enum class ErrKind { Config = 1, Runtime = 2, Comm = 3, Geometry = 4, Degenerate = 5, Cuda = 6 };

struct Error : std::runtime_error {
    ErrKind kind;
    Error(ErrKind k, const std::string& m) : std::runtime_error(m), kind(k) {}
};
[[noreturn]] inline void fail(ErrKind k, const std::string& m) { throw Error(k, m); }
[[noreturn]] inline void geometry_error(const std::string& m) { fail(ErrKind::Geometry, m); }
[[noreturn]] inline void config_error(const std::string& m) { fail(ErrKind::Config, m); }
[[noreturn]] inline void runtime_error(const std::string& m) { fail(ErrKind::Runtime, m); }

// ---- small helpers ---------------------------------------------------------
int hw_threads();
// Phase timer printed to stderr when SPLBCU_VERBOSE is set.
void phase(const char* what);
// Runs fn(begin, end, thread_index) over [0, n) split in contiguous chunks.
void parallel_for(uint64_t n, const std::function<void(uint64_t, uint64_t, int)>& fn,
                  uint64_t min_chunk = 1 << 15);

// (z, y, x) lexicographic key: the order sites take inside each collision
// type (geometry.hpp:189-195).  21 bits per axis with the reference's bias
// (geometry.hpp:82-86 uses the same bias, x-major; we need z-major).
constexpr int64_t kBias = int64_t{1} << 20;
inline uint64_t zyx_key(int32_t x, int32_t y, int32_t z) {
    return (uint64_t(int64_t(z) + kBias) << 42) | (uint64_t(int64_t(y) + kBias) << 21) |
           uint64_t(int64_t(x) + kBias);
}

struct IoletGeo {
    int32_t kind;  // 0 inlet, 1 outlet
    double center[3];
    double normal[3];
    double radius;
};

// Link tag per (site, direction i = 1..18) as in geometry.hpp:14-22.  Iolet
// ids are kept sparsely: only iolet links carry one.
struct Domain {
    double voxel_size = 1.0;
    uint64_t n = 0;
    std::vector<int32_t> coords;     // 3n, domain order
    std::vector<uint8_t> types;      // n
    std::vector<uint8_t> link_kind;  // 18n, [18*s + i-1]
    // sorted by (site, dir): iolet link -> iolet id
    std::vector<uint64_t> iolet_link_pos;  // 18*s + i-1
    std::vector<uint16_t> iolet_link_id;
    std::vector<IoletGeo> iolets;
    uint64_t type_ranges[6][2] = {};

    uint16_t link_iolet(uint64_t s, int i) const;  // 0 when not an iolet link
};

// Lookup of a site by coordinates: sites sorted by zyx key, with a CSR row
// index over (z, y) when the bounding box allows it.  Used for link closure,
// decomposition edges and (uploaded to the device) the neighbour table.
struct SiteIndex {
    std::vector<uint64_t> keys;   // ascending
    std::vector<uint32_t> value;  // payload per key (e.g. global site index)
    int32_t lo[3] = {0, 0, 0}, hi[3] = {-1, -1, -1};
    bool rows = false;
    std::vector<uint64_t> row_off;  // (ny*nz + 1) offsets when rows
    int64_t ny = 0, nz = 0;

    // dense occupancy bitmap over the bounding box (when it fits in 1 GiB)
    std::vector<uint64_t> bits;
    int64_t bnx = 0;

    void build_rows();
    void build_bitmap();
    // position in keys of (x,y,z) or -1
    int64_t find(int32_t x, int32_t y, int32_t z) const;
    bool contains(int32_t x, int32_t y, int32_t z) const {
        if (bits.empty()) return find(x, y, z) >= 0;
        if (x < lo[0] || x > hi[0] || y < lo[1] || y > hi[1] || z < lo[2] || z > hi[2]) return false;
        const uint64_t b = uint64_t(((int64_t(z) - lo[2]) * ny + (int64_t(y) - lo[1])) * bnx + (int64_t(x) - lo[0]));
        return (bits[b >> 6] >> (b & 63)) & 1u;
    }
};

// Builds the lookup over all sites of a domain (value = global site index).
SiteIndex index_domain(const Domain& d);

// ---- geometry (geometry.hpp) --------------------------------------------
Domain classify_sites(const std::vector<int32_t>& voxels, std::vector<IoletGeo> iolets,
                      double voxel_size);
void validate_domain(const Domain& d);
Domain build_pipe(int radius, int length, double voxel_size);
Domain build_bifurcation(int trunk_radius, int branch_radius, int trunk_length,
                         int branch_length, double voxel_size);
Domain build_tree(int root_radius, int root_length, int levels, double radius_ratio,
                  double length_ratio, double voxel_size);
Domain build_channel(int nx, int ny, int nz, double voxel_size);
Domain read_domain(const std::string& path);
void write_domain(const Domain& d, const std::string& path);

// ---- geometry sources (slab-local construction) --------------
// A generator evaluated one z-slice at a time.  The builders above are
// build_from_source(source_*(...)); a distributed engine instead classifies
// only its own slab (± halo planes) of the same source.
struct Source {
    double voxel_size = 1.0;
    int32_t z0 = 0, z1 = -1;  // slices [z0, z1]
    std::vector<IoletGeo> iolets;
    // fluid voxels of slice z as (x, y) pairs in ascending (y, x) order
    std::function<void(int32_t z, std::vector<int32_t>& xy)> slice;
};
Source source_pipe(int radius, int length, double voxel_size);
Source source_bifurcation(int trunk_radius, int branch_radius, int trunk_length, int branch_length,
                          double voxel_size);
Source source_tree(int root_radius, int root_length, int levels, double radius_ratio, double length_ratio,
                   double voxel_size);
Source source_channel(int nx, int ny, int nz, double voxel_size);
Domain build_from_source(const Source& src);

// Per-slice fluid counts and the x/y extent of a source (every slice voxelised).
struct SourcePlan {
    std::vector<uint64_t> plane_count;  // slice z0 + k
    int32_t lo[3] = {0, 0, 0}, hi[3] = {-1, -1, -1};
    uint64_t n = 0;
};
SourcePlan plan_source(const Source& src);

// Classified sites of slices [za, zb] of a source (clamped to its range).
// Sites of the first/last slice are classified as if the neighbouring slices
// were absent, so callers pass one extra slice on each side and discard it.
// Unlike classify_sites, an iolet without links here is not an error (it may
// lie in another slab); `io_links` counts each iolet's links.
Domain classify_slab(const Source& src, int32_t za, int32_t zb, std::vector<uint64_t>* io_links);

// ---- decomposition (decomp.hpp) ------------------------------------------
struct WorkerPart {
    std::vector<uint32_t> sites;  // global indices, worker-local order
    uint32_t n_edge = 0;
    uint64_t edge_ranges[6][2] = {};
    uint64_t mid_ranges[6][2] = {};
    std::vector<int> neighbors;
};

struct Partition {
    int n_workers = 1;
    int axis = 2;
    bool slab = true;               // greedy plane split (else contiguous fallback)
    int32_t plane_lo = 0;           // slab mode: plane coordinate range
    std::vector<int32_t> plane_owner;  // slab mode: owner per plane (plane_lo + k)
    std::vector<int32_t> owner;     // per global site
    std::vector<uint32_t> local_index;
    std::vector<WorkerPart> parts;
    double imbalance() const;
};

Partition partition(const Domain& d, int n_workers, const SiteIndex* index = nullptr);

// ---- slab-local construction (distributed engine) ----------
// The reference partition of a source computed from per-slice counts alone:
// valid when it is a z-slab split (longest axis z, at least as many non-empty
// slices as workers), which is then the same split partition() makes of the
// whole domain.
struct SlabPlan {
    bool ok = false;
    uint64_t n = 0;                     // global site count
    int32_t plane_lo = 0;               // first non-empty slice
    std::vector<int32_t> plane_owner;   // slice plane_lo + k -> worker
    std::vector<uint64_t> plane_count;  // slice plane_lo + k -> sites
    int32_t own_lo(int w) const;
    int32_t own_hi(int w) const;
};
SlabPlan plan_slabs(const SourcePlan& sp, int32_t z0, int n_workers);

// One worker's window: its slices plus one halo slice on each side, with
// sites in global (type-major zyx) order restricted to the window, so each
// type's window sites are one contiguous run of the global order.
struct Window {
    Domain dom;
    int worker = 0;
    int32_t own_lo = 0, own_hi = -1;
    uint64_t n_global = 0;
    uint64_t g_type_ranges[6][2] = {};
    uint64_t g_first[6] = {};  // global index of the window's first site of each type
    uint64_t global_of(uint64_t s) const {
        const int t = dom.types[s];
        return g_first[t] + (s - dom.type_ranges[t][0]);
    }
};
// Classifies the window of `worker`; `own_counts` receives the per-type
// counts of each own slice (6 per slice, own_lo first) and `io_links` each
// iolet's link count over the own slices.
Window classify_window(const Source& src, const SlabPlan& plan, int worker, std::vector<uint64_t>* own_counts,
                       std::vector<uint64_t>* io_links);
// Fixes the global indices from every slice's per-type counts (6 per slice,
// plane_lo first, all workers' own_counts concatenated in worker order).
void finish_window(Window& w, const SlabPlan& plan, const std::vector<uint64_t>& counts);
// partition() of the whole domain, restricted to what `w.worker` needs: the
// owner of every window site, and the worker's own part (sites as window
// indices) with its edge/mid groups and neighbours.  Other parts stay empty.
Partition partition_window(const Window& w, const SlabPlan& plan, int n_workers);

// ---- time tables (boundary.hpp:18-74) ------------------------------------
struct TimeTable {
    std::vector<double> t, v;
    double period = 0.0;
    void validate() const;
    double at(double tq) const;
};

}  // namespace splbcu
