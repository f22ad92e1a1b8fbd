// Sparse domain construction, validation, builders and SPLB file I/O.
// Semantics follow the reference geometry.hpp / geometry_io.hpp; the data
// structures are B200-host-first: structure-of-arrays, O(n) generation in
// (z,y,x) order, a CSR row index instead of a hash map, and parallel loops,
// so 10^8-site domains build in seconds.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <memory>
#include <mutex>
#include <thread>

#include "host.hpp"

namespace splbcu {

int hw_threads() {
    static int n = [] {
        unsigned h = std::thread::hardware_concurrency();
        return int(h == 0 ? 1 : std::min(h, 64u));
    }();
    return n;
}

void phase(const char* what) {
    static const bool on = std::getenv("SPLBCU_VERBOSE") != nullptr;
    static auto last = std::chrono::steady_clock::now();
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[splbcu] %-28s %8.3f s\n", what, std::chrono::duration<double>(now - last).count());
    last = now;
}

void parallel_for(uint64_t n, const std::function<void(uint64_t, uint64_t, int)>& fn,
                  uint64_t min_chunk) {
    const int nt = int(std::min<uint64_t>(hw_threads(), (n + min_chunk - 1) / std::max<uint64_t>(min_chunk, 1)));
    if (nt <= 1) {
        if (n) fn(0, n, 0);
        return;
    }
    std::vector<std::thread> th;
    std::vector<std::exception_ptr> err(nt);
    const uint64_t chunk = (n + nt - 1) / nt;
    for (int t = 0; t < nt; ++t) {
        const uint64_t b = uint64_t(t) * chunk, e = std::min(n, b + chunk);
        th.emplace_back([&, b, e, t] {
            try {
                if (b < e) fn(b, e, t);
            } catch (...) {
                err[t] = std::current_exception();
            }
        });
    }
    for (auto& t : th) t.join();
    for (auto& e : err)
        if (e) std::rethrow_exception(e);
}

uint16_t Domain::link_iolet(uint64_t s, int i) const {
    const uint64_t pos = 18 * s + uint64_t(i - 1);
    auto it = std::lower_bound(iolet_link_pos.begin(), iolet_link_pos.end(), pos);
    if (it == iolet_link_pos.end() || *it != pos) return 0;
    return iolet_link_id[size_t(it - iolet_link_pos.begin())];
}

// ---- SiteIndex --------------------------------------------------------------

static inline void key_coords(uint64_t k, int32_t& x, int32_t& y, int32_t& z) {
    const uint64_t m = (uint64_t(1) << 21) - 1;
    x = int32_t(int64_t(k & m) - kBias);
    y = int32_t(int64_t((k >> 21) & m) - kBias);
    z = int32_t(int64_t(k >> 42) - kBias);
}

void SiteIndex::build_rows() {
    rows = false;
    row_off.clear();
    if (keys.empty()) return;
    for (int a = 0; a < 3; ++a) lo[a] = INT32_MAX, hi[a] = INT32_MIN;
    // keys are sorted: z range from ends; x/y ranges need a scan
    int32_t x, y, z;
    key_coords(keys.front(), x, y, z);
    lo[2] = z;
    key_coords(keys.back(), x, y, z);
    hi[2] = z;
    std::vector<int32_t> lx(hw_threads(), INT32_MAX), hx(hw_threads(), INT32_MIN),
        ly(hw_threads(), INT32_MAX), hy(hw_threads(), INT32_MIN);
    parallel_for(keys.size(), [&](uint64_t b, uint64_t e, int t) {
        int32_t X, Y, Z;
        int32_t a0 = INT32_MAX, a1 = INT32_MIN, b0 = INT32_MAX, b1 = INT32_MIN;  // thread-local: no false sharing
        for (uint64_t k = b; k < e; ++k) {
            key_coords(keys[k], X, Y, Z);
            a0 = std::min(a0, X);
            a1 = std::max(a1, X);
            b0 = std::min(b0, Y);
            b1 = std::max(b1, Y);
        }
        lx[t] = a0, hx[t] = a1, ly[t] = b0, hy[t] = b1;
    });
    lo[0] = *std::min_element(lx.begin(), lx.end());
    hi[0] = *std::max_element(hx.begin(), hx.end());
    lo[1] = *std::min_element(ly.begin(), ly.end());
    hi[1] = *std::max_element(hy.begin(), hy.end());
    ny = int64_t(hi[1]) - lo[1] + 1;
    nz = int64_t(hi[2]) - lo[2] + 1;
    const double nrows = double(ny) * double(nz);
    if (nrows > double(uint64_t(1) << 28) || nrows > 8.0 * double(keys.size()) + 4096.0) return;
    row_off.assign(size_t(ny * nz + 1), 0);
    // count per row then prefix (keys sorted, so rows are contiguous)
    for (uint64_t k = 0; k < keys.size(); ++k) {
        key_coords(keys[k], x, y, z);
        ++row_off[size_t((int64_t(z) - lo[2]) * ny + (int64_t(y) - lo[1])) + 1];
    }
    for (size_t r = 1; r < row_off.size(); ++r) row_off[r] += row_off[r - 1];
    rows = true;
}

// Requires build_rows() first (bounding box).
void SiteIndex::build_bitmap() {
    bits.clear();
    if (keys.empty()) return;
    bnx = int64_t(hi[0]) - lo[0] + 1;
    const double cells = double(bnx) * double(ny) * double(nz);
    if (cells > double(uint64_t(1) << 33)) return;  // > 1 GiB: fall back to the row index
    bits.assign(size_t((uint64_t(cells) + 63) / 64), 0);
    uint64_t* w = bits.data();
    const int32_t lx = lo[0], ly = lo[1], lz = lo[2];
    const int64_t NY = ny, NX = bnx;
    parallel_for(keys.size(), [&](uint64_t b, uint64_t e, int) {
        int32_t x, y, z;
        for (uint64_t k = b; k < e; ++k) {
            key_coords(keys[k], x, y, z);
            const uint64_t c = uint64_t(((int64_t(z) - lz) * NY + (int64_t(y) - ly)) * NX + (int64_t(x) - lx));
            __atomic_fetch_or(&w[c >> 6], uint64_t(1) << (c & 63), __ATOMIC_RELAXED);
        }
    });
}

int64_t SiteIndex::find(int32_t x, int32_t y, int32_t z) const {
    const uint64_t key = zyx_key(x, y, z);
    uint64_t b = 0, e = keys.size();
    if (rows) {
        if (y < lo[1] || y > hi[1] || z < lo[2] || z > hi[2]) return -1;
        const size_t r = size_t((int64_t(z) - lo[2]) * ny + (int64_t(y) - lo[1]));
        b = row_off[r];
        e = row_off[r + 1];
    }
    auto it = std::lower_bound(keys.begin() + b, keys.begin() + e, key);
    if (it == keys.begin() + e || *it != key) return -1;
    return int64_t(it - keys.begin());
}

SiteIndex index_domain(const Domain& d) {
    SiteIndex ix;
    ix.keys.resize(d.n);
    std::vector<uint32_t> perm(d.n);
    parallel_for(d.n, [&](uint64_t b, uint64_t e, int) {
        for (uint64_t s = b; s < e; ++s) {
            ix.keys[s] = zyx_key(d.coords[3 * s], d.coords[3 * s + 1], d.coords[3 * s + 2]);
            perm[s] = uint32_t(s);
        }
    });
    // Domain order is type-major and zyx-sorted inside each type range: a
    // 6-way merge gives the global zyx order.
    std::vector<uint64_t> mk(d.n);
    std::vector<uint32_t> mv(d.n);
    {
        std::vector<std::pair<uint64_t, uint64_t>> runs;
        for (int t = 0; t < 6; ++t)
            if (d.type_ranges[t][1] > d.type_ranges[t][0])
                runs.push_back({d.type_ranges[t][0], d.type_ranges[t][1]});
        bool sorted_runs = true;
        for (auto& r : runs)
            for (uint64_t k = r.first + 1; k < r.second && sorted_runs; ++k)
                if (!(ix.keys[k - 1] < ix.keys[k])) sorted_runs = false;
        if (!sorted_runs || runs.empty()) {
            std::sort(perm.begin(), perm.end(),
                      [&](uint32_t a, uint32_t b) { return ix.keys[a] < ix.keys[b]; });
            for (uint64_t k = 0; k < d.n; ++k) mk[k] = ix.keys[perm[k]], mv[k] = perm[k];
        } else {
            // Bucket by z-plane (each run splits into contiguous per-plane
            // pieces found by binary search), then sort every plane's few
            // pieces independently, in parallel.
            const int32_t z0 = int32_t(int64_t(ix.keys[runs[0].first] >> 42) - kBias);
            int32_t zmin = z0, zmax = z0;
            for (auto& r : runs) {
                zmin = std::min(zmin, int32_t(int64_t(ix.keys[r.first] >> 42) - kBias));
                zmax = std::max(zmax, int32_t(int64_t(ix.keys[r.second - 1] >> 42) - kBias));
            }
            const size_t nzp = size_t(int64_t(zmax) - zmin + 1);
            // cut[r][p] = first position of run r with z >= zmin + p
            std::vector<std::vector<uint64_t>> cut(runs.size(), std::vector<uint64_t>(nzp + 1));
            for (size_t r = 0; r < runs.size(); ++r) {
                for (size_t p = 0; p <= nzp; ++p) {
                    const uint64_t kz = p == nzp ? UINT64_MAX : (uint64_t(int64_t(zmin) + int64_t(p) + kBias) << 42);
                    cut[r][p] = uint64_t(std::lower_bound(ix.keys.begin() + int64_t(runs[r].first),
                                                          ix.keys.begin() + int64_t(runs[r].second), kz) -
                                         ix.keys.begin());
                }
            }
            std::vector<uint64_t> out_off(nzp + 1, 0);
            for (size_t p = 0; p < nzp; ++p) {
                uint64_t c = 0;
                for (size_t r = 0; r < runs.size(); ++r) c += cut[r][p + 1] - cut[r][p];
                out_off[p + 1] = out_off[p] + c;
            }
            parallel_for(nzp, [&](uint64_t pb, uint64_t pe, int) {
                std::vector<std::pair<uint64_t, uint32_t>> buf;
                for (uint64_t p = pb; p < pe; ++p) {
                    buf.clear();
                    for (size_t r = 0; r < runs.size(); ++r)
                        for (uint64_t s = cut[r][p]; s < cut[r][p + 1]; ++s) buf.push_back({ix.keys[s], uint32_t(s)});
                    std::sort(buf.begin(), buf.end());
                    uint64_t o = out_off[p];
                    for (auto& kv : buf) mk[o] = kv.first, mv[o] = kv.second, ++o;
                }
            }, 1);
        }
    }
    phase("index_domain merge");
    ix.keys.swap(mk);
    ix.value.swap(mv);
    ix.build_rows();
    return ix;
}

// ---- classification (geometry.hpp:100-208) ----------------------------------

static double dot3(const double* a, const double* b) { return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2]; }

// crosses_iolet (geometry.hpp:102-113)
static bool crosses_iolet(const double a[3], const double b[3], const IoletGeo& io) {
    const double da[3] = {a[0] - io.center[0], a[1] - io.center[1], a[2] - io.center[2]};
    const double db[3] = {b[0] - io.center[0], b[1] - io.center[1], b[2] - io.center[2]};
    const double sa = dot3(da, io.normal);
    const double sb = dot3(db, io.normal);
    if (!(sa > 0.0 && sb <= 0.0)) return false;
    const double t = sa / (sa - sb);
    const double p[3] = {a[0] + t * (b[0] - a[0]), a[1] + t * (b[1] - a[1]), a[2] + t * (b[2] - a[2])};
    const double d[3] = {p[0] - io.center[0], p[1] - io.center[1], p[2] - io.center[2]};
    const double r2 = dot3(d, d);
    const double rmax = io.radius + 1.0;  // kIoletClassifyMargin (geometry.hpp:78)
    return r2 <= rmax * rmax;
}

static bool unit_normal(const IoletGeo& io) {
    return !(std::abs(std::sqrt(dot3(io.normal, io.normal)) - 1.0) > 1e-12);
}

static uint8_t type_of(bool wall, bool inlet, bool outlet) {
    if (inlet) return wall ? 4 : 2;
    if (outlet) return wall ? 5 : 3;
    return wall ? 1 : 0;
}

// Core of classify_sites for voxels already in strictly ascending zyx order
// (duplicates rejected by the caller).  input_index maps a sorted position
// back to the caller's order so error reports name the same site as the
// reference (the first offending voxel in input order).
// Slab mode (classify_slab): only sites with z in [za, zb] are kept and
// checked; an iolet without links is reported through io_links instead.
struct SlabKeep {
    int32_t za, zb;
    std::vector<uint64_t>* io_links;
};

static Domain classify_sorted(std::vector<int32_t>&& coords, const std::vector<uint64_t>& keys,
                              const std::vector<uint32_t>* input_index,
                              std::vector<IoletGeo>&& iolets, double voxel_size,
                              const SlabKeep* slab = nullptr) {
    uint64_t n = keys.size();
    auto kept = [&](uint64_t s) { return !slab || (coords[3 * s + 2] >= slab->za && coords[3 * s + 2] <= slab->zb); };
    SiteIndex ix;
    ix.keys = keys;
    ix.build_rows();
    ix.build_bitmap();
    phase("classify: rows+bitmap");

    std::vector<uint8_t> kind(18 * n);
    std::vector<uint8_t> type(n);
    const int nt = hw_threads();
    std::vector<std::vector<uint32_t>> io_count(nt, std::vector<uint32_t>(iolets.size(), 0));
    std::vector<std::vector<std::pair<uint64_t, uint16_t>>> io_links(nt);
    // per thread: smallest input index of an inlet+outlet site, and its position
    std::vector<uint64_t> bad_in(nt, UINT64_MAX), bad_pos(nt, UINT64_MAX);

    parallel_for(n, [&](uint64_t b, uint64_t e, int t) {
        for (uint64_t s = b; s < e; ++s) {
            const int32_t x = coords[3 * s], y = coords[3 * s + 1], z = coords[3 * s + 2];
            const double a[3] = {double(x), double(y), double(z)};
            bool wall = false, inlet = false, outlet = false;
            for (int i = 1; i < kQ; ++i) {
                const int32_t tx = x + cx(i), ty = y + cy(i), tz = z + cz(i);
                uint8_t k;
                // +-x neighbours are adjacent in zyx order
                bool member;
                if (cy(i) == 0 && cz(i) == 0) {
                    const int64_t p = int64_t(s) + cx(i);
                    member = p >= 0 && uint64_t(p) < n && keys[uint64_t(p)] == zyx_key(tx, ty, tz);
                } else {
                    member = ix.contains(tx, ty, tz);
                }
                if (member) {
                    k = 0;
                } else {
                    k = 1;
                    const double bb[3] = {double(tx), double(ty), double(tz)};
                    for (size_t io = 0; io < iolets.size(); ++io)
                        if (crosses_iolet(a, bb, iolets[io])) {
                            k = iolets[io].kind == 0 ? 2 : 3;
                            io_links[t].push_back({18 * s + uint64_t(i - 1), uint16_t(io)});
                            if (kept(s)) ++io_count[t][io];
                            break;
                        }
                }
                kind[18 * s + uint64_t(i - 1)] = k;
                wall |= k == 1;
                inlet |= k == 2;
                outlet |= k == 3;
            }
            if (inlet && outlet && kept(s)) {
                const uint64_t in_idx = input_index ? (*input_index)[s] : s;
                if (in_idx < bad_in[t]) bad_in[t] = in_idx, bad_pos[t] = s;
            }
            type[s] = type_of(wall, inlet, outlet);
        }
    });
    uint64_t s = UINT64_MAX, best_in = UINT64_MAX;
    for (int t = 0; t < nt; ++t)
        if (bad_in[t] < best_in) best_in = bad_in[t], s = bad_pos[t];
    if (s != UINT64_MAX) {
        geometry_error("classify_sites: site (" + std::to_string(coords[3 * s]) + "," +
                       std::to_string(coords[3 * s + 1]) + "," + std::to_string(coords[3 * s + 2]) +
                       ") carries both inlet and outlet links");
    }
    for (size_t io = 0; io < iolets.size(); ++io) {
        uint64_t c = 0;
        for (int t = 0; t < nt; ++t) c += io_count[t][io];
        if (slab) {
            if (slab->io_links) slab->io_links->push_back(c);
        } else if (c == 0) {
            geometry_error("classify_sites: iolet " + std::to_string(io) +
                           " intersects no boundary links");
        }
    }

    phase("classify: links");
    // Stable counting sort by type over the zyx order == sort by (type,z,y,x)
    // (geometry.hpp:189-195).
    Domain d;
    d.voxel_size = voxel_size;
    d.iolets = std::move(iolets);
    if (slab) {
        // drop the classification-only slices: compact the kept sites in place
        uint64_t m = 0;
        std::vector<uint64_t> newpos(n, UINT64_MAX);
        for (uint64_t s = 0; s < n; ++s)
            if (kept(s)) newpos[s] = m++;
        for (uint64_t s = 0; s < n; ++s) {
            const uint64_t q = newpos[s];
            if (q == UINT64_MAX || q == s) continue;
            std::memcpy(&coords[3 * q], &coords[3 * s], 12);
            std::memcpy(&kind[18 * q], &kind[18 * s], 18);
            type[q] = type[s];
        }
        for (auto& v : io_links) {
            size_t o = 0;
            for (auto& p : v)
                if (newpos[p.first / 18] != UINT64_MAX) v[o++] = {18 * newpos[p.first / 18] + p.first % 18, p.second};
            v.resize(o);
        }
        n = m;
    }
    d.n = n;
    uint64_t cnt[6] = {};
    for (uint64_t s = 0; s < n; ++s) ++cnt[type[s]];
    uint64_t pos = 0;
    for (int t = 0; t < 6; ++t) {
        d.type_ranges[t][0] = pos;
        pos += cnt[t];
        d.type_ranges[t][1] = pos;
    }
    std::vector<uint64_t> dst(n);
    {
        uint64_t next[6];
        for (int t = 0; t < 6; ++t) next[t] = d.type_ranges[t][0];
        for (uint64_t s = 0; s < n; ++s) dst[s] = next[type[s]]++;
    }
    d.coords.resize(3 * n);
    d.types.resize(n);
    d.link_kind.resize(18 * n);
    parallel_for(n, [&](uint64_t b, uint64_t e, int) {
        for (uint64_t s = b; s < e; ++s) {
            const uint64_t g = dst[s];
            std::memcpy(&d.coords[3 * g], &coords[3 * s], 12);
            d.types[g] = type[s];
            std::memcpy(&d.link_kind[18 * g], &kind[18 * s], 18);
        }
    });
    std::vector<std::pair<uint64_t, uint16_t>> links;
    for (auto& v : io_links)
        for (auto& p : v) links.push_back({18 * dst[p.first / 18] + p.first % 18, p.second});
    std::sort(links.begin(), links.end());
    d.iolet_link_pos.resize(links.size());
    d.iolet_link_id.resize(links.size());
    for (size_t k = 0; k < links.size(); ++k) {
        d.iolet_link_pos[k] = links[k].first;
        d.iolet_link_id[k] = links[k].second;
    }
    return d;
}

Domain classify_sites(const std::vector<int32_t>& voxels, std::vector<IoletGeo> iolets,
                      double voxel_size) {
    const uint64_t n = voxels.size() / 3;
    if (n == 0) geometry_error("classify_sites: empty voxel set");
    for (size_t k = 0; k < iolets.size(); ++k)
        if (!unit_normal(iolets[k]))
            geometry_error("classify_sites: iolet " + std::to_string(k) + " normal is not unit length");
    for (uint64_t s = 0; s < 3 * n; ++s)
        if (voxels[s] < -(int32_t(1) << 20) + 1 || voxels[s] >= (int32_t(1) << 20) - 1)
            geometry_error("classify_sites: voxel coordinate out of range");
    std::vector<uint64_t> keys(n);
    for (uint64_t s = 0; s < n; ++s) keys[s] = zyx_key(voxels[3 * s], voxels[3 * s + 1], voxels[3 * s + 2]);
    bool sorted = true;
    for (uint64_t s = 1; s < n && sorted; ++s) sorted = keys[s - 1] < keys[s];
    phase("classify: keys");
    if (sorted) {
        std::vector<int32_t> c(voxels);
        return classify_sorted(std::move(c), keys, nullptr, std::move(iolets), voxel_size);
    }
    std::vector<uint32_t> perm(n);
    for (uint64_t s = 0; s < n; ++s) perm[s] = uint32_t(s);
    std::sort(perm.begin(), perm.end(), [&](uint32_t a, uint32_t b) {
        return keys[a] < keys[b] || (keys[a] == keys[b] && a < b);
    });
    std::vector<uint64_t> sk(n);
    std::vector<int32_t> sc(3 * n);
    for (uint64_t k = 0; k < n; ++k) {
        sk[k] = keys[perm[k]];
        std::memcpy(&sc[3 * k], &voxels[3 * uint64_t(perm[k])], 12);
        if (k && sk[k] == sk[k - 1]) geometry_error("classify_sites: duplicate voxel");
    }
    return classify_sorted(std::move(sc), sk, &perm, std::move(iolets), voxel_size);
}

// validate_domain (geometry.hpp:212-271).  Checks run in parallel; the
// reported violation is the first one in the reference's sequential order.
void validate_domain(const Domain& d) {
    if (d.n == 0) geometry_error("domain: empty site list");
    if (!(d.voxel_size > 0.0)) geometry_error("domain: voxel size must be positive");
    for (size_t k = 0; k < d.iolets.size(); ++k)
        if (!unit_normal(d.iolets[k]))
            geometry_error("domain: iolet " + std::to_string(k) + " normal is not unit length");
    // duplicates (index_coords); index_domain merges the type runs when the
    // ranges are a valid partition of zyx-sorted runs, else sorts.
    bool ranges_ok = true;
    {
        uint64_t p = 0;
        for (int t = 0; t < 6; ++t) {
            if (d.type_ranges[t][0] != p || d.type_ranges[t][1] < p || d.type_ranges[t][1] > d.n) ranges_ok = false;
            p = d.type_ranges[t][1];
        }
        ranges_ok &= p == d.n;
    }
    std::vector<uint64_t> sk;
    if (ranges_ok) {
        sk = index_domain(d).keys;
    } else {
        sk.resize(d.n);
        for (uint64_t s = 0; s < d.n; ++s) sk[s] = zyx_key(d.coords[3 * s], d.coords[3 * s + 1], d.coords[3 * s + 2]);
        std::sort(sk.begin(), sk.end());
    }
    for (uint64_t k = 1; k < d.n; ++k)
        if (sk[k] == sk[k - 1]) geometry_error("classify_sites: duplicate voxel");
    uint64_t pos = 0;
    for (int t = 0; t < 6; ++t) {
        if (d.type_ranges[t][0] != pos || d.type_ranges[t][1] < pos || d.type_ranges[t][1] > d.n)
            geometry_error("domain: type_ranges do not partition the sites");
        pos = d.type_ranges[t][1];
        for (uint64_t s = d.type_ranges[t][0]; s < d.type_ranges[t][1]; ++s)
            if (int(d.types[s]) != t) geometry_error("domain: site type outside its range");
    }
    if (pos != d.n) geometry_error("domain: type_ranges do not partition the sites");

    SiteIndex ix;
    ix.keys = std::move(sk);
    ix.build_rows();
    ix.build_bitmap();
    phase("validate: index+bitmap");
    const int nt = hw_threads();
    std::vector<uint64_t> first_bad(nt, UINT64_MAX);
    std::vector<int> first_code(nt, 0);
    parallel_for(d.n, [&](uint64_t b, uint64_t e, int t) {
        size_t lk = size_t(std::lower_bound(d.iolet_link_pos.begin(), d.iolet_link_pos.end(), 18 * b) -
                           d.iolet_link_pos.begin());
        for (uint64_t s = b; s < e && first_bad[t] == UINT64_MAX; ++s) {
            bool wall = false, inlet = false, outlet = false;
            int code = 0;
            const int32_t x = d.coords[3 * s], y = d.coords[3 * s + 1], z = d.coords[3 * s + 2];
            for (int i = 1; i < kQ && !code; ++i) {
                const uint8_t k = d.link_kind[18 * s + uint64_t(i - 1)];
                uint16_t io = 0;
                while (lk < d.iolet_link_pos.size() && d.iolet_link_pos[lk] < 18 * s + uint64_t(i - 1)) ++lk;
                if (lk < d.iolet_link_pos.size() && d.iolet_link_pos[lk] == 18 * s + uint64_t(i - 1))
                    io = d.iolet_link_id[lk];
                const bool in_set = ix.contains(x + cx(i), y + cy(i), z + cz(i));
                if (k == 0) {
                    if (!in_set) code = 1;
                } else {
                    if (in_set) code = 1;
                    else if (k != 1 && io >= d.iolets.size()) code = 2;
                }
                wall |= k == 1;
                inlet |= k == 2;
                outlet |= k == 3;
            }
            if (!code && inlet && outlet) code = 3;
            if (!code && d.types[s] != type_of(wall, inlet, outlet)) code = 4;
            if (code) {
                first_bad[t] = s;
                first_code[t] = code;
            }
        }
    });
    phase("validate: links");
    uint64_t best = UINT64_MAX;
    int code = 0;
    for (int t = 0; t < nt; ++t)
        if (first_bad[t] < best) best = first_bad[t], code = first_code[t];
    switch (code) {
        case 1: geometry_error("domain: inconsistent link closure");
        case 2: geometry_error("domain: link references unknown iolet");
        case 3: geometry_error("domain: site carries both inlet and outlet links");
        case 4: geometry_error("domain: collision type inconsistent with links");
        default: break;
    }
}

// ---- builders ------------------------------------------------------------------

constexpr double kAxisOffsetX = 0.375;  // geometry.hpp:279
constexpr double kAxisOffsetY = 0.5;    // geometry.hpp:280

// ---- sources: generators evaluated slice by slice ------------------------------
// Every builder is build_from_source(source_*): the slice functions are the
// only definition of each geometry, so a slab classified by a distributed
// engine (classify_slab) sees exactly the voxels of the whole-domain build.

// build_pipe (geometry.hpp:285-308): every slice is the same disc.
Source source_pipe(int radius, int length, double voxel_size) {
    if (radius < 2 || length < 4) geometry_error("build_pipe: need radius >= 2 and length >= 4");
    const double r2 = double(radius) * radius;
    auto disc = std::make_shared<std::vector<int32_t>>();
    for (int y = -radius - 2; y <= radius + 2; ++y)
        for (int x = -radius - 2; x <= radius + 2; ++x) {
            const double dx = x - kAxisOffsetX, dy = y - kAxisOffsetY;
            if (dx * dx + dy * dy < r2) {
                disc->push_back(x);
                disc->push_back(y);
            }
        }
    Source s;
    s.voxel_size = voxel_size;
    s.z0 = 0;
    s.z1 = length - 1;
    s.iolets = {
        {0, {kAxisOffsetX, kAxisOffsetY, -0.5}, {0.0, 0.0, 1.0}, double(radius)},
        {1, {kAxisOffsetX, kAxisOffsetY, double(length - 1) + 0.5}, {0.0, 0.0, -1.0}, double(radius)},
    };
    s.slice = [disc](int32_t, std::vector<int32_t>& xy) { xy = *disc; };
    return s;
}

// build_bifurcation (geometry.hpp:313-363): a trunk disc, then two discs
// whose centres diverge linearly in x.
Source source_bifurcation(int tr, int br, int tl, int bl, double voxel_size) {
    if (tr < 2 || br < 2 || tl < 4 || bl < 4)
        geometry_error("build_bifurcation: need radii >= 2 and lengths >= 4");
    constexpr double kSlope = 0.5;
    const int xmax = int(std::ceil(kSlope * bl)) + tr + br + 2;
    const int rmax = std::max(tr, br) + 2;
    Source s;
    s.voxel_size = voxel_size;
    s.z0 = 0;
    s.z1 = tl + bl - 1;
    const double zend = double(tl + bl - 1) + 0.5;
    const double xend = kSlope * bl;
    s.iolets = {
        {0, {kAxisOffsetX, kAxisOffsetY, -0.5}, {0.0, 0.0, 1.0}, double(tr)},
        {1, {kAxisOffsetX + xend, kAxisOffsetY, zend}, {0.0, 0.0, -1.0}, double(br)},
        {1, {kAxisOffsetX - xend, kAxisOffsetY, zend}, {0.0, 0.0, -1.0}, double(br)},
    };
    s.slice = [=](int32_t z, std::vector<int32_t>& xy) {
        xy.clear();
        for (int y = -rmax; y <= rmax; ++y)
            for (int x = -xmax; x <= xmax; ++x) {
                const double dy = y - kAxisOffsetY;
                bool fluid;
                if (z < tl) {
                    const double dx = x - kAxisOffsetX;
                    fluid = dx * dx + dy * dy < tr * tr;
                } else {
                    const double xc = kSlope * (z - tl + 1);
                    const double dp = (x - kAxisOffsetX - xc);
                    const double dm = (x - kAxisOffsetX + xc);
                    fluid = dp * dp + dy * dy < br * br || dm * dm + dy * dy < br * br;
                }
                if (fluid) {
                    xy.push_back(x);
                    xy.push_back(y);
                }
            }
    };
    return s;
}

// Synthetic bifurcating vessel tree (configs C3 and C5; no reference
// equivalent — a recursive generalisation of build_bifurcation).  Level 0 is
// a trunk along +z; every vessel of level k splits into two level-(k+1)
// vessels whose centrelines diverge linearly, in x for odd levels and in y
// for even ones, by a lateral offset sized so sibling subtrees never touch.
// Each z-slice is a union of discs (one per active vessel).  One inlet at the
// trunk start, one outlet disc per leaf in the last slice + 0.5.
Source source_tree(int root_radius, int root_length, int levels, double radius_ratio, double length_ratio,
                   double voxel_size) {
    if (root_radius < 2 || root_length < 4 || levels < 0 || levels > 12 ||
        !(radius_ratio > 0.0 && radius_ratio <= 1.0) || !(length_ratio > 0.0))
        geometry_error("build_tree: need radius >= 2, length >= 4, 0 <= levels <= 12, "
                       "0 < radius_ratio <= 1, length_ratio > 0");
    struct Tree {
        int L = 0;
        std::vector<double> rad, disp;
        std::vector<int> len, z0;
        std::vector<std::vector<std::array<double, 4>>> seg;  // x0,y0,x1,y1 per vessel
    };
    auto t = std::make_shared<Tree>();
    const int L = levels + 1;
    t->L = L;
    t->rad.assign(L, 0.0);
    t->disp.assign(L, 0.0);
    t->len.assign(L, 0);
    for (int k = 0; k < L; ++k) t->rad[k] = std::max(2.0, root_radius * std::pow(radius_ratio, k));
    // lateral offset of a level-k vessel over its length (k >= 1), from the
    // leaves up: clear the widest descendant spread on the same axis.
    for (int k = L - 1; k >= 1; --k) {
        double spread = 0.0;
        for (int j = k + 2; j < L; j += 2) spread += t->disp[j];
        t->disp[k] = spread + t->rad[k] + 2.0;
    }
    for (int k = 0; k < L; ++k) {
        int l = int(std::lround(root_length * std::pow(length_ratio, k)));
        l = std::max(l, 4);
        if (k >= 1) l = std::max(l, int(std::ceil(1.5 * t->disp[k])));  // slope <= 2/3
        t->len[k] = l;
    }
    t->z0.assign(L + 1, 0);
    for (int k = 0; k < L; ++k) t->z0[k + 1] = t->z0[k] + t->len[k];
    const int nz = t->z0[L];
    // Vessel v of level k runs from its parent's end point to that point
    // +- disp[k] (level 0: the straight trunk).
    t->seg.resize(L);
    t->seg[0].push_back({kAxisOffsetX, kAxisOffsetY, kAxisOffsetX, kAxisOffsetY});
    for (int k = 1; k < L; ++k)
        for (auto& p : t->seg[k - 1]) {
            const double dx = (k % 2 == 1) ? t->disp[k] : 0.0;
            const double dy = (k % 2 == 0) ? t->disp[k] : 0.0;
            t->seg[k].push_back({p[2], p[3], p[2] - dx, p[3] - dy});
            t->seg[k].push_back({p[2], p[3], p[2] + dx, p[3] + dy});
        }
    Source s;
    s.voxel_size = voxel_size;
    s.z0 = 0;
    s.z1 = nz - 1;
    s.iolets.push_back({0, {kAxisOffsetX, kAxisOffsetY, -0.5}, {0.0, 0.0, 1.0}, t->rad[0]});
    {
        const int k = L - 1;
        const double zend = double(nz - 1) + 0.5;
        for (auto& sg : t->seg[size_t(k)]) {
            // leaf centre extrapolated to the outlet plane
            const double f = (zend - t->z0[k] + 1.0) / double(t->len[k]);
            s.iolets.push_back(
                {1, {sg[0] + f * (sg[2] - sg[0]), sg[1] + f * (sg[3] - sg[1]), zend}, {0.0, 0.0, -1.0}, t->rad[k]});
        }
    }
    s.slice = [t](int32_t z, std::vector<int32_t>& xy) {
        int k = 0;
        while (k + 1 < t->L && z >= t->z0[k + 1]) ++k;
        std::vector<uint64_t> keys;
        const double r = t->rad[k];
        const double r2 = r * r;
        const double f = t->len[k] > 1 ? double(z - t->z0[k] + 1) / double(t->len[k]) : 1.0;
        for (auto& sg : t->seg[size_t(k)]) {
            const double cx = sg[0] + f * (sg[2] - sg[0]);
            const double cy = sg[1] + f * (sg[3] - sg[1]);
            const int x0 = int(std::floor(cx - r)) - 1, x1 = int(std::ceil(cx + r)) + 1;
            const int y0 = int(std::floor(cy - r)) - 1, y1 = int(std::ceil(cy + r)) + 1;
            for (int y = y0; y <= y1; ++y)
                for (int x = x0; x <= x1; ++x) {
                    const double dx = x - cx, dy = y - cy;
                    if (dx * dx + dy * dy < r2)
                        keys.push_back((uint64_t(int64_t(y) + kBias) << 21) | uint64_t(int64_t(x) + kBias));
                }
        }
        std::sort(keys.begin(), keys.end());
        keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
        xy.resize(2 * keys.size());
        const uint64_t m = (uint64_t(1) << 21) - 1;
        for (size_t q = 0; q < keys.size(); ++q) {
            xy[2 * q] = int32_t(int64_t(keys[q] & m) - kBias);
            xy[2 * q + 1] = int32_t(int64_t(keys[q] >> 21) - kBias);
        }
    };
    return s;
}

// Dense rectangular channel (config C4): every voxel of [0,nx)x[0,ny)x[0,nz)
// is fluid; inlet/outlet discs cover the whole cross-section.
Source source_channel(int nx, int ny, int nz, double voxel_size) {
    if (nx < 2 || ny < 2 || nz < 4) geometry_error("build_channel: need nx, ny >= 2 and nz >= 4");
    Source s;
    s.voxel_size = voxel_size;
    s.z0 = 0;
    s.z1 = nz - 1;
    const double cx = 0.5 * (nx - 1), cy = 0.5 * (ny - 1);
    const double rad = 0.5 * std::sqrt(double(nx) * nx + double(ny) * ny);
    s.iolets = {
        {0, {cx, cy, -0.5}, {0.0, 0.0, 1.0}, rad},
        {1, {cx, cy, double(nz - 1) + 0.5}, {0.0, 0.0, -1.0}, rad},
    };
    s.slice = [nx, ny](int32_t, std::vector<int32_t>& xy) {
        xy.resize(2 * uint64_t(nx) * uint64_t(ny));
        uint64_t q = 0;
        for (int y = 0; y < ny; ++y)
            for (int x = 0; x < nx; ++x) xy[q++] = x, xy[q++] = y;
    };
    return s;
}

// Voxels of slices [za, zb] in zyx order (parallel over slices).
static std::vector<int32_t> voxelise(const Source& src, int32_t za, int32_t zb) {
    za = std::max(za, src.z0);
    zb = std::min(zb, src.z1);
    if (zb < za) return {};
    const uint64_t ns = uint64_t(int64_t(zb) - za + 1);
    std::vector<std::vector<int32_t>> slices(ns);
    parallel_for(ns, [&](uint64_t b, uint64_t e, int) {
        for (uint64_t k = b; k < e; ++k) src.slice(za + int32_t(k), slices[k]);
    }, 1);
    uint64_t total = 0;
    for (auto& s : slices) total += s.size() / 2;
    std::vector<int32_t> vox(3 * total);
    std::vector<uint64_t> off(ns + 1, 0);
    for (uint64_t k = 0; k < ns; ++k) off[k + 1] = off[k] + slices[k].size() / 2;
    parallel_for(ns, [&](uint64_t b, uint64_t e, int) {
        for (uint64_t k = b; k < e; ++k) {
            const std::vector<int32_t>& xy = slices[k];
            int32_t* v = &vox[3 * off[k]];
            for (uint64_t q = 0; q < xy.size() / 2; ++q) {
                v[3 * q] = xy[2 * q];
                v[3 * q + 1] = xy[2 * q + 1];
                v[3 * q + 2] = za + int32_t(k);
            }
            std::vector<int32_t>().swap(slices[k]);
        }
    }, 1);
    return vox;
}

Domain build_from_source(const Source& src) {
    std::vector<int32_t> vox = voxelise(src, src.z0, src.z1);
    phase("source: voxelise");
    return classify_sites(vox, src.iolets, src.voxel_size);
}

Domain build_pipe(int radius, int length, double voxel_size) {
    return build_from_source(source_pipe(radius, length, voxel_size));
}
Domain build_bifurcation(int tr, int br, int tl, int bl, double voxel_size) {
    return build_from_source(source_bifurcation(tr, br, tl, bl, voxel_size));
}
Domain build_tree(int root_radius, int root_length, int levels, double radius_ratio, double length_ratio,
                  double voxel_size) {
    return build_from_source(source_tree(root_radius, root_length, levels, radius_ratio, length_ratio, voxel_size));
}
Domain build_channel(int nx, int ny, int nz, double voxel_size) {
    return build_from_source(source_channel(nx, ny, nz, voxel_size));
}

SourcePlan plan_source(const Source& src) {
    SourcePlan p;
    if (src.z1 < src.z0) return p;
    const uint64_t ns = uint64_t(int64_t(src.z1) - src.z0 + 1);
    p.plane_count.assign(ns, 0);
    const int nt = hw_threads();
    std::vector<std::array<int32_t, 4>> ext(nt, {INT32_MAX, INT32_MIN, INT32_MAX, INT32_MIN});
    parallel_for(ns, [&](uint64_t b, uint64_t e, int t) {
        std::vector<int32_t> xy;
        for (uint64_t k = b; k < e; ++k) {
            src.slice(src.z0 + int32_t(k), xy);
            p.plane_count[k] = xy.size() / 2;
            for (size_t q = 0; q < xy.size(); q += 2) {
                ext[t][0] = std::min(ext[t][0], xy[q]);
                ext[t][1] = std::max(ext[t][1], xy[q]);
                ext[t][2] = std::min(ext[t][2], xy[q + 1]);
                ext[t][3] = std::max(ext[t][3], xy[q + 1]);
            }
        }
    }, 1);
    p.lo[0] = p.lo[1] = p.lo[2] = INT32_MAX;
    p.hi[0] = p.hi[1] = p.hi[2] = INT32_MIN;
    for (auto& x : ext) {
        p.lo[0] = std::min(p.lo[0], x[0]);
        p.hi[0] = std::max(p.hi[0], x[1]);
        p.lo[1] = std::min(p.lo[1], x[2]);
        p.hi[1] = std::max(p.hi[1], x[3]);
    }
    for (uint64_t k = 0; k < ns; ++k)
        if (p.plane_count[k]) {
            p.n += p.plane_count[k];
            p.lo[2] = std::min(p.lo[2], src.z0 + int32_t(k));
            p.hi[2] = std::max(p.hi[2], src.z0 + int32_t(k));
        }
    return p;
}

Domain classify_slab(const Source& src, int32_t za, int32_t zb, std::vector<uint64_t>* io_links) {
    for (size_t k = 0; k < src.iolets.size(); ++k)
        if (!unit_normal(src.iolets[k]))
            geometry_error("classify_sites: iolet " + std::to_string(k) + " normal is not unit length");
    std::vector<int32_t> vox = voxelise(src, za - 1, zb + 1);  // + one classification-only slice each side
    const uint64_t n = vox.size() / 3;
    for (uint64_t s = 0; s < 3 * n; ++s)
        if (vox[s] < -(int32_t(1) << 20) + 1 || vox[s] >= (int32_t(1) << 20) - 1)
            geometry_error("classify_sites: voxel coordinate out of range");
    std::vector<uint64_t> keys(n);
    parallel_for(n, [&](uint64_t b, uint64_t e, int) {
        for (uint64_t s = b; s < e; ++s) keys[s] = zyx_key(vox[3 * s], vox[3 * s + 1], vox[3 * s + 2]);
    });
    for (uint64_t s = 1; s < n; ++s)
        if (!(keys[s - 1] < keys[s])) geometry_error("classify_slab: source slice not strictly (y, x)-ordered");
    phase("slab: voxelise+keys");
    std::vector<IoletGeo> io(src.iolets);
    SlabKeep keep{za, zb, io_links};
    return classify_sorted(std::move(vox), keys, nullptr, std::move(io), src.voxel_size, &keep);
}

// ---- SPLB v1 file format (geometry_io.hpp:14-129) ----------------------------

namespace {
template <typename T>
void put(std::ostream& os, const T& v) {
    os.write(reinterpret_cast<const char*>(&v), sizeof(T));
}
template <typename T>
T get(std::istream& is) {
    T v;
    is.read(reinterpret_cast<char*>(&v), sizeof(T));
    if (!is) geometry_error("geometry load: truncated file");
    return v;
}
}  // namespace

void write_domain(const Domain& d, const std::string& path) {
    std::ofstream os(path, std::ios::binary);
    if (!os) geometry_error("geometry write: cannot open " + path);
    os.write("SPLB", 4);
    put(os, uint32_t(1));
    put(os, d.voxel_size);
    put(os, uint64_t(d.n));
    put(os, uint32_t(d.iolets.size()));
    for (const IoletGeo& io : d.iolets) {
        put(os, uint8_t(io.kind));
        for (double c : io.center) put(os, c);
        for (double c : io.normal) put(os, c);
        put(os, io.radius);
    }
    size_t lk = 0;
    for (uint64_t s = 0; s < d.n; ++s) {
        for (int a = 0; a < 3; ++a) put(os, d.coords[3 * s + a]);
        put(os, d.types[s]);
        for (int i = 1; i < kQ; ++i) {
            const uint8_t k = d.link_kind[18 * s + uint64_t(i - 1)];
            put(os, k);
            if (k >= 2) {
                while (lk < d.iolet_link_pos.size() && d.iolet_link_pos[lk] < 18 * s + uint64_t(i - 1)) ++lk;
                uint16_t id = 0;
                if (lk < d.iolet_link_pos.size() && d.iolet_link_pos[lk] == 18 * s + uint64_t(i - 1))
                    id = d.iolet_link_id[lk];
                put(os, id);
            }
        }
    }
    if (!os) geometry_error("geometry write: stream failure");
}

Domain read_domain(const std::string& path) {
    std::ifstream is(path, std::ios::binary);
    if (!is) geometry_error("geometry load: cannot open " + path);
    char magic[4];
    is.read(magic, 4);
    if (!is || std::memcmp(magic, "SPLB", 4) != 0) geometry_error("geometry load: not a SPLB file");
    const auto version = get<uint32_t>(is);
    if (version != 1)
        geometry_error("geometry load: version mismatch (file has " + std::to_string(version) +
                       ", expected 1)");
    Domain d;
    d.voxel_size = get<double>(is);
    const auto nsites = get<uint64_t>(is);
    const auto niolets = get<uint32_t>(is);
    d.iolets.resize(niolets);
    for (IoletGeo& io : d.iolets) {
        const auto kind = get<uint8_t>(is);
        if (kind > 1) geometry_error("geometry load: bad iolet kind");
        io.kind = kind;
        for (double& c : io.center) c = get<double>(is);
        for (double& c : io.normal) c = get<double>(is);
        io.radius = get<double>(is);
    }
    d.n = nsites;
    d.coords.resize(3 * nsites);
    d.types.resize(nsites);
    d.link_kind.resize(18 * nsites);
    for (uint64_t s = 0; s < nsites; ++s) {
        for (int a = 0; a < 3; ++a) d.coords[3 * s + a] = get<int32_t>(is);
        const auto type = get<uint8_t>(is);
        if (type >= 6) geometry_error("geometry load: bad collision type");
        d.types[s] = type;
        for (int i = 1; i < kQ; ++i) {
            const auto tag = get<uint8_t>(is);
            if (tag > 3) geometry_error("geometry load: bad link tag");
            d.link_kind[18 * s + uint64_t(i - 1)] = tag;
            if (tag >= 2) {
                const auto id = get<uint16_t>(is);
                d.iolet_link_pos.push_back(18 * s + uint64_t(i - 1));
                d.iolet_link_id.push_back(id);
            }
        }
    }
    uint64_t pos = 0;
    for (int t = 0; t < 6; ++t) {
        d.type_ranges[t][0] = pos;
        while (pos < d.n && int(d.types[pos]) == t) ++pos;
        d.type_ranges[t][1] = pos;
    }
    validate_domain(d);
    return d;
}

// ---- TimeTable (boundary.hpp:18-74) ------------------------------------------

void TimeTable::validate() const {
    if (t.empty()) config_error("time table: empty table");
    for (size_t k = 1; k < t.size(); ++k)
        if (!(t[k] > t[k - 1])) config_error("time table: times must be strictly ascending");
    if (period != 0.0) {
        if (!(period > 0.0)) config_error("time table: period must be > 0");
        if (!(t.back() < period)) config_error("time table: nodes must lie inside one period");
        if (!(t.front() >= 0.0)) config_error("time table: periodic table starts before t=0");
    }
}

double TimeTable::at(double tq) const {
    if (t.size() == 1 && period == 0.0) return v.front();
    double tb = tq;
    if (period > 0.0) {
        tb = std::fmod(tq, period);
        if (tb < 0.0) tb += period;
    }
    for (size_t k = 0; k < t.size(); ++k)
        if (tb == t[k]) return v[k];
    if (period == 0.0) {
        if (tb <= t.front()) return v.front();
        if (tb >= t.back()) return v.back();
    }
    const size_t after = size_t(std::upper_bound(t.begin(), t.end(), tb) - t.begin());
    double t0, v0, t1, v1;
    if (after == 0) {
        t0 = t.back() - period;
        v0 = v.back();
        t1 = t.front();
        v1 = v.front();
    } else if (after == t.size()) {
        t0 = t.back();
        v0 = v.back();
        t1 = t.front() + period;
        v1 = v.front();
    } else {
        t0 = t[after - 1];
        v0 = v[after - 1];
        t1 = t[after];
        v1 = v[after];
    }
    return v0 + (v1 - v0) * ((tb - t0) / (t1 - t0));
}

}  // namespace splbcu
