// Slab domain decomposition (reference decomp.hpp:16-188), bit-exact.
// B200-host changes: per-plane counts in a flat array instead of std::map,
// plane -> owner table, edge detection without a coordinate hash in slab mode
// (a neighbour's owner is a function of its plane), parallel loops.
#include <algorithm>
#include <limits>
#include <numeric>

#include "host.hpp"

namespace splbcu {

double Partition::imbalance() const {
    size_t lo = SIZE_MAX, hi = 0;
    for (const WorkerPart& p : parts) {
        lo = std::min(lo, p.sites.size());
        hi = std::max(hi, p.sites.size());
    }
    return lo == 0 ? std::numeric_limits<double>::infinity() : double(hi) / double(lo);
}

// longest_axis (decomp.hpp:44-56): ties prefer z.
static int longest_axis(const Domain& d) {
    int32_t lo[3] = {INT32_MAX, INT32_MAX, INT32_MAX};
    int32_t hi[3] = {INT32_MIN, INT32_MIN, INT32_MIN};
    for (uint64_t s = 0; s < d.n; ++s)
        for (int a = 0; a < 3; ++a) {
            lo[a] = std::min(lo[a], d.coords[3 * s + a]);
            hi[a] = std::max(hi[a], d.coords[3 * s + a]);
        }
    int best = 2;
    for (int a = 1; a >= 0; --a)
        if (hi[a] - lo[a] > hi[best] - lo[best]) best = a;
    return best;
}

// Greedy plane assignment (decomp.hpp:93-121) over per-plane counts
// (plane plo + k); needs n_workers <= number of non-empty planes.
static std::vector<int32_t> greedy_planes(const std::vector<uint64_t>& plane_count, int32_t plo, uint64_t n,
                                          int n_workers) {
    std::vector<int32_t> planes;  // non-empty planes, ascending (std::map keys)
    for (size_t k = 0; k < plane_count.size(); ++k)
        if (plane_count[k]) planes.push_back(plo + int32_t(k));
    std::vector<int32_t> cut_after;
    size_t it = 0;
    uint64_t remaining_sites = n;
    uint64_t remaining_planes = planes.size();
    for (int w = 0; w < n_workers - 1; ++w) {
        const uint64_t workers_left = uint64_t(n_workers - w);
        const uint64_t target = (remaining_sites + workers_left - 1) / workers_left;
        uint64_t taken = 0, planes_taken = 0;
        while (it != planes.size() && remaining_planes - planes_taken > uint64_t(n_workers - 1 - w)) {
            if (planes_taken > 0 && taken >= target) break;
            taken += plane_count[size_t(planes[it] - plo)];
            ++planes_taken;
            ++it;
        }
        cut_after.push_back(planes[it - 1]);
        remaining_sites -= taken;
        remaining_planes -= planes_taken;
    }
    std::vector<int32_t> owner(plane_count.size(), 0);
    int w = 0;
    for (size_t k = 0; k < plane_count.size(); ++k) {
        const int32_t c = plo + int32_t(k);
        while (w < int(cut_after.size()) && c > cut_after[size_t(w)]) ++w;
        owner[k] = w;
    }
    return owner;
}

// Edge/mid groups, neighbours and type sub-ranges of every part (or only of
// part `only` when >= 0: sites of other owners are then just halo).
static void finish_parts(const Domain& d, Partition& pa, const SiteIndex* index, int only) {
    const uint64_t n = d.n;
    const int n_workers = pa.n_workers;
    const int axis = pa.axis;
    const int32_t plo = pa.plane_lo;
    // Domain-edge sites: any fluid link to a site owned elsewhere (decomp.hpp:132-153).
    SiteIndex local_ix;
    if (!pa.slab && !index) {
        local_ix = index_domain(d);
        index = &local_ix;
    }
    std::vector<uint8_t> is_edge(n, 0);
    const int nt = hw_threads();
    std::vector<std::vector<std::pair<int, int>>> nbs(nt);
    parallel_for(n, [&](uint64_t b, uint64_t e, int t) {
        for (uint64_t s = b; s < e; ++s) {
            const int32_t* c = &d.coords[3 * s];
            const int ow = pa.owner[s];
            if (only >= 0 && ow != only) continue;
            for (int i = 1; i < kQ; ++i) {
                if (d.link_kind[18 * s + uint64_t(i - 1)] != 0) continue;
                int ot;
                if (pa.slab) {
                    const int dc = axis == 0 ? cx(i) : (axis == 1 ? cy(i) : cz(i));
                    ot = pa.plane_owner[size_t(c[axis] + dc - plo)];
                } else {
                    const int64_t p = index->find(c[0] + cx(i), c[1] + cy(i), c[2] + cz(i));
                    if (p < 0) runtime_error("partition: fluid link to a missing site");
                    ot = pa.owner[index->value[size_t(p)]];
                }
                if (ot != ow) {
                    is_edge[s] = 1;
                    if (nbs[t].empty() || nbs[t].back() != std::make_pair(ow, ot)) nbs[t].push_back({ow, ot});
                }
            }
        }
    });
    std::vector<std::pair<int, int>> allnb;
    for (auto& v : nbs) allnb.insert(allnb.end(), v.begin(), v.end());
    std::sort(allnb.begin(), allnb.end());
    allnb.erase(std::unique(allnb.begin(), allnb.end()), allnb.end());

    // Worker-local order: edge group then mid group, ascending global index
    // inside each (decomp.hpp:155-186).
    pa.parts.resize(size_t(n_workers));
    pa.local_index.assign(n, 0);
    {
        std::vector<uint64_t> ne(size_t(n_workers), 0), nm(size_t(n_workers), 0);
        for (uint64_t s = 0; s < n; ++s) (is_edge[s] ? ne : nm)[size_t(pa.owner[s])]++;
        if (only >= 0)
            for (int w = 0; w < n_workers; ++w)
                if (w != only) ne[size_t(w)] = nm[size_t(w)] = 0;
        for (int w = 0; w < n_workers; ++w) {
            pa.parts[size_t(w)].sites.resize(ne[size_t(w)] + nm[size_t(w)]);
            pa.parts[size_t(w)].n_edge = uint32_t(ne[size_t(w)]);
        }
        std::vector<uint64_t> pe(size_t(n_workers), 0), pm(ne);
        for (uint64_t s = 0; s < n; ++s) {
            const size_t w = size_t(pa.owner[s]);
            if (only >= 0 && int(w) != only) continue;
            const uint64_t k = is_edge[s] ? pe[w]++ : pm[w]++;
            pa.parts[w].sites[k] = uint32_t(s);
            pa.local_index[s] = uint32_t(k);
        }
    }
    for (auto& p : allnb) pa.parts[size_t(p.first)].neighbors.push_back(p.second);
    for (int w = 0; w < n_workers; ++w) {
        WorkerPart& part = pa.parts[size_t(w)];
        auto fill = [&](uint64_t begin, uint64_t end, uint64_t out[6][2]) {
            uint64_t pos = begin;
            for (int t = 0; t < 6; ++t) {
                out[t][0] = pos;
                while (pos < end && int(d.types[part.sites[pos]]) == t) ++pos;
                out[t][1] = pos;
            }
        };
        fill(0, part.n_edge, part.edge_ranges);
        fill(part.n_edge, part.sites.size(), part.mid_ranges);
    }
}

Partition partition(const Domain& d, int n_workers, const SiteIndex* index) {
    const uint64_t n = d.n;
    if (n_workers < 1) runtime_error("partition: nWorkers must be >= 1");
    if (uint64_t(n_workers) > n)
        runtime_error("partition: nWorkers (" + std::to_string(n_workers) + ") exceeds site count (" +
                      std::to_string(n) + ")");
    Partition pa;
    pa.n_workers = n_workers;
    pa.owner.assign(n, 0);
    const int axis = longest_axis(d);
    pa.axis = axis;

    int32_t plo = INT32_MAX, phi = INT32_MIN;
    for (uint64_t s = 0; s < n; ++s) {
        plo = std::min(plo, d.coords[3 * s + axis]);
        phi = std::max(phi, d.coords[3 * s + axis]);
    }
    std::vector<uint64_t> plane_count(size_t(int64_t(phi) - plo + 1), 0);
    for (uint64_t s = 0; s < n; ++s) ++plane_count[size_t(d.coords[3 * s + axis] - plo)];
    std::vector<int32_t> planes;  // non-empty planes, ascending (std::map keys)
    for (size_t k = 0; k < plane_count.size(); ++k)
        if (plane_count[k]) planes.push_back(plo + int32_t(k));

    if (uint64_t(n_workers) <= planes.size()) {
        pa.slab = true;
        pa.plane_lo = plo;
        pa.plane_owner = greedy_planes(plane_count, plo, n, n_workers);
        parallel_for(n, [&](uint64_t b, uint64_t e, int) {
            for (uint64_t s = b; s < e; ++s) pa.owner[s] = pa.plane_owner[size_t(d.coords[3 * s + axis] - plo)];
        });
    } else {
        // Contiguous balanced split of the (axis, z, y, x) order (decomp.hpp:122-130).
        pa.slab = false;
        std::vector<uint32_t> order(n);
        std::iota(order.begin(), order.end(), 0u);
        std::sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) {
            const int32_t* ca = &d.coords[3 * uint64_t(a)];
            const int32_t* cb = &d.coords[3 * uint64_t(b)];
            if (ca[axis] != cb[axis]) return ca[axis] < cb[axis];
            if (ca[2] != cb[2]) return ca[2] < cb[2];
            if (ca[1] != cb[1]) return ca[1] < cb[1];
            return ca[0] < cb[0];
        });
        const uint64_t q = n / uint64_t(n_workers), r = n % uint64_t(n_workers);
        uint64_t pos = 0;
        for (int w = 0; w < n_workers; ++w) {
            const uint64_t take = q + (uint64_t(w) < r ? 1 : 0);
            for (uint64_t k = 0; k < take; ++k) pa.owner[order[pos++]] = w;
        }
    }

    finish_parts(d, pa, index, -1);
    return pa;
}

// ---- slab-local construction -------------------------------------------------

int32_t SlabPlan::own_lo(int w) const {
    for (size_t k = 0; k < plane_owner.size(); ++k)
        if (plane_owner[k] == w) return plane_lo + int32_t(k);
    return plane_lo;
}
int32_t SlabPlan::own_hi(int w) const {
    for (size_t k = plane_owner.size(); k-- > 0;)
        if (plane_owner[k] == w) return plane_lo + int32_t(k);
    return plane_lo - 1;
}

SlabPlan plan_slabs(const SourcePlan& sp, int32_t z0, int n_workers) {
    SlabPlan p;
    p.n = sp.n;
    if (n_workers < 1) runtime_error("partition: nWorkers must be >= 1");
    if (uint64_t(n_workers) > sp.n)
        runtime_error("partition: nWorkers (" + std::to_string(n_workers) + ") exceeds site count (" +
                      std::to_string(sp.n) + ")");
    // longest_axis (decomp.hpp:44-56), ties prefer z: slabs only along z
    int best = 2;
    for (int a = 1; a >= 0; --a)
        if (sp.hi[a] - sp.lo[a] > sp.hi[best] - sp.lo[best]) best = a;
    if (best != 2) return p;
    const size_t k0 = size_t(sp.lo[2] - z0), k1 = size_t(sp.hi[2] - z0);
    p.plane_lo = sp.lo[2];
    p.plane_count.assign(sp.plane_count.begin() + int64_t(k0), sp.plane_count.begin() + int64_t(k1) + 1);
    uint64_t nonempty = 0;
    for (uint64_t c : p.plane_count) nonempty += c != 0;
    if (uint64_t(n_workers) > nonempty) return p;  // contiguous fallback split: needs the whole domain
    p.plane_owner = greedy_planes(p.plane_count, p.plane_lo, p.n, n_workers);
    p.ok = true;
    return p;
}

Window classify_window(const Source& src, const SlabPlan& plan, int worker, std::vector<uint64_t>* own_counts,
                       std::vector<uint64_t>* io_links) {
    Window w;
    w.worker = worker;
    w.own_lo = plan.own_lo(worker);
    w.own_hi = plan.own_hi(worker);
    w.n_global = plan.n;
    w.dom = classify_slab(src, w.own_lo - 1, w.own_hi + 1, nullptr);
    const Domain& d = w.dom;
    const uint64_t ns = uint64_t(int64_t(w.own_hi) - w.own_lo + 1);
    if (own_counts) {
        own_counts->assign(6 * ns, 0);
        for (uint64_t s = 0; s < d.n; ++s) {
            const int32_t z = d.coords[3 * s + 2];
            if (z >= w.own_lo && z <= w.own_hi) ++(*own_counts)[6 * uint64_t(z - w.own_lo) + d.types[s]];
        }
    }
    if (io_links) {
        io_links->assign(d.iolets.size(), 0);
        for (size_t q = 0; q < d.iolet_link_pos.size(); ++q) {
            const int32_t z = d.coords[3 * (d.iolet_link_pos[q] / 18) + 2];
            if (z >= w.own_lo && z <= w.own_hi) ++(*io_links)[d.iolet_link_id[q]];
        }
    }
    return w;
}

void finish_window(Window& w, const SlabPlan& plan, const std::vector<uint64_t>& counts) {
    const size_t np = plan.plane_owner.size();
    if (counts.size() != 6 * np) runtime_error("slab build: per-slice type counts have the wrong shape");
    uint64_t tot[6] = {}, below[6] = {};
    for (size_t k = 0; k < np; ++k) {
        uint64_t c = 0;
        for (int t = 0; t < 6; ++t) {
            tot[t] += counts[6 * k + size_t(t)];
            c += counts[6 * k + size_t(t)];
            if (plan.plane_lo + int32_t(k) < w.own_lo - 1) below[t] += counts[6 * k + size_t(t)];
        }
        if (c != plan.plane_count[k]) runtime_error("slab build: slice counts disagree between ranks");
    }
    uint64_t pos = 0;
    for (int t = 0; t < 6; ++t) {
        w.g_type_ranges[t][0] = pos;
        pos += tot[t];
        w.g_type_ranges[t][1] = pos;
        w.g_first[t] = w.g_type_ranges[t][0] + below[t];
    }
    if (pos != plan.n) runtime_error("slab build: site count mismatch");
    w.n_global = pos;
}

Partition partition_window(const Window& w, const SlabPlan& plan, int n_workers) {
    const Domain& d = w.dom;
    Partition pa;
    pa.n_workers = n_workers;
    pa.axis = 2;
    pa.slab = true;
    pa.plane_lo = plan.plane_lo;
    pa.plane_owner = plan.plane_owner;
    pa.owner.assign(d.n, 0);
    parallel_for(d.n, [&](uint64_t b, uint64_t e, int) {
        for (uint64_t s = b; s < e; ++s) pa.owner[s] = pa.plane_owner[size_t(d.coords[3 * s + 2] - pa.plane_lo)];
    });
    finish_parts(d, pa, nullptr, w.worker);
    return pa;
}

}  // namespace splbcu
