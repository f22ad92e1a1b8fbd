// B200 engine: GPU-resident workers, device-built neighbour table, fused
// collide+stream kernels, edge-then-inner overlap with the halo exchange
// (peer copies in-process, NCCL send/recv across processes).
//
// Reference: splb::Simulation (proj/include/splb/engine.hpp:121-650),
// build_streaming_map (layout.hpp:181-286), build_exchange_plan
// (exchange.hpp:36-83).
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <atomic>
#include <thread>

#include <cub/device/device_radix_sort.cuh>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: host ranges for Nsight tools, no-ops otherwise

#include "engine.hpp"
#include "kernels.cuh"
#include "nccl_dyn.hpp"

namespace splbcu {

// Host-side NVTX range (setup, run, each step's enqueue) for Nsight Systems /
// ncu --nvtx filtering (SURVEY §5 tracing).
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

#define CK(x)                                                                                \
    do {                                                                                     \
        cudaError_t e_ = (x);                                                                \
        if (e_ != cudaSuccess)                                                               \
            fail(ErrKind::Cuda, std::string("CUDA error: ") + cudaGetErrorString(e_) + " (" + \
                                    #x + ")");                                               \
    } while (0)

#define NK(x)                                                                                   \
    do {                                                                                        \
        ncclResult_t r_ = (x);                                                                  \
        if (r_ != ncclSuccess)                                                                  \
            fail(ErrKind::Comm, std::string("exchange failure: NCCL error: ") + nccl().GetErrorString(r_)); \
    } while (0)

static const NcclApi& nccl_checked() {
    const NcclApi& a = nccl();
    if (!a.ok) fail(ErrKind::Comm, "exchange failure: NCCL unavailable:" + a.error);
    return a;
}

std::string nccl_unique_id(void* out128) {
    ncclUniqueId id;
    NK(nccl_checked().GetUniqueId(&id));
    std::memcpy(out128, &id, sizeof(id));
    return {};
}

constexpr uint64_t kTilePad = 256;  // tail pad so the last TMA tile stays in bounds

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        CK(cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q));
        if (!p || q != cudaDriverEntryPointSuccess) fail(ErrKind::Cuda, "cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

// Stream memory operations (driver API) for the P2P halo's step flags.
using StreamValueFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
struct StreamMemOps {
    StreamValueFn wait = nullptr, write = nullptr;
};
static const StreamMemOps& stream_mem_ops() {
    static StreamMemOps ops = [] {
        StreamMemOps o;
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPointByVersion("cuStreamWaitValue32", &p, 12000, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            o.wait = reinterpret_cast<StreamValueFn>(p);
        p = nullptr;
        if (cudaGetDriverEntryPointByVersion("cuStreamWriteValue32", &p, 12000, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            o.write = reinterpret_cast<StreamValueFn>(p);
        return o;
    }();
    if (!ops.wait || !ops.write) fail(ErrKind::Cuda, "stream memory operations unavailable");
    return ops;
}
static void wait_geq(cudaStream_t s, const uint32_t* addr, uint32_t v) {
    const CUresult r = stream_mem_ops().wait(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(addr), v,
                                             CU_STREAM_WAIT_VALUE_GEQ);
    if (r != CUDA_SUCCESS) fail(ErrKind::Cuda, "cuStreamWaitValue32 failed (" + std::to_string(int(r)) + ")");
}
static void write_flag(cudaStream_t s, uint32_t* addr, uint32_t v) {
    // default flags: the write is ordered after the stream's prior work and
    // preceded by a memory barrier, so the halo stores are visible first
    const CUresult r = stream_mem_ops().write(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(addr), v,
                                              CU_STREAM_WRITE_VALUE_DEFAULT);
    if (r != CUDA_SUCCESS) fail(ErrKind::Cuda, "cuStreamWriteValue32 failed (" + std::to_string(int(r)) + ")");
}

// 2-D map over `planes` direction planes of pitch P: dim0 = site, dim1 = plane;
// one box = `box` sites x all planes.
static void encode_planes(CUtensorMap* m, void* base, bool f64, int planes, uint64_t P, uint32_t box) {
    std::memset(m, 0, sizeof(*m));
    const cuuint64_t dims[2] = {cuuint64_t(P), cuuint64_t(planes)};
    const cuuint64_t strides[1] = {cuuint64_t(P * (f64 ? 8 : 4))};
    const cuuint32_t boxd[2] = {box, cuuint32_t(planes)};
    const cuuint32_t es[2] = {1, 1};
    const CUresult r = encode_fn()(m, f64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, base,
                                   dims, strides, boxd, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail(ErrKind::Cuda, "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
}

namespace {

// SPLBCU_TRACE: host-side progress lines on stderr (run enqueue, watchdog).
static const bool g_trace = std::getenv("SPLBCU_TRACE") != nullptr;
#define TRACE(...)                                        \
    do {                                                  \
        if (g_trace) {                                    \
            std::fprintf(stderr, "[splbcu] " __VA_ARGS__); \
            std::fflush(stderr);                          \
        }                                                 \
    } while (0)

// Set once an exchange failure has left streams blocked on a dead
// neighbour's flags: freeing device or pinned memory would then wait on those
// streams forever (cudaFree synchronises the device), so the buffers of the
// failed engine are leaked instead and the caller can report and exit.
static std::atomic<bool> g_leak_on_free{false};

struct DevMem {
    void* p = nullptr;
    size_t bytes = 0;
    DevMem() = default;
    DevMem(const DevMem&) = delete;
    DevMem& operator=(const DevMem&) = delete;
    ~DevMem() { release(); }
    void release() {
        if (p && !g_leak_on_free.load()) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
    template <class T>
    T* alloc(size_t n) {
        release();
        bytes = std::max<size_t>(n * sizeof(T), 16);
        CK(cudaMalloc(&p, bytes));
        return static_cast<T*>(p);
    }
    // Keeps the allocation when it is already large enough (no cudaFree /
    // cudaMalloc, which synchronise the device, on the per-run path).
    template <class T>
    T* reserve(size_t n) {
        if (!p || bytes < n * sizeof(T)) return alloc<T>(n);
        return static_cast<T*>(p);
    }
    template <class T>
    T* get() const { return static_cast<T*>(p); }
};

// Page-locked host buffer (portable across the process's devices) so the
// per-run staging H2D and observation D2H are true async DMA.
struct PinnedMem {
    void* p = nullptr;
    size_t bytes = 0;
    PinnedMem() = default;
    PinnedMem(const PinnedMem&) = delete;
    PinnedMem& operator=(const PinnedMem&) = delete;
    ~PinnedMem() {
        if (p && !g_leak_on_free.load()) cudaFreeHost(p);
    }
    template <class T>
    T* reserve(size_t n) {
        const size_t need = std::max<size_t>(n * sizeof(T), 16);
        if (!p || bytes < need) {
            if (p) cudaFreeHost(p);
            p = nullptr;
            bytes = 0;
            CK(cudaHostAlloc(&p, need, cudaHostAllocPortable));
            bytes = need;
        }
        return static_cast<T*>(p);
    }
    template <class T>
    T* get() const { return static_cast<T*>(p); }
};

template <class T>
T* upload(DevMem& m, const std::vector<T>& v, cudaStream_t s) {
    T* d = m.alloc<T>(v.size());
    if (!v.empty()) CK(cudaMemcpyAsync(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s));
    return d;
}

inline unsigned blocks_for(uint64_t n, unsigned tpb = 256) { return unsigned((n + tpb - 1) / tpb); }

// ---- device lookup over the worker's own + halo sites ----------------------
struct DLookup {
    const uint64_t* keys;
    const int32_t* owner;
    const uint32_t* local;   // internal index when owner == this worker
    const uint32_t* global;  // global site index
    uint64_t n;
    const uint64_t* row_off;  // null: whole-array binary search
    int32_t lo1, hi1, lo2, hi2;
    int64_t ny;
};

__device__ __forceinline__ uint64_t d_zyx_key(int32_t x, int32_t y, int32_t z) {
    const int64_t b = int64_t(1) << 20;
    return (uint64_t(int64_t(z) + b) << 42) | (uint64_t(int64_t(y) + b) << 21) | uint64_t(int64_t(x) + b);
}

__device__ int64_t d_find(const DLookup& L, int32_t x, int32_t y, int32_t z) {
    const uint64_t key = d_zyx_key(x, y, z);
    uint64_t b = 0, e = L.n;
    if (L.row_off) {
        if (y < L.lo1 || y > L.hi1 || z < L.lo2 || z > L.hi2) return -1;
        const uint64_t r = uint64_t(int64_t(z - L.lo2) * L.ny + (y - L.lo1));
        b = L.row_off[r];
        e = L.row_off[r + 1];
    }
    while (b < e) {
        const uint64_t m = (b + e) >> 1;
        if (L.keys[m] < key) b = m + 1;
        else e = m;
    }
    return (b < L.n && L.keys[b] == key) ? int64_t(b) : -1;
}

// Neighbour table build (build_streaming_map, layout.hpp:181-286), one
// thread per (site, direction).  Cross-worker links are collected with the
// reference's canonical sort key (neighbour, sender global site, direction)
// and slotted after a device radix sort.
__global__ void build_links(uint32_t n, uint64_t P, const int32_t* __restrict__ coords,
                            const uint8_t* __restrict__ kind, const uint32_t* __restrict__ gidx,
                            int32_t w, DLookup L, uint32_t* __restrict__ tab,
                            unsigned long long* out_keys, unsigned long long* out_vals, unsigned* n_out,
                            unsigned long long* in_keys, unsigned long long* in_vals, unsigned* n_in,
                            unsigned* err) {
    const uint64_t idx = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= uint64_t(n) * 18) return;
    const uint32_t s = uint32_t(idx / 18);
    const int i = int(idx % 18) + 1;
    const int32_t x = coords[3 * uint64_t(s)], y = coords[3 * uint64_t(s) + 1], z = coords[3 * uint64_t(s) + 2];
    const uint8_t k = kind[18 * uint64_t(s) + uint64_t(i - 1)];
    const uint64_t tpos = uint64_t(i - 1) * P + s;
    if (k == 0) {
        const int64_t e = d_find(L, x + cx(i), y + cy(i), z + cz(i));
        if (e < 0) {
            atomicExch(err, 1u);
            return;
        }
        const int32_t o = L.owner[e];
        if (o == w) {
            tab[tpos] = L.local[e];
        } else {
            const unsigned p = atomicAdd(n_out, 1u);
            out_keys[p] = (static_cast<unsigned long long>(o) << 40) |
                          (static_cast<unsigned long long>(gidx[s]) * 18ull + unsigned(i - 1));
            out_vals[p] = tpos;
            tab[tpos] = kSpecial | (kOpShared << kOpShift);
        }
    } else if (k == 1) {
        tab[tpos] = kSpecial | (kOpBounce << kOpShift);
    } else {
        tab[tpos] = kSpecial | (kOpIolet << kOpShift);  // id patched below
    }
    // Incoming partner: the fluid site at x - c_i (this site's link inv(i)
    // is Fluid) streams into (s, i); record it when another worker owns it.
    if (kind[18 * uint64_t(s) + uint64_t(inv(i) - 1)] == 0) {
        const int64_t src = d_find(L, x - cx(i), y - cy(i), z - cz(i));
        if (src < 0) {
            atomicExch(err, 1u);
            return;
        }
        if (L.owner[src] != w) {
            const unsigned p = atomicAdd(n_in, 1u);
            in_keys[p] = (static_cast<unsigned long long>(L.owner[src]) << 40) |
                         (static_cast<unsigned long long>(L.global[src]) * 18ull + unsigned(i - 1));
            in_vals[p] = uint64_t(i) * P + s;
        }
    }
}

__global__ void patch_iolets(const uint64_t* __restrict__ pos, const uint16_t* __restrict__ id, uint32_t n,
                             uint32_t* __restrict__ tab) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n) tab[pos[k]] = kSpecial | (kOpIolet << kOpShift) | id[k];
}

__global__ void assign_slots(const unsigned long long* __restrict__ out_vals, const unsigned long long* __restrict__ in_vals,
                             uint32_t n, uint32_t* __restrict__ tab, uint64_t* __restrict__ recv_flat,
                             uint64_t* __restrict__ send_pos) {
    const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    tab[out_vals[r]] = kSpecial | (kOpShared << kOpShift) | r;
    send_pos[r] = out_vals[r];
    recv_flat[r] = in_vals[r];
}

struct Seg {
    int nb;
    uint32_t base, count;
};

}  // namespace

// ---------------------------------------------------------------------------
struct WorkerDev {
    int w = 0, dev = 0;
    cudaStream_t sE = nullptr, sM = nullptr;
    cudaStream_t sS = nullptr;  // dist mode: the series reduction beside the next run
    cudaEvent_t evSend = nullptr, evMid = nullptr, evEnd = nullptr;
    // run() bracket + host-copy completion, one set per run in flight (Engine::run_par)
    cudaEvent_t evRun0[2] = {}, evRun1[2] = {}, evDone[2] = {};
    cudaEvent_t evObsFree[2] = {};  // a run's observation rows gathered (N=1) / all-gathered (dist)
    cudaEvent_t evSerRead[2] = {};  // dist: the series gather has read the all-gathered rows
    PinnedMem h_obs;                                                   // observation rows, D2H target
    uint32_t n = 0, n_edge = 0, ep = 0, mp = 0;  // ranges: [0,ep) [ep,n_edge) [n_edge,n_edge+mp) [.., n)
    uint64_t P = 0;
    uint32_t shared = 0;
    std::vector<uint32_t> ref_of_int, int_of_ref, global_of_int;
    DevMem fbuf[2];
    int old = 0;
    DevMem tab, recv_flat, send_pos, io_coords, io_geo, staged, cap4, obs_site, obs_iolet, obs_buf;
    std::vector<Seg> segs;
    // observation: per iolet k, the internal sites in ascending global order
    std::vector<std::vector<uint32_t>> obs_sites;
    std::vector<uint32_t> obs_off;  // flattened offsets per iolet
    uint32_t n_obs = 0;
    uint64_t obs_row_base = 0, obs_rows = 0;
    // kernel timing (bulk launches), one list per run in flight
    std::vector<cudaEvent_t> tev[2];
    // end of each step in flight (ring of Engine::kDepth): the run()
    // watchdog's progress marks
    std::vector<cudaEvent_t> prog;
    // Online choice of the bulk (mid) plain kernel: just-in-time table loads
    // with a dynamic tile order (mid_pick 0), the prefetch kernel (1) or the
    // run-length table (2).  All give the same bits; which
    // is faster depends on the geometry and on the flow (from rest vs developed,
    // DESIGN §3), so every kTuneEvery mid launches the next 2 x kTuneReps
    // launches alternate the two under CUDA events and the faster is kept.
    static constexpr int kTuneReps = 3;
    static constexpr int kCand = 3;  // bulk-kernel candidates: 0 just-in-time, 1 prefetch, 2 run table
    static constexpr uint64_t kTuneEvery = 500;
    int mid_pick = 0;
    int tune_phase = 0;         // 0: exploit; k > 0: measuring launch k-1
    bool tune_pending = false;  // measured, events not read yet
    uint64_t mid_launches = 0;
    cudaEvent_t tune_ev[kCand * kTuneReps][2] = {};
    int n_cand = 2;  // candidates available on this worker (3 with a run table)
    // 2-D tensor maps over the direction-major planes (per f buffer, table)
    CUtensorMap tm_f[2][2];  // [buffer][box T variant: 0 -> 128 sites, 1 -> 256 sites]
    CUtensorMap tm_t[2];
    bool tma_ok = false;  // maps encoded (planes at least one box long)
    // compressed table of the mid-group plain range (kernels.cuh: compress_table)
    DevMem dtab, gbase;
    DevMem ctile;  // tile-major copy of dtab/gbase (T = 256), see build_table_tiles
    DevMem rtab;   // run-length table of the mid-group plain range (T = 256), see build_run_table
    DevMem tile_ctr;  // dynamic tile counters of the bulk launches of one step (lbm_push_dyn)
    uint32_t ctr_used = 0;
    bool rtab_ok = false;
    uint32_t rtab_escaped = 0;  // (direction, group)s read from the u32 table
    uint64_t PG = 0;
    bool ctab_ok = false;
    // fused P2P halo: per shared slot the neighbour index and final flat
    // destination; neighbours' f buffers and flag words (peer-mapped)
    DevMem slot_peer, slot_dst, flags;  // flags: [0,W) halo_in from v, [W,2W) peer_done of v
    std::vector<std::array<double*, 2>> peer_f;  // by segment index
    std::vector<uint32_t*> peer_flags;           // by segment index
    std::vector<void*> ipc_opened;               // dist mode: handles to close
    size_t tev_used[2] = {0, 0};

    double* f_old() const { return fbuf[old].get<double>(); }
    double* f_new() const { return fbuf[1 - old].get<double>(); }
    uint64_t fsize() const { return uint64_t(kQ) * P + shared; }
};

class Engine {
  public:
    Domain dom;
    std::vector<BCEntry> bcs;
    Params prm;
    double omega = 0.0;
    Partition part;
    std::vector<std::unique_ptr<WorkerDev>> W;  // index = worker id; null if not local
    bool dist = false;
    int rank = 0, nranks = 1;
    ncclComm_t comm = nullptr;
    std::vector<Capture> caps;
    Series series;
    DevMem obs_gather;   // dist mode: every rank's observation rows (padded)
    PinnedMem h_gather;
    // device-side series (reduce_series_async): entry lists in series order
    bool dev_series = false;
    uint32_t n_series_ent = 0, ser_host_ent = 0;
    std::vector<uint32_t> ser_host_k, ser_dev_k, ser_be;  // iolets reduced on host / device; entry ranges
    DevMem ser_w, ser_idx, ser_off, ser_tot, ser_kdev, ser_buf, ser_out;
    // double-buffered so a run's copies never land in the batch the host is
    // still reducing: the long iolets of run k are reduced on the host while
    // run k+1's steps execute (lazily, at the next run() or series() call)
    PinnedMem h_series[2], h_series_raw[2];
    int ser_next = 0;                 // buffer the next run's copies go to
    bool ser_pending = false;         // a run's batch awaits host reduction
    int ser_pend_buf = 0;
    uint64_t ser_pend_rows = 0;       // series rows once that batch is in

    uint64_t series_d2h_bytes() const {
        if (!prm.observe_iolets) return 0;
        if (dev_series) return 24 * (uint64_t(dom.iolets.size()) + ser_host_ent);
        uint64_t n = 0;  // host path: every local worker's rows
        for (auto& wp : W)
            if (wp) n += wp->n_obs;
        return 24 * n;
    }

    // dist mode: elements per rank in the padded all-gather of observation
    // rows (every rank's obs_buf is reserved to this size)
    uint64_t obs_gather_per(const WorkerDev& wk) const {
        const size_t n_io = dom.iolets.size();
        uint64_t maxn = 1;
        for (auto& o : obs_off_all) maxn = std::max<uint64_t>(maxn, o[n_io]);
        return 3 * wk.obs_rows * maxn;
    }
    std::vector<std::vector<std::pair<int, uint32_t>>> obs_order;  // per iolet: (worker, pos)
    std::vector<std::vector<uint32_t>> obs_off_all;  // per worker: per-iolet offsets (+ total), all workers
    uint64_t steps_run = 0;
    double loop_s = 0.0, dev_loop_s = 0.0, plain_s = 0.0;
    uint64_t plain_launches = 0, plain_sites = 0, launches = 0;
    bool kernel_timing = false;
    bool p2p_mode = false;
    bool aa_mode = false;  // single-buffer AA storage (params.storage == 1)
    bool pull_mode = false;  // scheme == pull with two buffers: update_pull + fill_send_slots
    std::vector<IoletDev> io_host;
    std::unique_ptr<Window> win;  // slab-local build: dom holds this rank's window only
    uint64_t n_global = 0;        // sites of the whole domain

    Engine(const Domain& d, std::vector<BCEntry> b, Params p, int rank_, int nranks_, const void* nccl_id)
        : dom(d), bcs(std::move(b)), prm(std::move(p)) {
        begin(rank_, nranks_, nccl_id);
        validate_setup();
        part = splbcu::partition(dom, prm.workers);
        n_global = dom.n;
        finish_setup();
    }

    // Distributed engine over a geometry source: when the
    // reference partition is a z-slab split, each rank classifies only its
    // own slices plus one halo slice on each side; per-slice type counts are
    // all-gathered to place its sites in the global order.  Otherwise (and
    // in-process) the whole domain is built, exactly as the builders do.
    Engine(const Source& src, std::vector<BCEntry> b, Params p, int rank_, int nranks_, const void* nccl_id)
        : bcs(std::move(b)), prm(std::move(p)) {
        begin(rank_, nranks_, nccl_id);
        SlabPlan plan;
        if (dist) {
            const SourcePlan sp = plan_source(src);
            phase("slab: plan");
            plan = plan_slabs(sp, src.z0, prm.workers);
        }
        if (!plan.ok) {
            dom = build_from_source(src);
            validate_setup();
            part = splbcu::partition(dom, prm.workers);
            n_global = dom.n;
        } else {
            std::vector<uint64_t> own, io_links;
            win = std::make_unique<Window>(classify_window(src, plan, rank, &own, &io_links));
            phase("slab: classify window");
            // every slice's per-type counts, in worker (= slice) order
            const std::vector<std::vector<uint64_t>> all = allgather_setup(own);
            std::vector<uint64_t> counts;
            for (auto& v : all) counts.insert(counts.end(), v.begin(), v.end());
            finish_window(*win, plan, counts);
            // classify_sites' global check (geometry.hpp:199-206): every iolet has links somewhere
            const std::vector<std::vector<uint64_t>> links = allgather_setup(io_links);
            for (size_t k = 0; k < src.iolets.size(); ++k) {
                uint64_t c = 0;
                for (auto& v : links) c += v[k];
                if (c == 0)
                    geometry_error("classify_sites: iolet " + std::to_string(k) + " intersects no boundary links");
            }
            part = partition_window(*win, plan, prm.workers);
            phase("slab: partition");
            dom = std::move(win->dom);  // the engine's domain is the window
            win->dom = Domain{};
            n_global = win->n_global;
            validate_params();
        }
        finish_setup();
    }

    // Global site index of a site of `dom` (identity unless slab-local).
    uint64_t global_of_site(uint64_t s) const {
        if (!win) return s;
        const int t = dom.types[s];
        return win->g_first[t] + (s - dom.type_ranges[t][0]);
    }

    // Host all-gather of one vector per rank (lengths may differ), usable
    // before the workers exist.
    std::vector<std::vector<uint64_t>> allgather_setup(const std::vector<uint64_t>& mine) {
        CK(cudaSetDevice(prm.devices[0]));
        cudaStream_t s = nullptr;
        CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        DevMem a, b;
        auto gather = [&](const std::vector<uint64_t>& v, size_t per) {
            uint64_t* da = a.reserve<uint64_t>(per);
            uint64_t* db = b.reserve<uint64_t>(per * size_t(nranks));
            CK(cudaMemsetAsync(da, 0, per * 8, s));
            if (!v.empty()) CK(cudaMemcpyAsync(da, v.data(), v.size() * 8, cudaMemcpyHostToDevice, s));
            NK(nccl().AllGather(da, db, per, ncclUint64, comm, s));
            std::vector<uint64_t> h(per * size_t(nranks));
            CK(cudaMemcpyAsync(h.data(), db, h.size() * 8, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            return h;
        };
        const std::vector<uint64_t> len = gather({uint64_t(mine.size())}, 1);
        size_t per = 1;
        for (uint64_t l : len) per = std::max<size_t>(per, size_t(l));
        const std::vector<uint64_t> all = gather(mine, per);
        CK(cudaStreamDestroy(s));
        std::vector<std::vector<uint64_t>> out{size_t(nranks)};
        for (int r = 0; r < nranks; ++r)
            out[size_t(r)].assign(all.begin() + int64_t(per) * r, all.begin() + int64_t(per) * r + int64_t(len[size_t(r)]));
        return out;
    }

    void begin(int rank_, int nranks_, const void* nccl_id) {
        dist = nccl_id != nullptr;
        if (!variant_built(plain_variant))
            config_error("engine: SPLBCU_PLAIN_VARIANT " + std::to_string(plain_variant) +
                         " is a tuning variant, not built (make TUNING=1)");
        rank = rank_;
        nranks = nranks_;
        aa_mode = prm.storage == 1;
        pull_mode = prm.scheme == 1 && !aa_mode;
        if (prm.devices.empty()) {
            int cur = 0;
            CK(cudaGetDevice(&cur));
            prm.devices.push_back(cur);
        }
        if (dist) {
            // Join the communicator first: every rank reaches this point at
            // the same time, before the (long) per-rank table build.
            if (nranks != prm.workers) config_error("engine: dist mode needs workers == nranks");
            CK(cudaSetDevice(prm.devices[0]));
            ncclUniqueId id;
            std::memcpy(&id, nccl_id, sizeof(id));
            NK(nccl_checked().CommInitRank(&comm, nranks, id, rank));
        }
    }

    void finish_setup() {
        NvtxRange nv("splbcu::setup");
        omega = 1.0 / prm.tau;  // RelaxationParams (lattice.hpp:83-84), dt = 1
        for (auto& g : dom.iolets) {
            IoletDev x{};
            for (int a = 0; a < 3; ++a) x.center[a] = g.center[a], x.normal[a] = g.normal[a];
            x.radius = g.radius;
            io_host.push_back(x);
        }
        for (size_t k = 0; k < bcs.size(); ++k) io_host[k].is_velocity = bcs[k].kind == 1;

        const SiteIndex ix = index_domain(dom);
        W.resize(size_t(prm.workers));
        for (int w = 0; w < prm.workers; ++w) {
            if (dist && w != rank) continue;
            const int dev = dist ? prm.devices[0] : prm.devices[size_t(w) % prm.devices.size()];
            W[size_t(w)] = std::make_unique<WorkerDev>();
            setup_worker(*W[size_t(w)], w, dev, ix);
        }
        if (!dist) {
            // exchange plan cross-check (exchange.hpp:43-83): both endpoints agree
            for (int w = 0; w < prm.workers; ++w)
                for (const Seg& sg : W[size_t(w)]->segs) {
                    const Seg* peer = find_seg(*W[size_t(sg.nb)], w);
                    if (!peer || peer->count != sg.count)
                        runtime_error("build_exchange_plan: endpoints disagree on link count for pair " +
                                      std::to_string(w) + " <-> " + std::to_string(sg.nb));
                }
            enable_peers();
        }
        p2p_mode = prm.halo_mode == 1 || (aa_mode && prm.workers > 1);
        if (aa_mode && p2p_mode) {
            setup_p2p();  // the AA scheme's odd steps read/write neighbours in place: no fallback
        } else if (p2p_mode) {
            // If peer mapping fails anywhere, every rank falls back to the
            // NCCL / peer-copy exchange (ranks agree through an all-reduce).
            int ok = 1;
            std::string why;
            try {
                setup_p2p();  // dist mode: collective, fails on all ranks together
            } catch (const Error& e) {
                if (e.kind == ErrKind::Comm) throw;
                ok = 0;
                why = e.what();
                cudaGetLastError();
            }
            if (!ok) {
                std::fprintf(stderr, "[splbcu] fused P2P halo unavailable (%s); using %s\n",
                             why.empty() ? "another rank failed" : why.c_str(),
                             dist ? "NCCL send/recv" : "peer copies");
                for (auto& wp : W)
                    if (wp) {
                        for (void* p : wp->ipc_opened) cudaIpcCloseMemHandle(p);
                        wp->ipc_opened.clear();
                    }
                p2p_mode = false;
            }
        }
        if (prm.observe_iolets) init_observation();
        for (auto& wp : W)
            if (wp) CK(cudaStreamSynchronize(wp->sM));
    }

    // NCCL all-reduce (min) of one int on the local worker's stream; also a barrier.
    int agree_min(int v) {
        WorkerDev& wk = *W[size_t(rank)];
        CK(cudaSetDevice(wk.dev));
        DevMem one;
        int* d = one.alloc<int>(1);
        CK(cudaMemcpyAsync(d, &v, sizeof(int), cudaMemcpyHostToDevice, wk.sE));
        NK(nccl().AllReduce(d, d, 1, ncclInt, ncclMin, comm, wk.sE));
        int out = 0;
        CK(cudaMemcpyAsync(&out, d, sizeof(int), cudaMemcpyDeviceToHost, wk.sE));
        CK(cudaStreamSynchronize(wk.sE));
        return out;
    }
    void dist_barrier() { (void)agree_min(1); }

    // Host-buffer collectives over the engine's NCCL communicator (dist mode).
    std::vector<double> allgather_host(const std::vector<double>& mine) {
        WorkerDev& wk = *W[size_t(rank)];
        CK(cudaSetDevice(wk.dev));
        DevMem s, r;
        double* ds = s.alloc<double>(mine.size());
        double* dr = r.alloc<double>(mine.size() * size_t(nranks));
        CK(cudaMemcpyAsync(ds, mine.data(), mine.size() * 8, cudaMemcpyHostToDevice, wk.sE));
        NK(nccl().AllGather(ds, dr, mine.size(), ncclDouble, comm, wk.sE));
        std::vector<double> all(mine.size() * size_t(nranks));
        CK(cudaMemcpyAsync(all.data(), dr, all.size() * 8, cudaMemcpyDeviceToHost, wk.sE));
        CK(cudaStreamSynchronize(wk.sE));
        return all;
    }
    // Sum over ranks of arrays that are disjoint (each rank's sites, zero
    // elsewhere): x + 0 == x exactly, so this assembles the global field.
    void allreduce_host_sum(double* x, size_t n) {
        WorkerDev& wk = *W[size_t(rank)];
        CK(cudaSetDevice(wk.dev));
        DevMem b;
        double* d = b.alloc<double>(n);
        CK(cudaMemcpyAsync(d, x, n * 8, cudaMemcpyHostToDevice, wk.sE));
        NK(nccl().AllReduce(d, d, n, ncclDouble, ncclSum, comm, wk.sE));
        CK(cudaMemcpyAsync(x, d, n * 8, cudaMemcpyDeviceToHost, wk.sE));
        CK(cudaStreamSynchronize(wk.sE));
    }

    // Fused P2P halo (§8f.4): map the neighbours' f buffers and flag words,
    // and give every outgoing shared slot its final destination in the
    // neighbour's f_new (the neighbour's recv_dest for that slot,
    // ExchangePlan::final_dest, exchange.hpp:20).
    void setup_p2p() {
        if (dist && !nccl().AllReduce) fail(ErrKind::Comm, "exchange failure: NCCL all-reduce unavailable");
        for (auto& wp : W) {
            if (!wp) continue;
            WorkerDev& wk = *wp;
            CK(cudaSetDevice(wk.dev));
            if (wk.segs.size() > size_t(kMaxPeers))
                config_error("engine: fused P2P halo supports at most " + std::to_string(kMaxPeers) + " neighbours");
            uint32_t* fl = wk.flags.alloc<uint32_t>(2 * size_t(prm.workers));
            CK(cudaMemset(fl, 0, 2 * size_t(prm.workers) * sizeof(uint32_t)));
        }
        if (!dist) {
            for (auto& wp : W) {
                WorkerDev& wk = *wp;
                std::vector<uint8_t> sp(std::max<uint32_t>(wk.shared, 1), 0);
                std::vector<uint64_t> sd(std::max<uint32_t>(wk.shared, 1), 0);
                wk.peer_f.clear();
                wk.peer_flags.clear();
                for (size_t k = 0; k < wk.segs.size(); ++k) {
                    const Seg& sg = wk.segs[k];
                    WorkerDev& peer = *W[size_t(sg.nb)];
                    const Seg* ps = find_seg(peer, wk.w);
                    if (peer.dev != wk.dev) {
                        int can = 0;
                        CK(cudaDeviceCanAccessPeer(&can, wk.dev, peer.dev));
                        if (!can)
                            fail(ErrKind::Cuda, "no peer access between devices " + std::to_string(wk.dev) + " and " +
                                                    std::to_string(peer.dev));
                    }
                    std::vector<uint64_t> prf(sg.count);
                    CK(cudaSetDevice(peer.dev));
                    if (sg.count)
                        CK(cudaMemcpy(prf.data(), peer.recv_flat.get<uint64_t>() + ps->base, sg.count * 8,
                                      cudaMemcpyDeviceToHost));
                    for (uint32_t j = 0; j < sg.count; ++j) sp[sg.base + j] = uint8_t(k), sd[sg.base + j] = prf[j];
                    wk.peer_f.push_back({peer.fbuf[0].get<double>(),
                                         peer.fbuf[aa_mode ? 0 : 1].get<double>()});
                    wk.peer_flags.push_back(peer.flags.get<uint32_t>());
                }
                CK(cudaSetDevice(wk.dev));
                upload(wk.slot_peer, sp, wk.sM);
                upload(wk.slot_dst, sd, wk.sM);
                CK(cudaStreamSynchronize(wk.sM));
            }
            return;
        }
        // one process per GPU: IPC handles all-gathered over NCCL
        WorkerDev& wk = *W[size_t(rank)];
        CK(cudaSetDevice(wk.dev));
        constexpr size_t H = sizeof(cudaIpcMemHandle_t);
        std::vector<cudaIpcMemHandle_t> mine(3);
        CK(cudaIpcGetMemHandle(&mine[0], wk.fbuf[0].p));
        CK(cudaIpcGetMemHandle(&mine[1], wk.fbuf[1].p));
        CK(cudaIpcGetMemHandle(&mine[2], wk.flags.p));
        DevMem dsend, drecv;
        char* ds = dsend.alloc<char>(3 * H);
        char* dr = drecv.alloc<char>(3 * H * size_t(nranks));
        CK(cudaMemcpyAsync(ds, mine.data(), 3 * H, cudaMemcpyHostToDevice, wk.sE));  // ordered before the all-gather
        NK(nccl().AllGather(ds, dr, 3 * H, ncclChar, comm, wk.sE));
        std::vector<cudaIpcMemHandle_t> all(3 * size_t(nranks));
        CK(cudaMemcpyAsync(all.data(), dr, 3 * H * size_t(nranks), cudaMemcpyDeviceToHost, wk.sE));
        CK(cudaStreamSynchronize(wk.sE));
        wk.peer_f.clear();
        wk.peer_flags.clear();
        int opened = 1;
        for (const Seg& sg : wk.segs) {
            std::array<double*, 2> pf{};
            for (int b = 0; b < 3 && opened; ++b) {
                void* p = nullptr;
                if (cudaIpcOpenMemHandle(&p, all[3 * size_t(sg.nb) + size_t(b)], cudaIpcMemLazyEnablePeerAccess) !=
                    cudaSuccess) {
                    cudaGetLastError();
                    opened = 0;
                    break;
                }
                wk.ipc_opened.push_back(p);
                if (b < 2) pf[size_t(b)] = static_cast<double*>(p);
                else wk.peer_flags.push_back(static_cast<uint32_t*>(p));
            }
            if (aa_mode) pf[1] = pf[0];  // single buffer
            wk.peer_f.push_back(pf);
        }
        // every rank must have mapped its neighbours before anyone proceeds
        if (!agree_min(opened)) fail(ErrKind::Cuda, "cudaIpcOpenMemHandle failed on some rank");
        // final destinations: each side sends its recv_dest slice for the pair
        uint64_t* sd = wk.slot_dst.alloc<uint64_t>(std::max<uint32_t>(wk.shared, 1));
        std::vector<uint8_t> sp(std::max<uint32_t>(wk.shared, 1), 0);
        for (size_t k = 0; k < wk.segs.size(); ++k)
            for (uint32_t j = 0; j < wk.segs[k].count; ++j) sp[wk.segs[k].base + j] = uint8_t(k);
        upload(wk.slot_peer, sp, wk.sE);
        const NcclApi& N = nccl();
        NK(N.GroupStart());
        for (const Seg& sg : wk.segs) {
            NK(N.Send(wk.recv_flat.get<uint64_t>() + sg.base, sg.count, ncclUint64, sg.nb, comm, wk.sE));
            NK(N.Recv(sd + sg.base, sg.count, ncclUint64, sg.nb, comm, wk.sE));
        }
        NK(N.GroupEnd());
        CK(cudaStreamSynchronize(wk.sE));
        dist_barrier();
    }

    ~Engine() {
        try {
            complete();  // a run still in flight
        } catch (...) {
        }
        if (p2p_mode && dist && comm && !failed) {
            try {
                dist_barrier();  // no neighbour still stores into our buffers
            } catch (...) {
            }
        }
        if (!failed)
            for (auto& wp : W)
                if (wp)
                    for (void* p : wp->ipc_opened) cudaIpcCloseMemHandle(p);
        if (comm) nccl().CommDestroy(comm);
        for (auto& wp : W) {
            if (!wp) continue;
            cudaSetDevice(wp->dev);
            for (auto& v : wp->tev)
                for (auto e : v) cudaEventDestroy(e);
            for (auto e : wp->prog) cudaEventDestroy(e);
            for (auto& pr : wp->tune_ev)
                for (auto ev : pr)
                    if (ev) cudaEventDestroy(ev);
            if (wp->evSend) cudaEventDestroy(wp->evSend);
            if (wp->evMid) cudaEventDestroy(wp->evMid);
            if (wp->evEnd) cudaEventDestroy(wp->evEnd);
            for (int b = 0; b < 2; ++b) {
                if (wp->evRun0[b]) cudaEventDestroy(wp->evRun0[b]);
                if (wp->evRun1[b]) cudaEventDestroy(wp->evRun1[b]);
                if (wp->evDone[b]) cudaEventDestroy(wp->evDone[b]);
                if (wp->evObsFree[b]) cudaEventDestroy(wp->evObsFree[b]);
                if (wp->evSerRead[b]) cudaEventDestroy(wp->evSerRead[b]);
            }
            if (wp->sE) cudaStreamDestroy(wp->sE);
            if (wp->sS) cudaStreamDestroy(wp->sS);
            if (wp->sM) cudaStreamDestroy(wp->sM);
        }
    }

    static const Seg* find_seg(const WorkerDev& wk, int nb) {
        for (const Seg& s : wk.segs)
            if (s.nb == nb) return &s;
        return nullptr;
    }

    // validate_setup (engine.hpp:223-241)
    void validate_setup() {
        validate_domain(dom);
        validate_params();
    }
    void validate_params() {
        if (prm.workers < 1) config_error("engine: workers must be >= 1");
        if (bcs.size() != dom.iolets.size())
            config_error("engine: boundary conditions configured for " + std::to_string(bcs.size()) +
                         " iolets but the geometry declares " + std::to_string(dom.iolets.size()));
        for (size_t k = 0; k < bcs.size(); ++k) {
            bcs[k].table.validate();
            if (bcs[k].kind == 0)  // PressureBC::validate (boundary.hpp:86-92)
                for (double vn : bcs[k].table.v)
                    if (!(vn / kCs2 > 0.0))
                        config_error("pressure BC: ghost density must stay positive (table value " +
                                     std::to_string(vn) + ")");
        }
        if (!(prm.tau > 0.5)) config_error("engine: tau must exceed 0.5");
    }

    void enable_peers() {
        std::vector<int> devs(prm.devices);
        std::sort(devs.begin(), devs.end());
        devs.erase(std::unique(devs.begin(), devs.end()), devs.end());
        for (int a : devs)
            for (int b : devs) {
                if (a == b) continue;
                int can = 0;
                CK(cudaDeviceCanAccessPeer(&can, a, b));
                if (!can) continue;
                CK(cudaSetDevice(a));
                cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
                if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
                else CK(e);
            }
    }

    void setup_worker(WorkerDev& wk, int w, int dev, const SiteIndex& ix) {
        wk.w = w;
        wk.dev = dev;
        CK(cudaSetDevice(dev));
        int lo_pri = 0, hi_pri = 0;
        CK(cudaDeviceGetStreamPriorityRange(&lo_pri, &hi_pri));
        CK(cudaStreamCreateWithPriority(&wk.sE, cudaStreamNonBlocking, hi_pri));
        CK(cudaStreamCreateWithPriority(&wk.sM, cudaStreamNonBlocking, lo_pri));
        CK(cudaStreamCreateWithPriority(&wk.sS, cudaStreamNonBlocking, lo_pri));
        CK(cudaEventCreateWithFlags(&wk.evSend, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&wk.evMid, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&wk.evEnd, cudaEventDisableTiming));
        for (int b = 0; b < 2; ++b) {
            CK(cudaEventCreate(&wk.evRun0[b]));
            CK(cudaEventCreate(&wk.evRun1[b]));
            CK(cudaEventCreateWithFlags(&wk.evDone[b], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&wk.evObsFree[b], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&wk.evSerRead[b], cudaEventDisableTiming));
        }
        cudaStream_t s = wk.sM;

        const WorkerPart& wp = part.parts[size_t(w)];
        wk.n = uint32_t(wp.sites.size());
        wk.n_edge = wp.n_edge;
        if (wk.n >= (1u << 29)) runtime_error("engine: worker holds too many sites for a u32 table");
        wk.P = (uint64_t(wk.n) + 63) / 64 * 64;
        if (wk.P == 0) wk.P = 64;

        // Internal order: per group, plain sites (types 0,1) merged in zyx
        // order, then iolet sites (types 2..5) in reference order.
        auto key_of = [&](uint32_t g) {
            return zyx_key(dom.coords[3 * uint64_t(g)], dom.coords[3 * uint64_t(g) + 1], dom.coords[3 * uint64_t(g) + 2]);
        };
        wk.ref_of_int.clear();
        wk.ref_of_int.reserve(wk.n);
        auto add_group = [&](const uint64_t ranges[6][2]) -> uint32_t {
            // plain: merge type-0 and type-1 runs by key
            uint64_t a = ranges[0][0], ae = ranges[0][1], b = ranges[1][0], be = ranges[1][1];
            while (a < ae || b < be) {
                if (b >= be || (a < ae && key_of(wp.sites[a]) < key_of(wp.sites[b])))
                    wk.ref_of_int.push_back(uint32_t(a++));
                else
                    wk.ref_of_int.push_back(uint32_t(b++));
            }
            const uint32_t plain = uint32_t((ae - ranges[0][0]) + (be - ranges[1][0]));
            for (uint64_t r = ranges[2][0]; r < ranges[5][1]; ++r) wk.ref_of_int.push_back(uint32_t(r));
            return plain;
        };
        wk.ep = add_group(wp.edge_ranges);
        wk.mp = add_group(wp.mid_ranges);
        wk.int_of_ref.assign(wk.n, 0);
        wk.global_of_int.resize(wk.n);
        for (uint32_t j = 0; j < wk.n; ++j) {
            wk.int_of_ref[wk.ref_of_int[j]] = j;
            wk.global_of_int[j] = uint32_t(global_of_site(wp.sites[wk.ref_of_int[j]]));
        }

        // Lookup subset: own sites + halo (slab: the two adjacent planes;
        // fallback split: every site), in zyx order.
        std::vector<uint64_t> lkeys;
        std::vector<int32_t> lowner;
        std::vector<uint32_t> llocal, lglobal;
        {
            int32_t pmin = INT32_MAX, pmax = INT32_MIN;
            if (part.slab) {
                for (size_t k = 0; k < part.plane_owner.size(); ++k)
                    if (part.plane_owner[k] == w) {
                        pmin = std::min(pmin, part.plane_lo + int32_t(k));
                        pmax = std::max(pmax, part.plane_lo + int32_t(k));
                    }
            }
            const int ax = part.axis;
            std::vector<uint32_t> g_int_local(0);
            for (uint64_t q = 0; q < ix.keys.size(); ++q) {
                const uint32_t g = ix.value[q];
                const int32_t c = dom.coords[3 * uint64_t(g) + ax];
                if (part.slab && (c < pmin - 1 || c > pmax + 1)) continue;
                lkeys.push_back(ix.keys[q]);
                lowner.push_back(part.owner[g]);
                lglobal.push_back(uint32_t(global_of_site(g)));
                llocal.push_back(part.owner[g] == w ? wk.int_of_ref[part.local_index[g]] : 0u);
            }
        }
        SiteIndex lix;
        lix.keys = lkeys;
        lix.build_rows();

        // upload build inputs
        std::vector<int32_t> coords(3 * uint64_t(wk.n));
        std::vector<uint8_t> kind(18 * uint64_t(wk.n));
        for (uint32_t j = 0; j < wk.n; ++j) {
            const uint64_t g = wp.sites[wk.ref_of_int[j]];  // index into dom
            std::memcpy(&coords[3 * uint64_t(j)], &dom.coords[3 * g], 12);
            std::memcpy(&kind[18 * uint64_t(j)], &dom.link_kind[18 * g], 18);
        }
        std::vector<uint64_t> io_pos;
        std::vector<uint16_t> io_id;
        for (size_t q = 0; q < dom.iolet_link_pos.size(); ++q) {
            const uint64_t g = dom.iolet_link_pos[q] / 18;
            if (part.owner[g] != w) continue;
            const uint32_t j = wk.int_of_ref[part.local_index[g]];
            const uint64_t i1 = dom.iolet_link_pos[q] % 18;  // i - 1
            io_pos.push_back(i1 * wk.P + j);
            io_id.push_back(dom.iolet_link_id[q]);
        }
        DevMem d_coords, d_kind, d_gidx, d_lk, d_lo, d_ll, d_lg, d_row, d_iop, d_ioi;
        const int32_t* dc = upload(d_coords, coords, s);
        const uint8_t* dk = upload(d_kind, kind, s);
        const uint32_t* dg = upload(d_gidx, wk.global_of_int, s);
        DLookup L{};
        L.keys = upload(d_lk, lkeys, s);
        L.owner = upload(d_lo, lowner, s);
        L.local = upload(d_ll, llocal, s);
        L.global = upload(d_lg, lglobal, s);
        L.n = lkeys.size();
        if (lix.rows) {
            L.row_off = upload(d_row, lix.row_off, s);
            L.lo1 = lix.lo[1];
            L.hi1 = lix.hi[1];
            L.lo2 = lix.lo[2];
            L.hi2 = lix.hi[2];
            L.ny = lix.ny;
        }
        uint32_t* tab = wk.tab.alloc<uint32_t>(18 * wk.P + kTilePad);
        CK(cudaMemsetAsync(tab, 0, (18 * wk.P + kTilePad) * sizeof(uint32_t), s));
        const uint64_t cap = 18 * uint64_t(wk.n_edge) + 1;
        DevMem ok_, ov_, ik_, iv_, cnt, ok2, ov2, ik2, iv2;
        auto* okeys = ok_.alloc<unsigned long long>(cap);
        auto* ovals = ov_.alloc<unsigned long long>(cap);
        auto* ikeys = ik_.alloc<unsigned long long>(cap);
        auto* ivals = iv_.alloc<unsigned long long>(cap);
        unsigned* counters = cnt.alloc<unsigned>(4);
        CK(cudaMemsetAsync(counters, 0, 4 * sizeof(unsigned), s));
        if (wk.n)
            build_links<<<blocks_for(uint64_t(wk.n) * 18), 256, 0, s>>>(
                wk.n, wk.P, dc, dk, dg, w, L, tab, okeys, ovals, counters + 0, ikeys, ivals, counters + 1,
                counters + 2);
        CK(cudaGetLastError());
        const uint64_t* dip = upload(d_iop, io_pos, s);
        const uint16_t* dii = upload(d_ioi, io_id, s);
        if (!io_pos.empty())
            patch_iolets<<<blocks_for(io_pos.size()), 256, 0, s>>>(dip, dii, uint32_t(io_pos.size()), tab);
        CK(cudaGetLastError());
        unsigned hc[4];
        CK(cudaMemcpyAsync(hc, counters, sizeof(hc), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (hc[2]) runtime_error("build_streaming_map: fluid link to a site outside the worker's halo");
        if (hc[0] > cap || hc[1] > cap) runtime_error("build_streaming_map: cross-link overflow");
        const uint32_t n_out = hc[0], n_in = hc[1];
        // canonical order: (neighbour, sender global site, direction)
        auto* okeys2 = ok2.alloc<unsigned long long>(cap);
        auto* ovals2 = ov2.alloc<unsigned long long>(cap);
        auto* ikeys2 = ik2.alloc<unsigned long long>(cap);
        auto* ivals2 = iv2.alloc<unsigned long long>(cap);
        auto radix = [&](unsigned long long* k, unsigned long long* v, unsigned long long* k2,
                         unsigned long long* v2, uint32_t m) {
            if (!m) return;
            size_t tmp = 0;
            CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, k, k2, v, v2, int(m), 0, 64, s));
            DevMem t;
            void* tp = t.alloc<char>(tmp);
            CK(cub::DeviceRadixSort::SortPairs(tp, tmp, k, k2, v, v2, int(m), 0, 64, s));
            CK(cudaStreamSynchronize(s));
        };
        radix(okeys, ovals, okeys2, ovals2, n_out);
        radix(ikeys, ivals, ikeys2, ivals2, n_in);
        std::vector<unsigned long long> hok(n_out), hik(n_in);
        if (n_out) CK(cudaMemcpy(hok.data(), okeys2, n_out * 8ull, cudaMemcpyDeviceToHost));
        if (n_in) CK(cudaMemcpy(hik.data(), ikeys2, n_in * 8ull, cudaMemcpyDeviceToHost));
        std::map<int, uint32_t> cout_, cin_;
        for (auto k : hok) ++cout_[int(k >> 40)];
        for (auto k : hik) ++cin_[int(k >> 40)];
        if (cout_ != cin_) runtime_error("build_streaming_map: asymmetric cross-link counts");
        // neighbours must match the partition's list (decomp.hpp:170-171)
        std::vector<int> nbs;
        for (auto& kv : cout_) nbs.push_back(kv.first);
        if (nbs != wp.neighbors) runtime_error("build_streaming_map: neighbour set mismatch");
        uint32_t base = 0;
        wk.segs.clear();
        for (auto& kv : cout_) {
            wk.segs.push_back({kv.first, base, kv.second});
            base += kv.second;
        }
        wk.shared = base;
        if (wk.shared >= (1u << 29)) runtime_error("engine: shared region exceeds the table payload");
        uint64_t* rf = wk.recv_flat.alloc<uint64_t>(std::max<uint32_t>(wk.shared, 1));
        uint64_t* sp = wk.send_pos.alloc<uint64_t>(std::max<uint32_t>(wk.shared, 1));
        if (wk.shared)
            assign_slots<<<blocks_for(wk.shared), 256, 0, s>>>(ovals2, ivals2, wk.shared, tab, rf, sp);
        CK(cudaGetLastError());

        // the table build's device temporaries go before the big allocations
        CK(cudaStreamSynchronize(s));
        for (DevMem* m : {&d_coords, &d_kind, &d_gidx, &d_lk, &d_lo, &d_ll, &d_lg, &d_row, &d_iop, &d_ioi, &ok_, &ov_,
                          &ik_, &iv_, &cnt, &ok2, &ov2, &ik2, &iv2})
            m->release();
        // distribution store, f_old = equilibrium(rho0, 0) (engine.hpp:243-260);
        // the AA scheme keeps a single buffer
        for (int b = 0; b < (aa_mode ? 1 : 2); ++b) {
            double* f = wk.fbuf[b].alloc<double>(wk.fsize() + kTilePad);
            CK(cudaMemsetAsync(f, 0, (wk.fsize() + kTilePad) * sizeof(double), s));
        }
        if (aa_mode) wk.fbuf[1].alloc<double>(1);
        wk.old = 0;
        Eq19 eq;
        feq_all(prm.rho0, 0.0, 0.0, 0.0, eq.v);
        if (wk.n) lbm_init_equilibrium<<<blocks_for(wk.n), 256, 0, s>>>(wk.f_old(), wk.P, wk.n, eq);
        CK(cudaGetLastError());

        // iolet sites' coordinates (edge iolet range then mid iolet range)
        std::vector<int32_t> ioc;
        for (uint32_t j = wk.ep; j < wk.n_edge; ++j)
            for (int a = 0; a < 3; ++a) ioc.push_back(coords[3 * uint64_t(j) + a]);
        for (uint32_t j = wk.n_edge + wk.mp; j < wk.n; ++j)
            for (int a = 0; a < 3; ++a) ioc.push_back(coords[3 * uint64_t(j) + a]);
        upload(wk.io_coords, ioc, s);
        upload(wk.io_geo, io_host, s);
        // tensor maps for the warp-specialised TMA kernel
        wk.tma_ok = wk.P >= 256;
        for (int v = 0; v < 2 && wk.tma_ok; ++v) {
            const uint32_t box = v == 0 ? 128 : 256;
            for (int b = 0; b < 2; ++b)
                encode_planes(&wk.tm_f[b][v], wk.fbuf[b].get<double>(), true, kQ, wk.P, box);
            encode_planes(&wk.tm_t[v], wk.tab.get<uint32_t>(), false, kQ - 1, wk.P, box);
        }
        // compressed table for the mid-group plain range
        wk.ctab_ok = false;
        if (wk.mp > 0) {
            // pitch of the group bases: a multiple of 4 (16-byte bulk copies) with
            // room for the last tile's overhang; deltas padded likewise
            wk.PG = (wk.P / 32 + 32 + 3) / 4 * 4;
            int16_t* dt = wk.dtab.alloc<int16_t>(18 * wk.P + 4 * kTilePad);
            uint32_t* gb = wk.gbase.alloc<uint32_t>(18 * wk.PG);
            CK(cudaMemsetAsync(dt, 0, (18 * wk.P + 4 * kTilePad) * sizeof(int16_t), s));
            CK(cudaMemsetAsync(gb, 0, 18 * wk.PG * sizeof(uint32_t), s));
            DevMem cerr;
            unsigned* ce = cerr.alloc<unsigned>(1);
            CK(cudaMemsetAsync(ce, 0, sizeof(unsigned), s));
            const uint32_t b0 = wk.n_edge, b1 = wk.n_edge + wk.mp;
            const uint64_t groups = ((b1 + 31) >> 5) - (b0 >> 5);
            compress_table<<<blocks_for(groups * 18 * 32), 256, 0, s>>>(wk.tab.get<uint32_t>(), wk.P, wk.PG, b0, b1,
                                                                       dt, gb, ce);
            CK(cudaGetLastError());
            unsigned he = 0;
            CK(cudaMemcpyAsync(&he, ce, sizeof(he), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            wk.ctab_ok = he == 0;
            if (std::getenv("SPLBCU_VERBOSE"))
                std::fprintf(stderr, "[splbcu] worker %d: compressed table %s (code %u)\n", wk.w,
                             wk.ctab_ok ? "on" : "off", he);
            if (!wk.ctab_ok) {
                wk.dtab.release();
                wk.gbase.release();
            }
            // run-length table (kernels.cuh: build_run_table), tiles of 256
            constexpr uint32_t T = 256;
            const uint32_t t0 = b0 / T, t1 = (b1 + T - 1) / T;
            unsigned char* rt = wk.rtab.alloc<unsigned char>(uint64_t(t1) * RunTab<T>::kBytes);
            unsigned* rc = cerr.alloc<unsigned>(2);
            CK(cudaMemsetAsync(rc, 0, 2 * sizeof(unsigned), s));
            const uint64_t warps = uint64_t(t1 - t0) * (kQ - 1) * RunTab<T>::kG;
            build_run_table<T><<<unsigned((warps * 32 + 255) / 256), 256, 0, s>>>(wk.tab.get<uint32_t>(), wk.P, b0, b1,
                                                                                  t0, t1, rt, rc, rc + 1);
            CK(cudaGetLastError());
            unsigned hr[2] = {0, 0};
            CK(cudaMemcpyAsync(hr, rc, sizeof(hr), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            wk.rtab_ok = hr[0] == 0;
            wk.n_cand = wk.rtab_ok && wk.ctab_ok ? 3 : 2;
            wk.rtab_escaped = hr[1];
            if (std::getenv("SPLBCU_VERBOSE"))
                std::fprintf(stderr, "[splbcu] worker %d: run table %s, %u of %llu (direction, group)s escaped\n", wk.w,
                             wk.rtab_ok ? "on" : "off", hr[1], (unsigned long long)(warps));
            if (!wk.rtab_ok) wk.rtab.release();
        }
        CK(cudaStreamSynchronize(s));
    }

    // init_observation (engine.hpp:262-288)
    void init_observation() {
        const size_t n_io = dom.iolets.size();
        obs_order.assign(n_io, {});
        for (auto& wp : W)
            if (wp) wp->obs_sites.assign(n_io, {});
        std::vector<std::vector<uint32_t>> per_w_count(size_t(prm.workers), std::vector<uint32_t>(n_io, 0));
        size_t q = 0;
        std::vector<uint8_t> member(n_io);
        std::vector<std::vector<uint64_t>> own_obs(n_io);  // slab-local: own sites' global indices
        while (q < dom.iolet_link_pos.size()) {
            const uint64_t g = dom.iolet_link_pos[q] / 18;
            std::fill(member.begin(), member.end(), 0);
            while (q < dom.iolet_link_pos.size() && dom.iolet_link_pos[q] / 18 == g) {
                member[dom.iolet_link_id[q]] = 1;
                ++q;
            }
            for (size_t k = 0; k < n_io; ++k) {
                if (!member[k]) continue;
                const int w = part.owner[g];
                if (win && w != rank) continue;  // halo site: its owner observes it
                if (win) own_obs[k].push_back(global_of_site(g));
                obs_order[k].push_back({w, per_w_count[size_t(w)][k]++});
                if (W[size_t(w)]) {
                    WorkerDev& wk = *W[size_t(w)];
                    wk.obs_sites[k].push_back(wk.int_of_ref[part.local_index[g]]);
                }
            }
        }
        if (win) {
            // every rank's observed sites (iolet-major, global indices): the
            // series order is ascending global index across ranks
            std::vector<uint64_t> mine;
            for (size_t k = 0; k < n_io; ++k) {
                mine.push_back(own_obs[k].size());
                mine.insert(mine.end(), own_obs[k].begin(), own_obs[k].end());
            }
            const std::vector<std::vector<uint64_t>> all = allgather_setup(mine);
            for (size_t k = 0; k < n_io; ++k) obs_order[k].clear();
            std::vector<std::vector<std::tuple<uint64_t, int, uint32_t>>> merged(n_io);
            for (int w = 0; w < prm.workers; ++w) {
                const std::vector<uint64_t>& v = all[size_t(w)];
                size_t p = 0;
                for (size_t k = 0; k < n_io; ++k) {
                    const uint64_t c = v.at(p++);
                    per_w_count[size_t(w)][k] = uint32_t(c);
                    for (uint64_t j = 0; j < c; ++j) merged[k].emplace_back(v.at(p++), w, uint32_t(j));
                }
            }
            for (size_t k = 0; k < n_io; ++k) {
                std::sort(merged[k].begin(), merged[k].end());
                for (auto& [g, w, pos] : merged[k]) obs_order[k].push_back({w, pos});
            }
        }
        obs_off_all.assign(size_t(prm.workers), std::vector<uint32_t>(n_io + 1, 0));
        for (size_t w = 0; w < size_t(prm.workers); ++w)
            for (size_t k = 0; k < n_io; ++k) obs_off_all[w][k + 1] = obs_off_all[w][k] + per_w_count[w][k];
        for (auto& wp : W) {
            if (!wp) continue;
            WorkerDev& wk = *wp;
            CK(cudaSetDevice(wk.dev));
            std::vector<uint32_t> site;
            std::vector<uint16_t> iol;
            wk.obs_off.assign(n_io + 1, 0);
            for (size_t k = 0; k < n_io; ++k) {
                wk.obs_off[k] = uint32_t(site.size());
                for (uint32_t j : wk.obs_sites[k]) {
                    site.push_back(j);
                    iol.push_back(uint16_t(k));
                }
            }
            wk.obs_off[n_io] = uint32_t(site.size());
            wk.n_obs = uint32_t(site.size());
            upload(wk.obs_site, site, wk.sM);
            upload(wk.obs_iolet, iol, wk.sM);
            CK(cudaStreamSynchronize(wk.sM));
        }
        // Series on the device when one worker's device sees every row: dist
        // mode (after the all-gather) or a single in-process worker.  A
        // gather kernel puts the entries in series order (long iolets first);
        // short iolets are reduced there by series_chain, long ones (whose
        // sequential chain the host runs ~5x faster) are copied out and
        // reduced on the host, in the same order.
        dev_series = (dist || prm.workers == 1) && getenv("SPLBCU_HOST_SERIES") == nullptr;
        if (dev_series) {
            WorkerDev& wk = *W[size_t(dist ? rank : 0)];
            CK(cudaSetDevice(wk.dev));
            constexpr size_t kHostChain = 2048;  // entries per iolet above which the host reduces it
            std::vector<uint16_t> ew;
            std::vector<uint32_t> ei, be(2 * n_io, 0), tot(size_t(prm.workers));
            ser_host_k.clear();
            ser_dev_k.clear();
            for (size_t k = 0; k < n_io; ++k) (obs_order[k].size() > kHostChain ? ser_host_k : ser_dev_k).push_back(uint32_t(k));
            for (const std::vector<uint32_t>* list : {&ser_host_k, &ser_dev_k})
                for (uint32_t k : *list) {
                    be[2 * k] = uint32_t(ew.size());
                    for (const auto& [w, pos] : obs_order[k]) {
                        ew.push_back(uint16_t(w));
                        ei.push_back(obs_off_all[size_t(w)][k] + pos);
                    }
                    be[2 * k + 1] = uint32_t(ew.size());
                }
            ser_host_ent = ser_host_k.empty() ? 0 : be[2 * ser_host_k.back() + 1];
            ser_be = be;
            for (int w = 0; w < prm.workers; ++w) tot[size_t(w)] = obs_off_all[size_t(w)][n_io];
            n_series_ent = uint32_t(ew.size());
            upload(ser_w, ew, wk.sM);
            upload(ser_idx, ei, wk.sM);
            upload(ser_off, be, wk.sM);
            upload(ser_tot, tot, wk.sM);
            upload(ser_kdev, ser_dev_k, wk.sM);
            CK(cudaStreamSynchronize(wk.sM));
        }
    }

    // run()'s series: gather this run's rows into series order, reduce the
    // short iolets on the device, and copy results + the long iolets' entries
    // to pinned host memory, on stream s (behind the step loop).
    // `gathered` (optional) is recorded once the rows at src have been read.
    void reduce_series_async(WorkerDev& wk, cudaStream_t s, const double* src, uint64_t per, int buf,
                             cudaEvent_t gathered = nullptr) {
        const uint32_t rows = uint32_t(wk.obs_rows), n_io = uint32_t(dom.iolets.size());
        if (!rows || !n_io) {
            if (gathered) CK(cudaEventRecord(gathered, s));
            return;
        }
        const uint64_t ne = std::max<uint32_t>(n_series_ent, 1);
        double* g = ser_buf.reserve<double>(3 * uint64_t(rows) * ne);
        double* o = ser_out.reserve<double>(3 * uint64_t(rows) * n_io);
        const uint64_t ng = uint64_t(n_series_ent) * rows;
        if (ng) {
            series_gather<<<unsigned((ng + 255) / 256), 256, 0, s>>>(src, per, ser_tot.get<uint32_t>(),
                                                                       ser_w.get<uint16_t>(), ser_idx.get<uint32_t>(),
                                                                       n_series_ent, rows, g);
            ++launches;
        }
        if (gathered) CK(cudaEventRecord(gathered, s));
        if (!ser_dev_k.empty()) {
            const uint64_t warps = uint64_t(ser_dev_k.size()) * rows;
            series_chain<<<unsigned(warps), 32, 0, s>>>(g, ser_kdev.get<uint32_t>(), ser_off.get<uint32_t>(),
                                                        uint32_t(ser_dev_k.size()), n_io, rows, n_series_ent, o);
            ++launches;
        }
        CK(cudaGetLastError());
        double* h = h_series[buf].reserve<double>(3 * uint64_t(rows) * n_io);
        CK(cudaMemcpyAsync(h, o, 3 * uint64_t(rows) * n_io * 8, cudaMemcpyDeviceToHost, s));
        if (ser_host_ent) {
            double* hr = h_series_raw[buf].reserve<double>(3 * uint64_t(rows) * ser_host_ent);
            CK(cudaMemcpy2DAsync(hr, 3 * size_t(ser_host_ent) * 8, g, 3 * size_t(ne) * 8, 3 * size_t(ser_host_ent) * 8,
                                 rows, cudaMemcpyDeviceToHost, s));
        }
    }

    // ---- stepping -----------------------------------------------------------
    // Launch-shape variants of the plain kernel (SPLBCU_PLAIN_VARIANT picks
    // one for tuning; the default is the measured best).
    int plain_variant = [] {
        const char* v = getenv("SPLBCU_PLAIN_VARIANT");
        return v ? atoi(v) : 0;
    }();
    // online choice of the bulk kernel (off: keep the prior; forced variants never tune)
    bool autotune = plain_variant == 0 && getenv("SPLBCU_NO_AUTOTUNE") == nullptr;
    // Resident CTAs per device for a persistent kernel (occupancy x SMs),
    // with its dynamic shared-memory limit raised once per (kernel, device).
    std::map<std::pair<const void*, int>, int> resident_;
    template <class Fn>
    int resident_ctas(Fn* fn, int dev, int threads, uint32_t smem) {
        const auto key = std::make_pair(reinterpret_cast<const void*>(fn), dev);
        const auto it = resident_.find(key);
        if (it != resident_.end()) return it->second;
        CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        int per_sm = 0, sms = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem));
        CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        return resident_[key] = std::max(1, per_sm) * sms;
    }
    // The persistent TMA kernels copy whole tiles: the last tile may run past
    // `end` into the tail pad (f: shared tail + kTilePad; deltas: 4 kTilePad;
    // group bases: PG slack).  Checked on the host at every launch (a bad
    // range would otherwise read past the allocation; compute-sanitizer is
    // not available on this pool).
    static void check_tiles(const WorkerDev& wk, uint32_t base, uint32_t ntiles, uint32_t T) {
        const uint64_t last = uint64_t(base) + uint64_t(ntiles) * T;
        if (last > wk.P + kTilePad || (wk.ctab_ok && (last + 31) / 32 > wk.PG))
            runtime_error("engine: tile range [" + std::to_string(base) + ", " + std::to_string(last) +
                          ") exceeds the padded planes (P = " + std::to_string(wk.P) + ")");
    }

    template <int T, int B>
    void launch_plain_t(WorkerDev& wk, cudaStream_t s, uint32_t b, uint32_t e, const IoletArgs& ia) {
        lbm_push<false, T, B><<<unsigned((e - b + T - 1) / T), T, 0, s>>>(
            wk.f_old(), wk.f_new(), wk.tab.get<uint32_t>(), wk.P, b, e, omega, ia, HaloArgs{});
    }
    // The tile-major compressed table (built on first use from dtab/gbase).
    const int16_t* tile_table(WorkerDev& wk) {
        if (!wk.ctile.p) {
            constexpr uint32_t T = 256;
            constexpr uint64_t kTab = uint64_t(kQ - 1) * T * 2 + uint64_t(kQ - 1) * (T / 32) * 4;
            const uint32_t t0 = wk.n_edge / T, t1 = (wk.n_edge + wk.mp + T - 1) / T;
            wk.ctile.alloc<unsigned char>(uint64_t(t1) * kTab);
            const uint64_t work = uint64_t(t1 - t0) * (uint64_t(kQ - 1) * T + (kQ - 1) * (T / 32));
            if (work)
                build_table_tiles<T><<<unsigned((work + 255) / 256), 256, 0, wk.sM>>>(
                    wk.dtab.get<int16_t>(), wk.gbase.get<uint32_t>(), wk.P, wk.PG, t0, t1, wk.ctile.get<unsigned char>());
            CK(cudaGetLastError());
            CK(cudaStreamSynchronize(wk.sM));
        }
        return wk.ctile.get<int16_t>();
    }

    // Persistent TMA kernel over the compressed table (mid-group range only).
    template <int T, int S, int B, int H = 2>
    void launch_tmc(WorkerDev& wk, cudaStream_t s, uint32_t b, uint32_t e) {
        using L0 = PushTmaSmem<T, S, false>;
        // + the int16 delta planes per stage when H & 8
        constexpr bool tm = (H & 16384) != 0;
        constexpr uint32_t kBytes = S * (L0::kF + ((H & 8) || tm ? uint32_t(kQ - 1) * T * 2 : 0u) +
                                         ((H & 136) == 136 || tm ? uint32_t(kQ - 1) * (T / 32) * 4 : 0u)) + S * 8;
        const int resident = resident_ctas(lbm_push_tmc<T, S, B, H>, wk.dev, T, kBytes);
        const uint32_t base = b & ((H & 16384) ? ~uint32_t(T - 1) : ((H & 136) == 136 ? ~127u : ~31u));
        const uint32_t ntiles = (e - base + T - 1) / T;
        const unsigned grid = unsigned(std::min<uint32_t>(ntiles, uint32_t(resident)));
        check_tiles(wk, base, ntiles, T);
        Planes19 pl;
        for (int i = 0; i < kQ; ++i) pl.p[i] = wk.f_new() + uint64_t(i) * wk.P;
        const int16_t* dt = (H & 16384) ? tile_table(wk) : wk.dtab.get<int16_t>();
        lbm_push_tmc<T, S, B, H><<<grid, T, kBytes, s>>>(wk.f_old(), wk.f_new(), dt,
                                                              wk.gbase.get<uint32_t>(), wk.tab.get<uint32_t>(), wk.P,
                                                              wk.PG, b, e, omega, pl);
    }

#ifdef SPLBCU_TUNING
    // Warp-autonomous push kernel over the delta table (mid-group range only).
    template <int NW, int B>
    void launch_push_w(WorkerDev& wk, cudaStream_t s, uint32_t b, uint32_t e) {
        using Lm = PushW<NW, B>;
        const int resident = resident_ctas(lbm_push_w<NW, B>, wk.dev, NW * 32, Lm::kBytes);
        const uint32_t ntiles = (e - (b & ~31u) + 31) / 32;
        const unsigned grid = unsigned(std::min<uint32_t>((ntiles + NW - 1) / NW, uint32_t(resident)));
        check_tiles(wk, b & ~31u, ntiles, 32);
        Planes19 pl;
        for (int i = 0; i < kQ; ++i) pl.p[i] = wk.f_new() + uint64_t(i) * wk.P;
        lbm_push_w<NW, B><<<grid, NW * 32, Lm::kBytes, s>>>(wk.f_old(), wk.f_new(), wk.dtab.get<int16_t>(),
                                                         wk.gbase.get<uint32_t>(), wk.tab.get<uint32_t>(), wk.P, wk.PG, b,
                                                         e, omega, pl);
    }
#endif

    // A zeroed tile counter for one dynamic-order launch on stream s (a ring of
    // slots, each zeroed stream-ordered right before its launch).
    unsigned* tile_counter(WorkerDev& wk, cudaStream_t s) {
        constexpr uint32_t kCtr = 256;
        if (!wk.tile_ctr.p) wk.tile_ctr.alloc<unsigned>(kCtr);
        if (wk.ctr_used + 1 > kCtr) wk.ctr_used = 0;
        unsigned* ctr = wk.tile_ctr.get<unsigned>() + wk.ctr_used++;
        CK(cudaMemsetAsync(ctr, 0, sizeof(unsigned), s));
        return ctr;
    }

    // Persistent TMA kernel with a dynamic tile order (mid-group range only).
    template <int T, int S, int B>
    void launch_dyn(WorkerDev& wk, cudaStream_t s, uint32_t b, uint32_t e) {
        using L0 = PushTmaSmem<T, S, false>;
        constexpr uint32_t kBytes = S * L0::kF + S * 8 + S * 4;
        const int resident = resident_ctas(lbm_push_dyn<T, S, B>, wk.dev, T, kBytes);
        const uint32_t base = b & ~31u;
        const uint32_t ntiles = (e - base + T - 1) / T;
        const unsigned grid = unsigned(std::min<uint32_t>(ntiles, uint32_t(resident)));
        check_tiles(wk, base, ntiles, T);
        unsigned* ctr = tile_counter(wk, s);
        Planes19 pl;
        for (int i = 0; i < kQ; ++i) pl.p[i] = wk.f_new() + uint64_t(i) * wk.P;
        lbm_push_dyn<T, S, B><<<grid, T, kBytes, s>>>(wk.f_old(), wk.f_new(), wk.dtab.get<int16_t>(),
                                                      wk.gbase.get<uint32_t>(), wk.tab.get<uint32_t>(), wk.P, wk.PG, b,
                                                      e, omega, ctr, pl);
    }

    // Persistent TMA kernel over the run-length table (mid-group range only).
    template <int T, int S, int B>
    void launch_run(WorkerDev& wk, cudaStream_t s, uint32_t b, uint32_t e, bool dyn = false) {
        constexpr uint32_t kBytes = S * (uint32_t(kQ) * T * 8 + RunTab<T>::kBytes) + S * 8 + S * 4;
        const int resident = resident_ctas(lbm_push_run<T, S, B>, wk.dev, T, kBytes);
        const uint32_t base = b & ~uint32_t(T - 1);
        const uint32_t ntiles = (e - base + T - 1) / T;
        const unsigned grid = unsigned(std::min<uint32_t>(ntiles, uint32_t(resident)));
        check_tiles(wk, base, ntiles, T);
        Planes19 pl;
        for (int i = 0; i < kQ; ++i) pl.p[i] = wk.f_new() + uint64_t(i) * wk.P;
        unsigned* ctr = dyn ? tile_counter(wk, s) : nullptr;
        lbm_push_run<T, S, B><<<grid, T, kBytes, s>>>(wk.f_old(), wk.f_new(), wk.rtab.get<unsigned char>(),
                                                      wk.tab.get<uint32_t>(), wk.P, b, e, omega, pl, ctr);
    }

    // Which kernel the bulk (mid) plain range launches now on this process's
    // first worker:
    // 0 dynamic tile order (just-in-time table loads), 1 prefetch kernel,
    // 2 run-length table, 3 the fixed-order just-in-time kernel; -1 other.
    int bulk_kernel_of(const WorkerDev& wk) const {
        if (!wk.ctab_ok) return -1;
        if (plain_variant == 43) return 3;
        if (plain_variant == 76 || (plain_variant >= 82 && plain_variant <= 84)) return 0;
        if (plain_variant == 59) return 1;
        if (plain_variant == 71 || plain_variant == 77) return wk.rtab_ok ? 2 : -1;
        return plain_variant == 0 ? wk.mid_pick : -1;
    }
    int bulk_kernel() const {
        for (const auto& wp : W)
            if (wp) return bulk_kernel_of(*wp);
        return -1;
    }

    // The bulk range as `parts` launches of about equal size (at most
    // ~kBulkChunk sites each), cut at absolute 256-site boundaries.  Measured
    // on B200, C3 tree 1.07e8 sites, just-in-time kernel: from rest one launch
    // 16,190 MSUPS, 13.5e6-site parts 17,941 (profiles/r01_sweep_chunk.log);
    // in a developed flow 13.5e6-site parts 16,684, 9e6 17,192, 6.75e6
    // 17,028-17,330, 4.5e6 17,396, 3.4e6 17,312, while from rest 6.75e6 and
    // 13.5e6 tie (17,932 / 17,957) and the 1e7-site pipe gains 5 % with the
    // run-length table (profiles/r02/sweep4_*).  SPLBCU_BULK_CHUNK overrides
    // the part size (0: one launch).
    static constexpr uint64_t kBulkChunk = 6750000;
    uint64_t bulk_chunk = [] {
        const char* v = getenv("SPLBCU_BULK_CHUNK");
        return v ? uint64_t(atoll(v)) : kBulkChunk;
    }();
    const bool parts_forced = getenv("SPLBCU_BULK_CHUNK") != nullptr;
    template <class Fn>
    void for_parts(uint32_t b, uint32_t e, Fn&& fn) {
        const uint64_t n = uint64_t(e - b);
        const uint64_t parts = bulk_chunk < 256 ? 1 : (n + bulk_chunk - 1) / bulk_chunk;
        uint64_t c = b;
        for (uint64_t k = 1; k <= parts; ++k) {
            const uint64_t c1 = k == parts ? uint64_t(e) : ((uint64_t(b) + k * n / parts) & ~uint64_t(255));
            if (c1 <= c) continue;
            fn(uint32_t(c), uint32_t(c1));
            if (c != b) ++launches;  // the step's launch count holds one bulk launch
            c = c1;
        }
    }
    void launch_bulk(WorkerDev& wk, cudaStream_t s, uint32_t b, uint32_t e, const IoletArgs& ia) {
        // the dynamic tile order keeps the CTAs together by itself: one launch
        // (C3 developed 17,631 vs 17,186 in 6.75e6-site parts, profiles/r02/dyn_*)
        if ((bulk_kernel_of(wk) == 0 || plain_variant == 77) && !parts_forced) return launch_plain(wk, s, b, e, ia, true);
        for_parts(b, e, [&](uint32_t c, uint32_t c1) { launch_plain(wk, s, c, c1, ia, true); });
    }

    // The bulk plain launch through the online kernel choice (WorkerDev::mid_pick).
    // Measurement windows start at every multiple of kTuneEvery bulk launches
    // (0, 500, 1000, ...): n_cand x kTuneReps launches cycle through the candidates
    // under CUDA events, each kernel's fastest launch counts (the first launch
    // of a template also carries its one-time setup), and the faster kernel
    // is kept from the moment the events have completed.
    void launch_mid_tuned(WorkerDev& wk, cudaStream_t s, uint32_t b, uint32_t e, const IoletArgs& ia) {
        // prior before the first measurement: the dynamic-order kernel
        if (wk.mid_launches == 0) wk.mid_pick = 0;
        if (!autotune || !wk.ctab_ok) {
            launch_bulk(wk, s, b, e, ia);
            ++wk.mid_launches;
            return;
        }
        const int nc = wk.n_cand, nlaunch = nc * WorkerDev::kTuneReps;
        if (wk.tune_pending) {
            // read the measurement once its last launch has finished (no sync)
            const cudaError_t q = cudaEventQuery(wk.tune_ev[nlaunch - 1][1]);
            if (q == cudaSuccess) {
                float t[WorkerDev::kCand] = {3.4e38f, 3.4e38f, 3.4e38f};
                for (int k = 0; k < nlaunch; ++k) {
                    float ms = 0.f;
                    CK(cudaEventElapsedTime(&ms, wk.tune_ev[k][0], wk.tune_ev[k][1]));
                    t[k % nc] = std::min(t[k % nc], ms);
                }
                int best = 0;
                for (int c = 1; c < nc; ++c)
                    if (t[c] < t[best]) best = c;
                wk.mid_pick = best;
                wk.tune_pending = false;
            } else if (q != cudaErrorNotReady) {
                CK(q);
            }
        }
        if (wk.tune_phase == 0 && !wk.tune_pending && wk.mid_launches % WorkerDev::kTuneEvery == 0)
            wk.tune_phase = 1;
        if (wk.tune_phase > 0) {
            const int k = wk.tune_phase - 1;
            for (auto& ev : wk.tune_ev[k])
                if (!ev) CK(cudaEventCreate(&ev));
            const int keep = wk.mid_pick;
            wk.mid_pick = k % nc;
            CK(cudaEventRecord(wk.tune_ev[k][0], s));
            launch_bulk(wk, s, b, e, ia);
            CK(cudaEventRecord(wk.tune_ev[k][1], s));
            wk.mid_pick = keep;
            if (++wk.tune_phase > nlaunch) {
                wk.tune_phase = 0;
                wk.tune_pending = true;
            }
        } else {
            launch_bulk(wk, s, b, e, ia);
        }
        ++wk.mid_launches;
    }

    // The plain (Inner+Wall) range.  Built kernels: the bulk mid range runs
    // the compressed-table TMA kernel, just-in-time table loads (<256,2,2,6>)
    // or the next tile's table prefetched after the divisions
    // (<256,2,2,4102>), chosen online (launch_mid_tuned; both measured best
    // somewhere); edge ranges and workers without a compressed
    // table run the u32-table TMA kernel.  Forced: SPLBCU_PLAIN_VARIANT 43 /
    // 59 (one bulk kernel), 24 (u32 table everywhere).  The measured-slower
    // launch shapes and hints of the tuning sweeps are built with
    // `make TUNING=1` only (profiles/sweep_variants.py).
    static bool variant_built(int v) {
#ifdef SPLBCU_TUNING
        (void)v;
        return true;
#else
        return v == 0 || v == 24 || v == 43 || v == 59 || v == 60 || v == 64 || v == 71 || v == 72 || v == 76 ||
               v == 77 || v == 78 || v == 79 || v == 80 || v == 81 || v == 94;
#endif
    }
    void launch_plain(WorkerDev& wk, cudaStream_t s, uint32_t b, uint32_t e, const IoletArgs& ia, bool mid) {
#ifdef SPLBCU_TUNING
        if (launch_tuning_variant(wk, s, b, e, ia, mid)) return;
#endif
        if (plain_variant == 24) return launch_tma<256, 2, 2, false, 2>(wk, s, b, e);
        if (plain_variant == 71 && mid && wk.rtab_ok) return launch_run<256, 2, 2>(wk, s, b, e);
        if (plain_variant == 77 && mid && wk.rtab_ok) return launch_run<256, 2, 2>(wk, s, b, e, true);
#ifdef SPLBCU_TUNING
        // warp-autonomous push kernel: measured slower (C3 developed 14.8-15.1k
        // vs 16.6-16.7k for the CTA-wide TMA pipeline, profiles/r02/sweep_dev_pushw.jsonl)
        if ((plain_variant == 74 || plain_variant == 75) && mid && wk.ctab_ok) {
            if (plain_variant == 74) return launch_push_w<4, 4>(wk, s, b, e);
            return launch_push_w<4, 3>(wk, s, b, e);
        }
#endif
        if (mid && wk.rtab_ok && plain_variant == 0 && wk.mid_pick == 2) return launch_run<256, 2, 2>(wk, s, b, e);
        if (mid && wk.ctab_ok) {
            const bool pf = plain_variant == 59 || (plain_variant == 0 && wk.mid_pick == 1);
            if (pf) launch_tmc<256, 2, 2, 4102>(wk, s, b, e);
            else if (plain_variant == 43) launch_tmc<256, 2, 2, 6>(wk, s, b, e);
#ifdef SPLBCU_TUNING
            else if (plain_variant == 82) launch_dyn<128, 2, 4>(wk, s, b, e);
            else if (plain_variant == 83) launch_dyn<128, 3, 3>(wk, s, b, e);
            else if (plain_variant == 84) launch_dyn<256, 3, 1>(wk, s, b, e);
#endif
            else launch_dyn<256, 2, 2>(wk, s, b, e);
        } else {
            launch_tma<256, 2, 2, false, 6>(wk, s, b, e);
        }
    }

#ifdef SPLBCU_TUNING
    // Tuning sweep variants (SPLBCU_PLAIN_VARIANT; measured slower than the
    // defaults, profiles/r01_sweep_*.log).  Returns false for the built-in ones.
    bool launch_tuning_variant(WorkerDev& wk, cudaStream_t s, uint32_t b, uint32_t e, const IoletArgs& ia, bool mid) {
        if (plain_variant == 0 || plain_variant == 24 || plain_variant == 43 || plain_variant == 59 ||
            plain_variant == 60 || plain_variant == 64 || plain_variant == 71 || plain_variant == 72 ||
            plain_variant == 76 || plain_variant == 77 || plain_variant == 78 || plain_variant == 79 ||
            plain_variant == 80 || plain_variant == 81 || (plain_variant >= 82 && plain_variant <= 84) ||
            (plain_variant >= 88 && plain_variant <= 96))
            return false;
        if (plain_variant == 69 || plain_variant == 70) {  // tile-major table, one bulk copy per tile
            if (!(mid && wk.ctab_ok)) launch_tma<256, 2, 2, false, 6>(wk, s, b, e);
            else if (plain_variant == 69) launch_tmc<256, 2, 2, 16386>(wk, s, b, e);
            else launch_tmc<256, 2, 2, 16386 | 8192>(wk, s, b, e);
            return true;
        }
        if (plain_variant == 67 || plain_variant == 68) {  // bounce-back as a signed offset in plane i
            if (!(mid && wk.ctab_ok)) launch_tma<256, 2, 2, false, 6>(wk, s, b, e);
            else if (plain_variant == 67) launch_tmc<256, 2, 2, 8198>(wk, s, b, e);
            else launch_tmc<256, 2, 2, 12294>(wk, s, b, e);
            return true;
        }
        if (plain_variant >= 40 && plain_variant < 60) {
            if (mid && wk.ctab_ok) {
                switch (plain_variant) {
                    case 40: launch_tmc<256, 2, 2>(wk, s, b, e); return true;
                    case 41: launch_tmc<128, 2, 4>(wk, s, b, e); return true;
                    case 42: launch_tmc<128, 2, 3>(wk, s, b, e); return true;
                    case 43: launch_tmc<256, 2, 2, 6>(wk, s, b, e); return true;
                    case 44: launch_tmc<256, 2, 2, 0>(wk, s, b, e); return true;
                    case 45: launch_tmc<192, 2, 3, 6>(wk, s, b, e); return true;
                    case 46: launch_tmc<128, 2, 4, 6>(wk, s, b, e); return true;
                    case 47: launch_tmc<128, 3, 3, 6>(wk, s, b, e); return true;
                    case 48: launch_tmc<96, 2, 5, 6>(wk, s, b, e); return true;
                    case 49: launch_tmc<256, 2, 2, 10>(wk, s, b, e); return true;
                    case 52: launch_tmc<256, 2, 2, 38>(wk, s, b, e); return true;   // 43 + evict-last stores
                    case 53: launch_tmc<256, 2, 2, 36>(wk, s, b, e); return true;   // evict-first loads, evict-last stores
                    case 54: launch_tmc<256, 2, 2, 102>(wk, s, b, e); return true;  // 52 with fraction 0.5
                    case 55: launch_tmc<256, 2, 2, 100>(wk, s, b, e); return true;  // 53 with fraction 0.5
                    case 56: launch_tmc<256, 2, 2, 142>(wk, s, b, e); return true;  // deltas + group bases by TMA
                    case 57: launch_tmc<256, 2, 2, 138>(wk, s, b, e); return true;  // 56, evict-first bulk loads
                    case 58: launch_tmc<128, 3, 3, 142>(wk, s, b, e); return true;  // 56, 3 stages of 128
                    case 59: launch_tmc<256, 2, 2, 4102>(wk, s, b, e); return true;  // 43 + table prefetch after the divisions
                    default: launch_tmc<256, 2, 2>(wk, s, b, e); return true;
                }
            }
            launch_tma<256, 2, 2, false, 2>(wk, s, b, e);
            return true;
        }
        switch (plain_variant) {
            case 1: launch_plain_t<256, 1>(wk, s, b, e, ia); break;
            case 2: launch_plain_t<256, 2>(wk, s, b, e, ia); break;
            case 3: launch_plain_t<128, 4>(wk, s, b, e, ia); break;
            case 4: launch_plain_t<128, 5>(wk, s, b, e, ia); break;
            case 5: launch_plain_t<64, 8>(wk, s, b, e, ia); break;
            case 6: launch_plain_t<256, 3>(wk, s, b, e, ia); break;
            case 10: launch_tma<128, 3, 2>(wk, s, b, e); break;
            case 11: launch_tma<128, 2, 3>(wk, s, b, e); break;
            case 12: launch_tma<64, 3, 4>(wk, s, b, e); break;
            case 13: launch_tma<256, 2, 1>(wk, s, b, e); break;
            case 14: launch_tma<128, 4, 1>(wk, s, b, e); break;
            case 15: launch_tma<64, 4, 3>(wk, s, b, e); break;
            case 16: launch_tma<96, 2, 5>(wk, s, b, e); break;
            case 17: launch_tma<160, 2, 3>(wk, s, b, e); break;
            case 18: launch_tma<64, 2, 7>(wk, s, b, e); break;
            case 19: launch_tma<128, 2, 5, false>(wk, s, b, e); break;
            case 20: launch_tma<128, 2, 4, false>(wk, s, b, e); break;
            case 21: launch_tma<256, 2, 2, false>(wk, s, b, e); break;
            case 22: launch_tma<64, 2, 10, false>(wk, s, b, e); break;
            case 23: launch_tma<256, 2, 2, false, 1>(wk, s, b, e); break;
            case 24: launch_tma<256, 2, 2, false, 2>(wk, s, b, e); break;
            case 25: launch_tma<256, 2, 2, false, 3>(wk, s, b, e); break;
            case 26: launch_tma<256, 3, 1, false>(wk, s, b, e); break;
            case 27: launch_tma<192, 2, 2, false>(wk, s, b, e); break;
            case 28: launch_tma<256, 2, 2, false, 6>(wk, s, b, e); break;
            case 29: launch_tma<128, 2, 4, false, 2>(wk, s, b, e); break;
            case 30: launch_ws<128, 2, 3, true>(wk, s, b, e); break;
            case 31: launch_ws<128, 3, 2, true>(wk, s, b, e); break;
            case 32: launch_ws<256, 2, 1, true>(wk, s, b, e); break;
            case 33: launch_ws<128, 2, 3, false>(wk, s, b, e); break;
            case 34: launch_ws<256, 2, 2, false>(wk, s, b, e); break;
            case 35: launch_ws<128, 3, 3, false>(wk, s, b, e); break;
            case 36: launch_ws<128, 4, 2, false>(wk, s, b, e); break;
            case 37: launch_plain_t<128, 4>(wk, s, b, e, ia); break;
            default: return false;
        }
        return true;
    }
#endif

#ifdef SPLBCU_TUNING
    // Warp-specialised 2-D TMA launch (producer warp + T/32 consumer warps).
    template <int T, int S, int B, bool TS>
    void launch_ws(WorkerDev& wk, cudaStream_t s, uint32_t b, uint32_t e) {
        using Lm = PushWsSmem<T, S, TS>;
        if (!wk.tma_ok) {  // tiny worker: planes shorter than one TMA box
            IoletArgs ia{};
            return launch_plain_t<128, 4>(wk, s, b, e, ia);
        }
        const int resident = resident_ctas(lbm_push_ws<T, S, B, TS>, wk.dev, T + 32, Lm::kBytes);
        const int v = T == 128 ? 0 : 1;
        const uint32_t base = b & ~3u;
        const uint32_t ntiles = (e - base + T - 1) / T;
        const unsigned grid = unsigned(std::min<uint32_t>(ntiles, uint32_t(resident)));
        check_tiles(wk, base, ntiles, T);
        lbm_push_ws<T, S, B, TS><<<grid, T + 32, Lm::kBytes, s>>>(wk.tm_f[wk.old][v], wk.tm_t[v], wk.f_new(),
                                                                   wk.tab.get<uint32_t>(), wk.P, b, e, omega);
    }
#endif

    // Persistent TMA-pipelined launch: grid = resident CTAs (occupancy x SMs).
    template <int T, int S, int B, bool TS = true, int H = 0, bool P2 = false>
    void launch_tma(WorkerDev& wk, cudaStream_t s, uint32_t b, uint32_t e, const HaloArgs& halo = HaloArgs{}) {
        using Lm = PushTmaSmem<T, S, TS>;
        const int resident = resident_ctas(lbm_push_tma<T, S, B, TS, H, P2>, wk.dev, T, Lm::kBytes);
        const uint32_t base = b & ~3u;
        const uint32_t ntiles = (e - base + T - 1) / T;
        const unsigned grid = unsigned(std::min<uint32_t>(ntiles, uint32_t(resident)));
        check_tiles(wk, base, ntiles, T);
        lbm_push_tma<T, S, B, TS, H, P2><<<grid, T, Lm::kBytes, s>>>(wk.f_old(), wk.f_new(), wk.tab.get<uint32_t>(),
                                                                   wk.P, b, e, omega, halo);
    }

    // Halo arguments of this step for the fused P2P path: the neighbours'
    // current f_new (all workers swap in lockstep, so the parity is ours).
    HaloArgs halo_args(const WorkerDev& wk) const {
        HaloArgs h{};
        for (size_t k = 0; k < wk.peer_f.size(); ++k) h.peer_fn[k] = wk.peer_f[k][1 - wk.old];
        h.slot_peer = wk.slot_peer.get<uint8_t>();
        h.slot_dst = wk.slot_dst.get<uint64_t>();
        return h;
    }

    // Records the start event of a timed bulk launch; returns its end event.
    cudaEvent_t timing_begin(WorkerDev& wk, cudaStream_t s) {
        std::vector<cudaEvent_t>& tv = wk.tev[run_par];
        size_t& used = wk.tev_used[run_par];
        if (used + 2 > tv.size())
            for (int k = 0; k < 2; ++k) {
                cudaEvent_t ev;
                CK(cudaEventCreate(&ev));
                tv.push_back(ev);
            }
        CK(cudaEventRecord(tv[used++], s));
        return tv[used++];
    }

    // fill_send_slots (engine.hpp:489-502), pull scheme only.
    void fill_send_slots(WorkerDev& wk, cudaStream_t s) {
        if (!wk.shared) return;
        if (p2p_mode)
            lbm_fill_send_slots<true><<<blocks_for(wk.shared), 256, 0, s>>>(
                wk.f_old(), wk.f_new(), wk.send_pos.get<uint64_t>(), wk.P, wk.shared, omega, halo_args(wk));
        else
            lbm_fill_send_slots<false><<<blocks_for(wk.shared), 256, 0, s>>>(
                wk.f_old(), wk.f_new(), wk.send_pos.get<uint64_t>(), wk.P, wk.shared, omega, HaloArgs{});
        launches++;
        CK(cudaGetLastError());
    }

    // `timed`: the bulk (mid-group) plain launch, whose CUDA-event duration
    // feeds the roofline; the small edge launches overlap it on another stream.
    // `edge` launches store cut-crossing links to the neighbours in P2P mode.
    void launch_range(WorkerDev& wk, cudaStream_t s, uint32_t b, uint32_t e, bool iolet, const double* staged,
                      const int32_t* coords, bool timed, bool edge = false) {
        if (e <= b) return;
        IoletArgs ia{wk.io_geo.get<IoletDev>(), staged, coords};
        if (pull_mode) {
            cudaEvent_t e1 = timed && kernel_timing ? timing_begin(wk, s) : nullptr;
            const unsigned nb = blocks_for(e - b, 128);
            if (iolet) lbm_pull<true><<<nb, 128, 0, s>>>(wk.f_old(), wk.f_new(), wk.tab.get<uint32_t>(), wk.P, b, e, omega, ia);
            else lbm_pull<false><<<nb, 128, 0, s>>>(wk.f_old(), wk.f_new(), wk.tab.get<uint32_t>(), wk.P, b, e, omega, ia);
            if (e1) CK(cudaEventRecord(e1, s));
            if (timed) {
                plain_launches++;
                plain_sites += e - b;
            }
            launches++;
            CK(cudaGetLastError());
            return;
        }
        const unsigned nb = blocks_for(e - b);
        const bool p2p = edge && p2p_mode && wk.shared > 0;
        if (iolet) {
            if (p2p)
                lbm_push<true, 256, 1, true><<<nb, 256, 0, s>>>(wk.f_old(), wk.f_new(), wk.tab.get<uint32_t>(), wk.P, b,
                                                                e, omega, ia, halo_args(wk));
            else
                lbm_push<true, 256, 1><<<nb, 256, 0, s>>>(wk.f_old(), wk.f_new(), wk.tab.get<uint32_t>(), wk.P, b, e,
                                                          omega, ia, HaloArgs{});
        } else if (p2p) {
            if (wk.tma_ok) launch_tma<256, 2, 2, false, 6, true>(wk, s, b, e, halo_args(wk));
            else
                lbm_push<false, 128, 4, true><<<unsigned((e - b + 127) / 128), 128, 0, s>>>(
                    wk.f_old(), wk.f_new(), wk.tab.get<uint32_t>(), wk.P, b, e, omega, ia, halo_args(wk));
        } else if (!timed) {
            launch_plain(wk, s, b, e, ia, false);
        } else {
            cudaEvent_t e1 = kernel_timing ? timing_begin(wk, s) : nullptr;
            launch_mid_tuned(wk, s, b, e, ia);
            if (e1) CK(cudaEventRecord(e1, s));
            plain_launches++;
            plain_sites += e - b;
        }
        launches++;
        CK(cudaGetLastError());
    }

    void advance_group(WorkerDev& wk, cudaStream_t s, bool edge, const double* staged) {
        const int32_t* ioc = wk.io_coords.get<int32_t>();
        if (edge) {
            launch_range(wk, s, 0, wk.ep, false, staged, ioc, false, true);
            launch_range(wk, s, wk.ep, wk.n_edge, true, staged, ioc, false, true);
            if (pull_mode) fill_send_slots(wk, s);
        } else {
            launch_range(wk, s, wk.n_edge, wk.n_edge + wk.mp, false, staged, ioc, true);
            launch_range(wk, s, wk.n_edge + wk.mp, wk.n, true, staged, ioc + 3 * uint64_t(wk.n_edge - wk.ep), false);
        }
    }

    void send_inproc(WorkerDev& wk) {
        for (const Seg& sg : wk.segs) {
            WorkerDev& peer = *W[size_t(sg.nb)];
            const Seg* ps = find_seg(peer, wk.w);
            const double* src = wk.f_new() + uint64_t(kQ) * wk.P + sg.base;
            double* dst = peer.f_old() + uint64_t(kQ) * peer.P + ps->base;
            if (wk.dev == peer.dev)
                CK(cudaMemcpyAsync(dst, src, sg.count * sizeof(double), cudaMemcpyDeviceToDevice, wk.sE));
            else
                CK(cudaMemcpyPeerAsync(dst, peer.dev, src, wk.dev, sg.count * sizeof(double), wk.sE));
        }
        CK(cudaEventRecord(wk.evSend, wk.sE));
    }

    void exchange_nccl(WorkerDev& wk) {
        const NcclApi& N = nccl();
        NK(N.GroupStart());
        for (const Seg& sg : wk.segs) {
            NK(N.Send(wk.f_new() + uint64_t(kQ) * wk.P + sg.base, sg.count, ncclDouble, sg.nb, comm, wk.sE));
            NK(N.Recv(wk.f_old() + uint64_t(kQ) * wk.P + sg.base, sg.count, ncclDouble, sg.nb, comm, wk.sE));
        }
        NK(N.GroupEnd());
    }

    void post_receive(WorkerDev& wk) {
        if (!wk.shared) return;
        lbm_post_receive<<<blocks_for(wk.shared), 256, 0, wk.sE>>>(
            wk.f_old() + uint64_t(kQ) * wk.P, wk.f_new(), wk.recv_flat.get<uint64_t>(), wk.shared);
        launches++;
        CK(cudaGetLastError());
    }

    void observe(WorkerDev& wk, cudaStream_t s, const double* f, uint64_t row) {
        if (!wk.n_obs) return;
        double* out = wk.obs_buf.get<double>() + 3 * (row - wk.obs_row_base) * wk.n_obs;
        if (aa_mode) {
            const int st = int(row & 1);  // AA state after `row` steps: S when odd
            if (p2p_mode)
                lbm_aa_observe<true><<<blocks_for(wk.n_obs), 256, 0, s>>>(
                    f, wk.tab.get<uint32_t>(), wk.P, wk.n_obs, st, halo_args(wk), wk.obs_site.get<uint32_t>(),
                    wk.obs_iolet.get<uint16_t>(), wk.io_geo.get<IoletDev>(), out);
            else
                lbm_aa_observe<false><<<blocks_for(wk.n_obs), 256, 0, s>>>(
                    f, wk.tab.get<uint32_t>(), wk.P, wk.n_obs, st, HaloArgs{}, wk.obs_site.get<uint32_t>(),
                    wk.obs_iolet.get<uint16_t>(), wk.io_geo.get<IoletDev>(), out);
        } else {
            lbm_iolet_observe<<<blocks_for(wk.n_obs), 256, 0, s>>>(f, wk.P, wk.n_obs, wk.obs_site.get<uint32_t>(),
                                                                   wk.obs_iolet.get<uint16_t>(),
                                                                   wk.io_geo.get<IoletDev>(), out);
        }
        launches++;
        CK(cudaGetLastError());
    }

    // Moments of every local site into wk.cap4 (internal order), either
    // storage scheme; `steps` = steps completed (AA state parity).
    void moments_to_cap4(WorkerDev& wk, cudaStream_t s, const double* f, uint64_t steps) {
        if (!wk.n) return;
        wk.cap4.reserve<double>(4 * uint64_t(wk.n));  // first capture / snapshot only
        if (aa_mode) {
            const int st = int(steps & 1);
            if (p2p_mode)
                lbm_aa_capture<true><<<blocks_for(wk.n), 256, 0, s>>>(f, wk.tab.get<uint32_t>(), wk.P, wk.n, st,
                                                                      halo_args(wk), wk.cap4.get<double>());
            else
                lbm_aa_capture<false><<<blocks_for(wk.n), 256, 0, s>>>(f, wk.tab.get<uint32_t>(), wk.P, wk.n, st,
                                                                       HaloArgs{}, wk.cap4.get<double>());
        } else {
            lbm_capture_moments<<<blocks_for(wk.n), 256, 0, s>>>(f, wk.P, wk.n, wk.cap4.get<double>());
        }
    }

    void capture(WorkerDev& wk, cudaStream_t s, const double* f, uint64_t step) {
        Capture* c = nullptr;
        for (Capture& x : caps)
            if (x.step == step) c = &x;
        if (!c) return;
        moments_to_cap4(wk, s, f, step);
        launches++;
        CK(cudaGetLastError());
        std::vector<double> h(4 * uint64_t(wk.n));
        if (wk.n) CK(cudaMemcpyAsync(h.data(), wk.cap4.get<double>(), h.size() * 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        for (uint32_t j = 0; j < wk.n; ++j)
            std::memcpy(&c->fields[4 * uint64_t(wk.global_of_int[j])], &h[4 * uint64_t(j)], 32);
    }

    // record_state (engine.hpp:546-555)
    void record_state(WorkerDev& wk, cudaStream_t s, uint64_t step, const double* f) {
        if (prm.capture_period > 0 && step % prm.capture_period == 0) capture(wk, s, f, step);
        if (prm.observe_iolets) observe(wk, s, f, step);
    }

    // prepare_records (engine.hpp:290-315)
    void prepare_records(uint64_t n) {
        if (prm.capture_period > 0) {
            const uint64_t p = prm.capture_period;
            for (uint64_t st = steps_run; st <= steps_run + n; ++st) {
                if (st % p != 0) continue;
                if (!caps.empty() && caps.back().step == st) continue;
                Capture c;
                c.step = st;
                c.fields.assign(4 * n_global, 0.0);
                caps.push_back(std::move(c));
            }
        }
        if (prm.observe_iolets) {
            const uint64_t rows = steps_run + n + 1;
            const uint64_t first = steps_run == 0 ? 0 : steps_run + 1;
            for (auto& wp : W) {
                if (!wp) continue;
                wp->obs_row_base = first;
                wp->obs_rows = rows - first;
                CK(cudaSetDevice(wp->dev));
                wp->obs_buf.reserve<double>(dist ? obs_gather_per(*wp)
                                                 : 3 * std::max<uint64_t>(wp->obs_rows * wp->n_obs, 1));
            }
        }
    }

    // ---- run(n): enqueue, then complete the previous run ---------------------
    // A run is enqueued in full (steps, observation gather, series kernels and
    // copies) and then the PREVIOUS run is completed — so consecutive run()
    // calls keep the GPU busy while the host waits for, times and reduces the
    // run before (its long iolets' series on the host overlap these steps).
    // Every accessor of results completes the pending run first.  Runs that
    // do host work inside the loop (captures) or reduce the series from a
    // single host buffer complete before returning.
    struct PendingRun {
        bool active = false, timing = false, series = false;
        int par = 0, ser_buf = 0;
        uint64_t ser_rows = 0;
        size_t caps_before = 0;
        bool first_run = false;
        std::chrono::steady_clock::time_point h0;
    };
    PendingRun pend;
    uint64_t max_run_n = 0;  // the longest run so far (buffer sizes follow it)
    const bool sync_runs = std::getenv("SPLBCU_SYNC_RUN") != nullptr;  // A/B knob: every run completes before returning
    const bool wait_series_off = std::getenv("SPLBCU_NO_SERIES_FIRST") != nullptr;  // A/B knob for the ordering below
    const bool series_on_main = std::getenv("SPLBCU_SERIES_ON_MAIN") != nullptr;  // A/B knob: N=1 series behind the steps
    const bool series_side_off = std::getenv("SPLBCU_SERIES_SIDE_OFF") != nullptr;  // A/B knob: dist series before the next run
    int run_par = 0;                                     // event / staging set of the run being enqueued
    PinnedMem h_staged2[2];                              // per-run iolet values, one per run in flight
    std::chrono::steady_clock::time_point last_done{};  // host clock at the last completion

    void run(uint64_t n) {
        if (failed) runtime_error("engine: an exchange failure left this simulation unusable");
        NvtxRange nv("splbcu::run");
        bool has_caps = false;
        if (prm.capture_period > 0)
            for (uint64_t st = steps_run == 0 ? 0 : steps_run + 1; st <= steps_run + n && !has_caps; ++st)
                has_caps = st % prm.capture_period == 0;
        const bool sync_run = has_caps || (prm.observe_iolets && !dev_series) || sync_runs;
        // A longer run than any before may grow the staging / observation
        // buffers, and cudaFree waits for every stream: complete the run in
        // flight first, under the watchdog (a dead neighbour must surface as an
        // exchange failure, not as a hang inside cudaFree).
        const bool grows = n > max_run_n;
        max_run_n = std::max(max_run_n, n);
        TRACE("run(%llu): rank %d, completing the run in flight: %d\n", (unsigned long long)n, rank,
              int(sync_run || grows));
        if (sync_run || grows) complete();
        const int par = run_par;
        const size_t caps_before = caps.size();
        const bool first_run = steps_run == 0;
        prepare_records(n);
        if (steps_run == 0)
            for (auto& wp : W)
                if (wp) {
                    CK(cudaSetDevice(wp->dev));
                    record_state(*wp, wp->sM, 0, wp->f_old());
                }
        // host staging of the per-step iolet values (engine.hpp:332-341) into
        // this run's pinned buffer (the run that used it before has completed),
        // copied stream-ordered ahead of the step loop
        const size_t n_io = bcs.size();
        const size_t n_staged = std::max<size_t>(n * n_io, 1);
        double* staged = h_staged2[par].reserve<double>(n_staged);
        staged[0] = 0.0;
        for (uint64_t k = 0; k < n; ++k) {
            const double t = double(steps_run + k + 1) * prm.dt_s;
            for (size_t io = 0; io < n_io; ++io) {
                const double v = bcs[io].table.at(t);
                staged[k * n_io + io] = bcs[io].kind == 1 ? v : v / kCs2;
            }
        }
        for (auto& wp : W) {
            if (!wp) continue;
            CK(cudaSetDevice(wp->dev));
            // dist mode with observation: the previous run's all-gather and
            // series kernels (on sE) go first.  Otherwise this run's persistent
            // bulk kernel can take every SM before the NCCL kernel, which then
            // lands after it and delays this run's edge kernels behind it.
            if (pend.active && dist && prm.observe_iolets && !wait_series_off)
                CK(cudaStreamWaitEvent(wp->sM, (pend.series && !series_side_off) ? wp->evObsFree[pend.par]
                                                                                 : wp->evDone[pend.par], 0));
            // one worker: this run's observations overwrite obs_buf once the
            // previous run's rows are gathered
            if (pend.active && !dist && pend.series) CK(cudaStreamWaitEvent(wp->sM, wp->evObsFree[pend.par], 0));
            double* d = wp->staged.reserve<double>(n_staged);
            CK(cudaMemcpyAsync(d, staged, n_staged * sizeof(double), cudaMemcpyHostToDevice, wp->sM));
            wp->tev_used[par] = 0;
        }
        const auto h0 = std::chrono::steady_clock::now();
        for (auto& wp : W)
            if (wp) {
                CK(cudaSetDevice(wp->dev));
                CK(cudaEventRecord(wp->evRun0[par], wp->sM));
                CK(cudaStreamWaitEvent(wp->sE, wp->evRun0[par], 0));
            }
        last_progress = std::chrono::steady_clock::now();
        try {
            for (uint64_t k = 0; k < n; ++k) {
                // at most kDepth steps in flight: the host waits for step
                // k - kDepth first, under the exchange watchdog
                if (k >= kDepth) wait_step(k - kDepth);
                if (k < 2 || k == kDepth) TRACE("run: enqueue step %llu\n", (unsigned long long)k);
                step_once(k, k * n_io);
                mark_step(k);
            }
        } catch (const Error& e) {
            if (e.kind == ErrKind::Comm) throw Error(ErrKind::Comm, "worker " + std::to_string(rank) + ": " + e.what());
            throw;
        }
        const bool series = prm.observe_iolets && dev_series;
        for (auto& wp : W) {
            if (!wp) continue;
            WorkerDev& wk = *wp;
            CK(cudaSetDevice(wk.dev));
            CK(cudaEventRecord(wk.evRun1[par], wk.sM));
            // this run's observation rows, behind the loop: one device
            // all-gather (dist mode) and one async copy into pinned memory
            if (prm.observe_iolets && dist) {
                const uint64_t per = obs_gather_per(wk);
                CK(cudaStreamWaitEvent(wk.sE, wk.evRun1[par], 0));
                const bool side = dev_series && !series_side_off;
                // the previous run's series gather has read the all-gathered rows
                if (side && pend.active && pend.series) CK(cudaStreamWaitEvent(wk.sE, wk.evSerRead[pend.par], 0));
                double* dr = obs_gather.reserve<double>(per * uint64_t(nranks));
                NK(nccl().AllGather(wk.obs_buf.get<double>(), dr, per, ncclDouble, comm, wk.sE));
                if (side) {
                    // the next run's steps wait for the all-gather only (it must
                    // not queue behind their persistent bulk kernel); the series
                    // kernels and copies run beside them on sS
                    CK(cudaEventRecord(wk.evObsFree[par], wk.sE));
                    CK(cudaStreamWaitEvent(wk.sS, wk.evObsFree[par], 0));
                    reduce_series_async(wk, wk.sS, dr, per, ser_next, wk.evSerRead[par]);
                    CK(cudaEventRecord(wk.evDone[par], wk.sS));
                    continue;
                }
                if (dev_series) {
                    reduce_series_async(wk, wk.sE, dr, per, ser_next);
                } else {
                    double* h = h_gather.reserve<double>(per * uint64_t(nranks));
                    CK(cudaMemcpyAsync(h, dr, per * uint64_t(nranks) * 8, cudaMemcpyDeviceToHost, wk.sE));
                }
                CK(cudaEventRecord(wk.evDone[par], wk.sE));
                continue;
            }
            if (series) {
                // one worker: the reduction and its copies run on the idle
                // edge stream beside the next run's steps, which wait only
                // for the rows to be gathered out of obs_buf (evObsFree)
                cudaStream_t ss = series_on_main ? wk.sM : wk.sE;
                if (!series_on_main) CK(cudaStreamWaitEvent(wk.sE, wk.evRun1[par], 0));
                reduce_series_async(wk, ss, wk.obs_buf.get<double>(), 0, ser_next, wk.evObsFree[par]);
                CK(cudaEventRecord(wk.evDone[par], ss));
                continue;
            }
            const size_t nb = prm.observe_iolets ? 3 * wk.obs_rows * wk.n_obs : 0;
            if (nb) {
                double* h = wk.h_obs.reserve<double>(nb);
                CK(cudaMemcpyAsync(h, wk.obs_buf.get<double>(), nb * 8, cudaMemcpyDeviceToHost, wk.sM));
            }
            CK(cudaEventRecord(wk.evDone[par], wk.sM));
        }
        // the previous run completes while these steps execute
        complete();
        steps_run += n;
        pend.active = true;
        pend.par = par;
        pend.timing = kernel_timing;
        pend.series = series;
        pend.ser_buf = ser_next;
        pend.ser_rows = steps_run + 1;
        pend.caps_before = caps_before;
        pend.first_run = first_run;
        pend.h0 = h0;
        if (series) ser_next ^= 1;
        run_par ^= 1;
        if (sync_run) complete();
    }

    // Completes the run in flight (if any): waits under the watchdog, adds its
    // device / host loop time and bulk-kernel times, reduces its series rows
    // and (dist mode) assembles its captures across ranks.
    void complete() {
        if (!pend.active) return;
        pend.active = false;
        last_progress = std::chrono::steady_clock::now();
        const int par = pend.par;
        std::vector<cudaEvent_t> done(W.size(), nullptr);
        for (size_t w = 0; w < W.size(); ++w)
            if (W[w]) done[w] = W[w]->evDone[par];
        try {
            wait_all(done);
        } catch (const Error& e) {
            if (e.kind == ErrKind::Comm) throw Error(ErrKind::Comm, "worker " + std::to_string(rank) + ": " + e.what());
            throw;
        }
        const auto h1 = std::chrono::steady_clock::now();
        double dmax = 0.0;
        for (auto& wp : W)
            if (wp) {
                float ms = 0.f;
                CK(cudaEventElapsedTime(&ms, wp->evRun0[par], wp->evRun1[par]));
                dmax = std::max(dmax, double(ms) * 1e-3);
                if (pend.timing)
                    for (size_t q = 0; q + 1 < wp->tev_used[par]; q += 2) {
                        float kms = 0.f;
                        CK(cudaEventElapsedTime(&kms, wp->tev[par][q], wp->tev[par][q + 1]));
                        plain_s += double(kms) * 1e-3;
                    }
            }
        dev_loop_s += dmax;
        // host loop time: from this run's enqueue (or the previous completion,
        // when the runs overlapped) to its completion
        loop_s += std::chrono::duration<double>(h1 - std::max(pend.h0, last_done)).count();
        last_done = h1;
        if (pend.series) {
            ser_pending = true;
            ser_pend_buf = pend.ser_buf;
            ser_pend_rows = pend.ser_rows;
            flush_series();  // the long iolets, on the host while the next run executes
        } else {
            assemble_series();
        }
        if (dist) {
            // captures of this run hold this rank's sites only: assemble them
            for (size_t c = 0; c < caps.size(); ++c)
                if (c >= pend.caps_before || (pend.first_run && caps[c].step == 0))
                    allreduce_host_sum(caps[c].fields.data(), caps[c].fields.size());
        }
    }

    // ---- progress watchdog (Mailbox::take, engine.hpp:92-101) ----------------
    // The reference fails a worker whose neighbour's message does not arrive
    // within exchange_timeout_s.  Here every step ends with a progress event
    // per local worker; the host keeps at most kDepth steps in flight and, in
    // dist mode, fails the run when no step has completed for
    // exchange_timeout_s (a dead or stuck neighbour), checking NCCL's
    // asynchronous errors while it waits.
    // 16 steps keep the GPU fed (>= 16 x the shortest step) while a stuck
    // neighbour can never fill the streams' command queues: the host always
    // reaches the watchdog instead of blocking inside a launch
    static constexpr uint64_t kDepth = 16;
    bool failed = false;  // an exchange failure left the streams unusable
    std::chrono::steady_clock::time_point last_progress;

    void mark_step(uint64_t k) {
        for (auto& wp : W) {
            if (!wp) continue;
            WorkerDev& wk = *wp;
            CK(cudaSetDevice(wk.dev));
            if (wk.prog.empty()) {
                wk.prog.resize(kDepth, nullptr);
                for (auto& ev : wk.prog) CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
            }
            CK(cudaEventRecord(wk.prog[k % kDepth], wk.sM));
        }
    }

    void wait_step(uint64_t k) {
        for (size_t w = 0; w < W.size(); ++w)
            if (W[w]) wait_event(int(w), W[w]->prog[k % kDepth]);
    }

    void wait_event(int w, cudaEvent_t ev) {
        CK(cudaSetDevice(W[size_t(w)]->dev));
        if (!dist) {
            CK(cudaEventSynchronize(ev));
            return;
        }
        for (int spins = 0;; ++spins) {
            const cudaError_t q = cudaEventQuery(ev);
            if (q == cudaSuccess) {
                last_progress = std::chrono::steady_clock::now();
                return;
            }
            if (q != cudaErrorNotReady) CK(q);
            ncclResult_t ar = ncclSuccess;
            NK(nccl().CommGetAsyncError(comm, &ar));
            if (ar != ncclSuccess && ar != ncclInProgress)
                fail(ErrKind::Comm, std::string("exchange failure: NCCL async error: ") + nccl().GetErrorString(ar));
            const double el =
                std::chrono::duration<double>(std::chrono::steady_clock::now() - last_progress).count();
            if (spins % 20000 == 0) TRACE("watchdog: worker %d waiting %.1f s\n", w, el);
            if (el > prm.exchange_timeout_s) exchange_timeout(w);
            if (spins < 2000) std::this_thread::yield();
            else std::this_thread::sleep_for(std::chrono::microseconds(50));
        }
    }

    // No progress for exchange_timeout_s: fail.  No CUDA call follows: a stream
    // operation queued now could sit behind the streams blocked on the dead
    // neighbour's flags (they share hardware queues), so the failed engine's
    // memory is leaked at teardown instead.
    [[noreturn]] void exchange_timeout(int w) {
        failed = true;
        g_leak_on_free.store(true);
        const WorkerDev& wk = *W[size_t(w)];
        const int nb = wk.segs.empty() ? -1 : wk.segs.front().nb;
        // NCCL halo: abort the communicator (its kernels wait for the dead
        // peer).  Fused P2P halo: the communicator is idle, and aborting it
        // frees device memory — cudaFree waits for every stream, including the
        // ones blocked on the peer's flags — so it is left to process exit.
        TRACE("watchdog: worker %d timed out; %s the communicator\n", w, p2p_mode ? "leaving" : "aborting");
        if (comm && !p2p_mode) nccl().CommAbort(comm);
        comm = nullptr;
        fail(ErrKind::Comm, "exchange failure: worker " + std::to_string(w) + " timed out waiting for neighbor " +
                                std::to_string(nb));
    }

    // Waits for this run's trailing work (observation copies) under the same watchdog.
    void wait_all(const std::vector<cudaEvent_t>& ev) {
        for (size_t w = 0; w < W.size(); ++w)
            if (W[w]) wait_event(int(w), ev[w]);
    }

    // advance_one (engine.hpp:330-363) for every local worker.
    // ---- AA single-buffer scheme ------------------------------------------------
    template <int T, int S, int B>
    void launch_aa_even_tma(WorkerDev& wk, cudaStream_t s, uint32_t b, uint32_t e, bool dyn = false) {
        using Lm = PushTmaSmem<T, S, false>;
        const int resident = resident_ctas(lbm_aa_even_tma<T, S, B>, wk.dev, T, Lm::kBytes + S * 4);
        const uint32_t base = b & ~3u;
        const uint32_t ntiles = (e - base + T - 1) / T;
        const unsigned grid = unsigned(std::min<uint32_t>(ntiles, uint32_t(resident)));
        check_tiles(wk, base, ntiles, T);
        unsigned* ctr = dyn ? tile_counter(wk, s) : nullptr;
        lbm_aa_even_tma<T, S, B><<<grid, T, Lm::kBytes + S * 4, s>>>(wk.f_old(), wk.P, b, e, omega, ctr);
    }

#ifdef SPLBCU_TUNING
    template <int T, int S, int B>
    void launch_aa_odd_tmc(WorkerDev& wk, cudaStream_t s, uint32_t b, uint32_t e) {
        using Lm = AaOddSmem<T, S, B>;
        const int resident = resident_ctas(lbm_aa_odd_tmc<T, S, B>, wk.dev, T, Lm::kBytes);
        const uint32_t base = b & ~127u;
        const uint32_t ntiles = (e - base + T - 1) / T;
        const unsigned grid = unsigned(std::min<uint32_t>(ntiles, uint32_t(resident)));
        check_tiles(wk, base, ntiles, T);
        lbm_aa_odd_tmc<T, S, B><<<grid, T, Lm::kBytes, s>>>(wk.f_old(), wk.dtab.get<int16_t>(), wk.gbase.get<uint32_t>(),
                                                             wk.tab.get<uint32_t>(), wk.P, wk.PG, b, e, omega);
    }
#endif

#ifdef SPLBCU_TUNING
    template <int T, int B>
    void launch_aa_odd_async(WorkerDev& wk, cudaStream_t s, uint32_t b, uint32_t e) {
        using Lm = AaAsyncSmem<T>;
        const int resident = resident_ctas(lbm_aa_odd_async<T, B>, wk.dev, T, Lm::kBytes);
        const uint32_t base = b & ~127u;
        const uint32_t ntiles = (e - base + T - 1) / T;
        const unsigned grid = unsigned(std::min<uint32_t>(ntiles, uint32_t(resident)));
        check_tiles(wk, base, ntiles, T);
        Planes19 pl;
        for (int i = 0; i < kQ; ++i) pl.p[i] = wk.f_old() + uint64_t(i) * wk.P;
        lbm_aa_odd_async<T, B><<<grid, T, Lm::kBytes, s>>>(wk.f_old(), wk.dtab.get<int16_t>(), wk.gbase.get<uint32_t>(),
                                                             wk.tab.get<uint32_t>(), wk.P, wk.PG, b, e, omega, pl);
    }
#endif

    // Warp-autonomous AA odd kernel (persistent; cp.async gathers one tile ahead).
    template <int NW, int B, int O = 1>
    void launch_aa_odd_w(WorkerDev& wk, cudaStream_t s, uint32_t b, uint32_t e, bool dyn = false) {
        using Lm = AaOddW<NW, B>;
        const int resident = resident_ctas(lbm_aa_odd_w<NW, B, O>, wk.dev, NW * 32, Lm::kBytes);
        const uint32_t ntiles = (e - (b & ~31u) + 31) / 32;
        const unsigned grid = unsigned(std::min<uint32_t>((ntiles + NW - 1) / NW, uint32_t(resident)));
        Planes19 pl;
        for (int i = 0; i < kQ; ++i) pl.p[i] = wk.f_old() + uint64_t(i) * wk.P;
        unsigned* ctr = dyn ? tile_counter(wk, s) : nullptr;
        lbm_aa_odd_w<NW, B, O><<<grid, NW * 32, Lm::kBytes, s>>>(wk.f_old(), wk.dtab.get<int16_t>(), wk.gbase.get<uint32_t>(),
                                                           wk.tab.get<uint32_t>(), wk.P, wk.PG, b, e, omega, pl, ctr);
    }

#ifdef SPLBCU_TUNING
    // The same with the table staged in shared memory (decoded twice, not held).
    template <int NW, int B>
    void launch_aa_odd_s(WorkerDev& wk, cudaStream_t s, uint32_t b, uint32_t e, bool dyn = true) {
        using Lm = AaOddS<NW, B>;
        const int resident = resident_ctas(lbm_aa_odd_s<NW, B>, wk.dev, NW * 32, Lm::kBytes);
        const uint32_t ntiles = (e - (b & ~31u) + 31) / 32;
        const unsigned grid = unsigned(std::min<uint32_t>((ntiles + NW - 1) / NW, uint32_t(resident)));
        Planes19 pl;
        for (int i = 0; i < kQ; ++i) pl.p[i] = wk.f_old() + uint64_t(i) * wk.P;
        unsigned* ctr = dyn ? tile_counter(wk, s) : nullptr;
        lbm_aa_odd_s<NW, B><<<grid, NW * 32, Lm::kBytes, s>>>(wk.f_old(), wk.dtab.get<int16_t>(), wk.gbase.get<uint32_t>(),
                                                           wk.tab.get<uint32_t>(), wk.P, wk.PG, b, e, omega, pl, ctr);
    }
#endif

    void launch_aa_range(WorkerDev& wk, cudaStream_t s, uint32_t b, uint32_t e, bool iolet, const double* staged,
                         const int32_t* coords, bool timed, bool edge, bool odd) {
        if (e <= b) return;
        IoletArgs ia{wk.io_geo.get<IoletDev>(), staged, coords};
        const bool remote = edge && p2p_mode && wk.shared > 0;
        const HaloArgs h = remote ? halo_args(wk) : HaloArgs{};
        cudaEvent_t e1 = timed && kernel_timing ? timing_begin(wk, s) : nullptr;
        double* F = wk.f_old();
        const uint32_t* tab = wk.tab.get<uint32_t>();
        const unsigned nb = blocks_for(e - b, 128);
        if (!odd) {
            if (iolet) lbm_aa_even<true><<<blocks_for(e - b), 256, 0, s>>>(F, tab, wk.P, b, e, omega, ia);
            else if (wk.tma_ok)  // the bulk (mid) range in one launch, dynamic tile order
                // (C3 developed even step 22,201 vs 19,532 fixed order; 79 forces the fixed order)
                launch_aa_even_tma<256, 2, 2>(wk, s, b, e, timed && plain_variant != 79);
            else lbm_aa_even<false><<<blocks_for(e - b), 256, 0, s>>>(F, tab, wk.P, b, e, omega, ia);
        } else if (remote) {
            if (iolet) lbm_aa_odd<true, true, 128, 4><<<nb, 128, 0, s>>>(F, tab, wk.P, b, e, omega, ia, h);
            else lbm_aa_odd<false, true, 128, 4><<<nb, 128, 0, s>>>(F, tab, wk.P, b, e, omega, ia, h);
        } else {
            const int v = plain_variant;
            if (iolet) lbm_aa_odd<true, false, 128, 4><<<nb, 128, 0, s>>>(F, tab, wk.P, b, e, omega, ia, h);
#ifdef SPLBCU_TUNING
            else if (timed && wk.ctab_ok && v >= 61 && v <= 66 && v != 64) {
                if (v == 61) launch_aa_odd_tmc<128, 2, 4>(wk, s, b, e);
                else if (v == 62) launch_aa_odd_tmc<256, 3, 2>(wk, s, b, e);
                else if (v == 63) launch_aa_odd_tmc<256, 2, 2>(wk, s, b, e);
                else if (v == 66)  // cp.async gathers (C3 developed: 13.1k vs 13.6k default)
                    for_parts(b, e, [&](uint32_t c, uint32_t c1) { launch_aa_odd_async<256, 2>(wk, s, c, c1); });
                else
                    lbm_aa_odd_c<256, 2><<<unsigned((e - (b & ~31u) + 255) / 256), 256, 0, s>>>(
                        F, wk.dtab.get<int16_t>(), wk.gbase.get<uint32_t>(), tab, wk.P, wk.PG, b, e, omega);
            }
#endif
            else if (timed && wk.ctab_ok && v == 72) {
                launch_aa_odd_w<4, 4>(wk, s, b, e);  // 128 registers: spills (C3 odd 9.6k)
            }
#ifdef SPLBCU_TUNING
            // table staged in shared memory (C3 developed odd step: 14.3k at 12
            // warps/SM, 11.2k at 15 — shared-memory pipe stalls — vs 14.65k)
            else if (timed && wk.ctab_ok && v >= 88 && v <= 91) {
                if (v == 88) launch_aa_odd_s<5, 3>(wk, s, b, e);
                else if (v == 89) launch_aa_odd_s<4, 3>(wk, s, b, e);
                else if (v == 90) launch_aa_odd_s<7, 2>(wk, s, b, e);
                else launch_aa_odd_s<4, 3>(wk, s, b, e, false);
            }
#endif
#ifdef SPLBCU_TUNING
            // knobs of the default odd kernel (C3 odd step, profiles/r02/aa_split_rawtab*.jsonl):
            // 92 + the next batch's atomic requested ahead (15.9k vs 16.0k), 93 that alone
            // with the packed table (14.2k), 95/96 batches of 8 (15.0k / 14.5-14.9k vs 15.2k)
            else if (timed && wk.ctab_ok && (v == 92 || v == 93 || v == 95 || v == 96)) {
                if (v == 92) launch_aa_odd_w<4, 3, 3>(wk, s, b, e, true);
                else if (v == 93) launch_aa_odd_w<4, 3, 2>(wk, s, b, e, true);
                else if (v == 95) launch_aa_odd_w<4, 3, 5>(wk, s, b, e, true);
                else launch_aa_odd_w<4, 3, 7>(wk, s, b, e, true);
            }
#endif
            else if (timed && wk.ctab_ok && v == 94) {
                // the previous default: deltas packed two per register — the packing
                // waits for the table loads, a memory latency per tile (C3 odd 14.1k vs 15.4k)
                launch_aa_odd_w<4, 3, 0>(wk, s, b, e, true);
            } else if (timed && wk.ctab_ok && v == 64) {
                // round-1 default: one thread per site, register gather over the
                // compressed table (C3 developed, odd step: 13.7k MSUPS)
                const uint32_t b0 = b & ~31u;
                lbm_aa_odd_c<128, 4><<<unsigned((e - b0 + 127) / 128), 128, 0, s>>>(
                    F, wk.dtab.get<int16_t>(), wk.gbase.get<uint32_t>(), tab, wk.P, wk.PG, b, e, omega);
            } else if (timed && wk.ctab_ok && v != 60) {
                // default: warp-autonomous pipeline, cp.async gathers one tile
                // ahead (C3 developed, odd step: 14.2k MSUPS; C2 14.9k vs 13.6k)
                // with the dynamic warp-tile order (C3 odd step 14.2k vs 13.9k; 81: fixed order)
                // and the table one delta per register (15.4k vs 14.1k packed, 94)
                launch_aa_odd_w<4, 3>(wk, s, b, e, v != 81);
            } else lbm_aa_odd<false, false, 128, 4><<<nb, 128, 0, s>>>(F, tab, wk.P, b, e, omega, ia, h);
        }
        if (timed) {
            if (e1) CK(cudaEventRecord(e1, s));
            plain_launches++;
            plain_sites += e - b;
        }
        launches++;
        CK(cudaGetLastError());
    }

    void advance_group_aa(WorkerDev& wk, cudaStream_t s, bool edge, const double* staged, bool odd) {
        const int32_t* ioc = wk.io_coords.get<int32_t>();
        if (edge) {
            launch_aa_range(wk, s, 0, wk.ep, false, staged, ioc, false, true, odd);
            launch_aa_range(wk, s, wk.ep, wk.n_edge, true, staged, ioc, false, true, odd);
        } else {
            launch_aa_range(wk, s, wk.n_edge, wk.n_edge + wk.mp, false, staged, ioc, true, false, odd);
            launch_aa_range(wk, s, wk.n_edge + wk.mp, wk.n, true, staged, ioc + 3 * uint64_t(wk.n_edge - wk.ep),
                            false, false, odd);
        }
    }

    // One AA step for every local worker.  Only the odd steps' edge kernels
    // touch a neighbour (remote gathers and stores, in place); a neighbour
    // may start its next edge kernel once ours is done (flag word), while
    // the interior kernels never conflict across workers.
    void step_once_aa(uint64_t k, uint64_t staged_off) {
        const uint32_t g = uint32_t(steps_run + k);
        const bool odd = (g & 1u) != 0;
        for (auto& wp : W) {
            if (!wp) continue;
            WorkerDev& wk = *wp;
            CK(cudaSetDevice(wk.dev));
            const uint32_t* fl = wk.flags.get<uint32_t>();
            if (p2p_mode)
                for (const Seg& sg : wk.segs) wait_geq(wk.sE, fl + size_t(sg.nb), g);
            advance_group_aa(wk, wk.sE, true, wk.staged.get<double>() + staged_off, odd);
            if (p2p_mode)
                for (size_t j = 0; j < wk.segs.size(); ++j) write_flag(wk.sE, wk.peer_flags[j] + wk.w, g + 1);
        }
        for (auto& wp : W) {
            if (!wp) continue;
            WorkerDev& wk = *wp;
            CK(cudaSetDevice(wk.dev));
            advance_group_aa(wk, wk.sM, false, wk.staged.get<double>() + staged_off, odd);
            CK(cudaEventRecord(wk.evMid, wk.sM));
        }
        const uint64_t done = steps_run + k + 1;
        for (auto& wp : W) {
            if (!wp) continue;
            WorkerDev& wk = *wp;
            CK(cudaSetDevice(wk.dev));
            CK(cudaStreamWaitEvent(wk.sE, wk.evMid, 0));
            const bool rec = (prm.capture_period > 0 && done % prm.capture_period == 0) || prm.observe_iolets;
            if (rec && p2p_mode) {  // state-S gathers read the neighbours' edge slots of this step
                const uint32_t* fl = wk.flags.get<uint32_t>();
                for (const Seg& sg : wk.segs) wait_geq(wk.sE, fl + size_t(sg.nb), g + 1);
            }
            if (prm.capture_period > 0 && done % prm.capture_period == 0)
                record_state(wk, wk.sE, done, wk.f_old());
            else if (prm.observe_iolets)
                observe(wk, wk.sE, wk.f_old(), done);
            CK(cudaEventRecord(wk.evEnd, wk.sE));
            CK(cudaStreamWaitEvent(wk.sM, wk.evEnd, 0));
        }
    }

    // Fused P2P step: the edge kernels store cut-crossing links straight into
    // the neighbours' f_new over NVLink; stream-ordered flag words replace
    // send/recv: wait until a neighbour is done reading the buffer we write
    // (its previous step), publish "halo delivered" after the edge kernels,
    // and wait for every neighbour's delivery before the step ends.
    void step_once_p2p(uint64_t k, uint64_t staged_off) {
        const uint32_t g = uint32_t(steps_run + k);  // global step index
        const size_t Wn = size_t(prm.workers);
        for (auto& wp : W) {
            if (!wp) continue;
            WorkerDev& wk = *wp;
            CK(cudaSetDevice(wk.dev));
            const uint32_t* fl = wk.flags.get<uint32_t>();
            for (const Seg& sg : wk.segs) wait_geq(wk.sE, fl + Wn + size_t(sg.nb), g);  // peer_done
            advance_group(wk, wk.sE, true, wk.staged.get<double>() + staged_off);
            for (size_t j = 0; j < wk.segs.size(); ++j) write_flag(wk.sE, wk.peer_flags[j] + wk.w, g + 1);  // halo_in
        }
        for (auto& wp : W) {
            if (!wp) continue;
            WorkerDev& wk = *wp;
            CK(cudaSetDevice(wk.dev));
            advance_group(wk, wk.sM, false, wk.staged.get<double>() + staged_off);
            CK(cudaEventRecord(wk.evMid, wk.sM));
        }
        const uint64_t done = steps_run + k + 1;
        for (auto& wp : W) {
            if (!wp) continue;
            WorkerDev& wk = *wp;
            CK(cudaSetDevice(wk.dev));
            CK(cudaStreamWaitEvent(wk.sE, wk.evMid, 0));
            const uint32_t* fl = wk.flags.get<uint32_t>();
            for (const Seg& sg : wk.segs) wait_geq(wk.sE, fl + size_t(sg.nb), g + 1);  // halos landed
            if (prm.capture_period > 0 && done % prm.capture_period == 0)
                record_state(wk, wk.sE, done, wk.f_new());
            else if (prm.observe_iolets)
                observe(wk, wk.sE, wk.f_new(), done);
            for (size_t j = 0; j < wk.segs.size(); ++j)
                write_flag(wk.sE, wk.peer_flags[j] + Wn + size_t(wk.w), g + 1);  // done reading f_old(g)
            CK(cudaEventRecord(wk.evEnd, wk.sE));
            CK(cudaStreamWaitEvent(wk.sM, wk.evEnd, 0));
            wk.old = 1 - wk.old;
        }
    }

    void step_once(uint64_t k, uint64_t staged_off) {
        NvtxRange nv("splbcu::step");
        if (aa_mode) return step_once_aa(k, staged_off);
        if (p2p_mode) return step_once_p2p(k, staged_off);
        const bool classic = prm.sequence == 0;
        // PreSend: edge sites
        for (auto& wp : W) {
            if (!wp) continue;
            WorkerDev& wk = *wp;
            CK(cudaSetDevice(wk.dev));
            advance_group(wk, wk.sE, true, wk.staged.get<double>() + staged_off);
            if (classic) {
                if (dist) exchange_nccl(wk);
                else send_inproc(wk);
            }
        }
        // PreReceive: mid sites on the second stream
        for (auto& wp : W) {
            if (!wp) continue;
            WorkerDev& wk = *wp;
            CK(cudaSetDevice(wk.dev));
            advance_group(wk, wk.sM, false, wk.staged.get<double>() + staged_off);
            CK(cudaEventRecord(wk.evMid, wk.sM));
            if (!classic) {
                CK(cudaStreamWaitEvent(wk.sE, wk.evMid, 0));
                if (dist) exchange_nccl(wk);
                else send_inproc(wk);
            }
        }
        // Receive + PostReceive
        for (auto& wp : W) {
            if (!wp) continue;
            WorkerDev& wk = *wp;
            CK(cudaSetDevice(wk.dev));
            if (!dist)
                for (const Seg& sg : wk.segs) CK(cudaStreamWaitEvent(wk.sE, W[size_t(sg.nb)]->evSend, 0));
            post_receive(wk);
        }
        // EndIteration: join, record, swap
        const uint64_t done = steps_run + k + 1;
        for (auto& wp : W) {
            if (!wp) continue;
            WorkerDev& wk = *wp;
            CK(cudaSetDevice(wk.dev));
            CK(cudaStreamWaitEvent(wk.sE, wk.evMid, 0));
            if (prm.capture_period > 0 && done % prm.capture_period == 0)
                record_state(wk, wk.sE, done, wk.f_new());
            else if (prm.observe_iolets)
                observe(wk, wk.sE, wk.f_new(), done);
            CK(cudaEventRecord(wk.evEnd, wk.sE));
            CK(cudaStreamWaitEvent(wk.sM, wk.evEnd, 0));
            wk.old = 1 - wk.old;
        }
    }

    // assemble_series (engine.hpp:602-629): reduce in ascending global order.
    // Completes the series with the pending run's batch (device path).
    void flush_series() {
        if (!ser_pending) return;
        ser_pending = false;
        assemble_series();
    }

    void assemble_series() {
        if (!prm.observe_iolets) return;
        const size_t n_io = dom.iolets.size();
        if (dev_series) {
            // (vmax, pressure, flow) per (row, iolet): short iolets reduced on
            // the device by run(); long ones here from their gathered entries
            const uint64_t first_row = series.rows, rows = ser_pend_rows;
            double* h = h_series[ser_pend_buf].get<double>();
            const double* raw = h_series_raw[ser_pend_buf].get<double>();
            for (uint64_t r = 0; r < rows - first_row; ++r)
                for (uint32_t k : ser_host_k) {
                    const uint32_t b = ser_be[2 * k], e = ser_be[2 * k + 1];
                    const double* v = raw + 3 * (r * ser_host_ent + b);
                    double vmax = 0.0, psum = 0.0, qsum = 0.0;
                    for (uint32_t j = b; j < e; ++j, v += 3) {
                        vmax = std::max(vmax, v[0]);
                        psum += v[1];
                        qsum += v[2];
                    }
                    double* o = h + 3 * (r * n_io + k);
                    o[0] = vmax;
                    o[1] = psum / double(e - b);
                    o[2] = qsum;
                }
            series.max_speed.resize(n_io);
            series.pressure.resize(n_io);
            series.flow.resize(n_io);
            for (size_t k = 0; k < n_io; ++k)
                for (uint64_t row = first_row; row < rows; ++row) {
                    const double* v = h + 3 * ((row - first_row) * n_io + k);
                    series.max_speed[k].push_back(v[0]);
                    series.pressure[k].push_back(v[1]);
                    series.flow[k].push_back(v[2]);
                }
            series.rows = rows;
            return;
        }
        // this run's rows were copied into each worker's pinned h_obs by run()
        std::vector<const double*> hb(W.size(), nullptr);
        for (size_t w = 0; w < W.size(); ++w)
            if (W[w]) hb[w] = W[w]->h_obs.get<double>();
        const uint64_t first_row = series.rows;
        const uint64_t rows = steps_run + 1;
        uint64_t row_base = 0;
        for (auto& wp : W)
            if (wp) row_base = wp->obs_row_base;
        if (dist) {
            // every worker's rows, all-gathered (padded) on the device by run()
            const uint64_t per = obs_gather_per(*W[size_t(rank)]);
            for (int w = 0; w < prm.workers; ++w) hb[size_t(w)] = h_gather.get<double>() + per * uint64_t(w);
        }
        series.max_speed.resize(n_io);
        series.pressure.resize(n_io);
        series.flow.resize(n_io);
        for (size_t k = 0; k < n_io; ++k) {
            series.max_speed[k].resize(rows);
            series.pressure[k].resize(rows);
            series.flow[k].resize(rows);
        }
        // each iolet's rows are an independent ordered reduction: iolets are
        // handed out one at a time to a few threads when there is enough work
        uint64_t work = 0;
        for (size_t k = 0; k < n_io; ++k) work += obs_order[k].size();
        work *= rows - first_row;
        std::atomic<size_t> next{0};
        auto reduce = [&] {
            for (size_t k; (k = next.fetch_add(1)) < n_io;)
                    for (uint64_t row = first_row; row < rows; ++row) {
                        double vmax = 0.0, psum = 0.0, qsum = 0.0;
                        for (const auto& [w, pos] : obs_order[k]) {
                            const std::vector<uint32_t>& off = obs_off_all[size_t(w)];
                            const double* v = hb[size_t(w)] + 3 * ((row - row_base) * off[n_io] + off[k] + pos);
                            vmax = std::max(vmax, v[0]);
                            psum += v[1];
                            qsum += v[2];
                        }
                        const double n_obs = double(obs_order[k].size());
                        series.max_speed[k][row] = vmax;
                        series.pressure[k][row] = psum / n_obs;
                        series.flow[k][row] = qsum;
                    }
        };
        const int nt = work > (1u << 16) ? int(std::min<size_t>({size_t(hw_threads()), size_t(8), n_io})) : 1;
        std::vector<std::thread> th;
        for (int t = 1; t < nt; ++t) th.emplace_back(reduce);
        reduce();
        for (auto& t : th) t.join();
        series.rows = rows;
    }

    // ---- host views -----------------------------------------------------------
    WorkerDev& local(int w) const {
        if (w < 0 || w >= prm.workers || !W[size_t(w)])
            runtime_error("engine: worker " + std::to_string(w) + " is not held by this process");
        return *W[size_t(w)];
    }

    void snapshot(double* out) {
        if (dist) std::fill(out, out + 4 * n_global, 0.0);
        for (auto& wp : W) {
            if (!wp) continue;
            WorkerDev& wk = *wp;
            CK(cudaSetDevice(wk.dev));
            moments_to_cap4(wk, wk.sM, wk.f_old(), steps_run);
            CK(cudaGetLastError());
            std::vector<double> h(4 * uint64_t(wk.n));
            if (wk.n) CK(cudaMemcpyAsync(h.data(), wk.cap4.get<double>(), h.size() * 8, cudaMemcpyDeviceToHost, wk.sM));
            CK(cudaStreamSynchronize(wk.sM));
            for (uint32_t j = 0; j < wk.n; ++j)
                std::memcpy(&out[4 * uint64_t(wk.global_of_int[j])], &h[4 * uint64_t(j)], 32);
        }
        if (dist) allreduce_host_sum(out, 4 * n_global);  // every rank returns the whole domain
    }

    // AA storage: f in the reference meaning, as 19 planes of P (internal order).
    std::vector<double> aa_planes(WorkerDev& wk) {
        DevMem tmp;
        double* d = tmp.alloc<double>(uint64_t(kQ) * wk.P);
        if (wk.n) {
            const int st = int(steps_run & 1);
            if (p2p_mode)
                lbm_aa_export<true><<<blocks_for(wk.n), 256, 0, wk.sM>>>(wk.f_old(), wk.tab.get<uint32_t>(), wk.P,
                                                                         wk.n, st, halo_args(wk), d);
            else
                lbm_aa_export<false><<<blocks_for(wk.n), 256, 0, wk.sM>>>(wk.f_old(), wk.tab.get<uint32_t>(), wk.P,
                                                                          wk.n, st, HaloArgs{}, d);
            CK(cudaGetLastError());
        }
        std::vector<double> h(uint64_t(kQ) * wk.P);
        CK(cudaMemcpyAsync(h.data(), d, h.size() * 8, cudaMemcpyDeviceToHost, wk.sM));
        CK(cudaStreamSynchronize(wk.sM));
        return h;
    }

    uint64_t ref_idx(const WorkerDev& wk, uint32_t r, int i) const {
        return prm.layout == 0 ? uint64_t(kQ) * r + uint64_t(i) : uint64_t(i) * wk.n + r;
    }

    void get_f(int w, int which, double* host) {
        WorkerDev& wk = local(w);
        CK(cudaSetDevice(wk.dev));
        CK(cudaDeviceSynchronize());
        if (aa_mode) {
            // one buffer: f_old is the current state (gathered by the AA rule);
            // f_new has no storage of its own (zeros); no shared tail
            std::fill(host, host + uint64_t(kQ) * wk.n + wk.shared, 0.0);
            if (which != 0) return;
            const std::vector<double> h = aa_planes(wk);
            for (uint32_t r = 0; r < wk.n; ++r) {
                const uint32_t j = wk.int_of_ref[r];
                for (int i = 0; i < kQ; ++i) host[ref_idx(wk, r, i)] = h[uint64_t(i) * wk.P + j];
            }
            return;
        }
        std::vector<double> h(wk.fsize());
        const double* src = which == 0 ? wk.f_old() : wk.f_new();
        CK(cudaMemcpy(h.data(), src, h.size() * 8, cudaMemcpyDeviceToHost));
        for (uint32_t r = 0; r < wk.n; ++r) {
            const uint32_t j = wk.int_of_ref[r];
            for (int i = 0; i < kQ; ++i) host[ref_idx(wk, r, i)] = h[uint64_t(i) * wk.P + j];
        }
        for (uint32_t k = 0; k < wk.shared; ++k) host[uint64_t(kQ) * wk.n + k] = h[uint64_t(kQ) * wk.P + k];
    }

    void set_f(int w, int which, const double* host) {
        WorkerDev& wk = local(w);
        CK(cudaSetDevice(wk.dev));
        CK(cudaDeviceSynchronize());
        if (aa_mode) {
            if (which != 0) return;  // no separate f_new in the single-buffer scheme
            if ((steps_run & 1) && prm.workers > 1)
                config_error("store(w): the AA scheme accepts f_old writes across workers after an even step count");
            std::vector<double> h(uint64_t(kQ) * wk.P, 0.0);
            for (uint32_t r = 0; r < wk.n; ++r) {
                const uint32_t j = wk.int_of_ref[r];
                for (int i = 0; i < kQ; ++i) h[uint64_t(i) * wk.P + j] = host[ref_idx(wk, r, i)];
            }
            DevMem tmp;
            double* d = tmp.alloc<double>(h.size());
            // stream-ordered: a legacy cudaMemcpy from pageable memory may
            // return before its DMA lands, and wk.sM does not wait for it
            CK(cudaMemcpyAsync(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice, wk.sM));
            if (wk.n)
                lbm_aa_import<<<blocks_for(wk.n), 256, 0, wk.sM>>>(wk.f_old(), wk.tab.get<uint32_t>(), wk.P, wk.n,
                                                                   int(steps_run & 1), d);
            CK(cudaGetLastError());
            CK(cudaStreamSynchronize(wk.sM));
            return;
        }
        std::vector<double> h(wk.fsize(), 0.0);
        for (uint32_t r = 0; r < wk.n; ++r) {
            const uint32_t j = wk.int_of_ref[r];
            for (int i = 0; i < kQ; ++i) h[uint64_t(i) * wk.P + j] = host[ref_idx(wk, r, i)];
        }
        for (uint32_t k = 0; k < wk.shared; ++k) h[uint64_t(kQ) * wk.P + k] = host[uint64_t(kQ) * wk.n + k];
        double* dst = which == 0 ? wk.f_old() : wk.f_new();
        CK(cudaMemcpyAsync(dst, h.data(), h.size() * 8, cudaMemcpyHostToDevice, wk.sM));
        CK(cudaStreamSynchronize(wk.sM));  // the steps' streams are non-blocking: land the data first
    }

    // StreamingMap in the reference encoding (layout.hpp:181-286) from the
    // device-built table.
    ExportedMap export_map(int w) {
        WorkerDev& wk = local(w);
        CK(cudaSetDevice(wk.dev));
        CK(cudaDeviceSynchronize());
        std::vector<uint32_t> tab(18 * wk.P);
        CK(cudaMemcpy(tab.data(), wk.tab.get<uint32_t>(), tab.size() * 4, cudaMemcpyDeviceToHost));
        std::vector<uint64_t> rf(wk.shared), sp(wk.shared);
        if (wk.shared) {
            CK(cudaMemcpy(rf.data(), wk.recv_flat.get<uint64_t>(), rf.size() * 8, cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(sp.data(), wk.send_pos.get<uint64_t>(), sp.size() * 8, cudaMemcpyDeviceToHost));
        }
        ExportedMap m;
        m.n_local = wk.n;
        m.shared_size = wk.shared;
        m.dest.resize(18 * uint64_t(wk.n));
        m.op.resize(18 * uint64_t(wk.n));
        m.iolet.resize(18 * uint64_t(wk.n));
        m.src_site.resize(18 * uint64_t(wk.n));
        m.src_op.resize(18 * uint64_t(wk.n));
        m.src_iolet.resize(18 * uint64_t(wk.n));
        for (uint32_t j = 0; j < wk.n; ++j) {
            const uint32_t r = wk.ref_of_int[j];
            for (int i = 1; i < kQ; ++i) {
                const uint32_t v = tab[uint64_t(i - 1) * wk.P + j];
                const uint64_t q = 18 * uint64_t(r) + uint64_t(i - 1);
                uint32_t dest;
                uint8_t op;
                uint16_t io = 0;
                if (v < kSpecial) {
                    dest = uint32_t(ref_idx(wk, wk.ref_of_int[v], i));
                    op = 0;
                } else {
                    const uint32_t o = (v >> kOpShift) & 3u;
                    if (o == kOpShared) {
                        dest = uint32_t(uint64_t(kQ) * wk.n + (v & kPayload));
                        op = 1;
                    } else if (o == kOpBounce) {
                        dest = uint32_t(ref_idx(wk, r, inv(i)));
                        op = 2;
                    } else {
                        dest = uint32_t(ref_idx(wk, r, inv(i)));
                        op = 3;
                        io = uint16_t(v & kPayload);
                    }
                }
                m.dest[q] = dest;
                m.op[q] = op;
                m.iolet[q] = io;
                // the pull-side source of (r, inverse(i)) follows from link i
                // (layout.hpp:243-282): FromLocal / FromRemote / SelfBounce / SelfIolet
                const uint64_t g = 18 * uint64_t(r) + uint64_t(inv(i) - 1);
                m.src_site[g] = op == 0 ? wk.ref_of_int[v] : (op == 1 ? 0u : r);
                m.src_op[g] = op;
                m.src_iolet[g] = io;
            }
        }
        m.recv_dest.resize(wk.shared);
        m.send_site.resize(wk.shared);
        m.send_dir.resize(wk.shared);
        for (uint32_t k = 0; k < wk.shared; ++k) {
            const uint64_t i = rf[k] / wk.P, j = rf[k] % wk.P;
            m.recv_dest[k] = uint32_t(ref_idx(wk, wk.ref_of_int[j], int(i)));
            const uint64_t i1 = sp[k] / wk.P, js = sp[k] % wk.P;
            m.send_site[k] = wk.ref_of_int[js];
            m.send_dir[k] = uint8_t(i1 + 1);
        }
        for (const Seg& sg : wk.segs) {
            m.seg_neighbor.push_back(sg.nb);
            m.seg_base.push_back(sg.base);
            m.seg_count.push_back(sg.count);
        }
        return m;
    }
};

// ---------------------------------------------------------------------------
Simulation::Simulation(const Domain& d, std::vector<BCEntry> bcs, Params p)
    : e_(std::make_unique<Engine>(d, std::move(bcs), std::move(p), 0, 1, nullptr)) {}
Simulation::Simulation(const Domain& d, std::vector<BCEntry> bcs, Params p, int rank, int nranks,
                       const void* nccl_id)
    : e_(std::make_unique<Engine>(d, std::move(bcs), std::move(p), rank, nranks, nccl_id)) {}
Simulation::Simulation(const Source& src, std::vector<BCEntry> bcs, Params p, int rank, int nranks,
                       const void* nccl_id)
    : e_(std::make_unique<Engine>(src, std::move(bcs), std::move(p), rank, nranks, nccl_id)) {}
Simulation::~Simulation() = default;
bool Simulation::slab_local() const { return e_->win != nullptr; }
uint64_t Simulation::n_sites() const { return e_->n_global; }
uint64_t Simulation::series_d2h_bytes() const { return e_->series_d2h_bytes(); }
void Simulation::run(uint64_t n) { e_->run(n); }
uint64_t Simulation::steps_run() const { return e_->steps_run; }
double Simulation::step_loop_seconds() const {
    e_->complete();
    return e_->loop_s;
}
double Simulation::device_loop_seconds() const {
    e_->complete();
    return e_->dev_loop_s;
}
double Simulation::plain_kernel_seconds() const {
    e_->complete();
    return e_->plain_s;
}
uint64_t Simulation::plain_kernel_launches() const { return e_->plain_launches; }
uint64_t Simulation::plain_kernel_sites() const { return e_->plain_sites; }
void Simulation::set_kernel_timing(bool on) { e_->kernel_timing = on; }
uint64_t Simulation::launch_count() const { return e_->launches; }
int Simulation::bulk_kernel() const { return e_->bulk_kernel(); }
void Simulation::snapshot(double* out) {
    e_->complete();
    e_->snapshot(out);
}
int Simulation::n_workers() const { return e_->prm.workers; }
bool Simulation::is_local(int w) const {
    return w >= 0 && w < e_->prm.workers && e_->W[size_t(w)] != nullptr;
}
void Simulation::store_shape(int w, uint32_t* n, uint32_t* shared) const {
    WorkerDev& wk = e_->local(w);
    if (n) *n = wk.n;
    if (shared) *shared = wk.shared;
}
void Simulation::get_f(int w, int which, double* host) {
    e_->complete();
    e_->get_f(w, which, host);
}
void Simulation::set_f(int w, int which, const double* host) {
    e_->complete();
    e_->set_f(w, which, host);
}
ExportedMap Simulation::export_map(int w) {
    e_->complete();
    return e_->export_map(w);
}
const Partition& Simulation::partition() const { return e_->part; }
const std::vector<Capture>& Simulation::captures() const {
    e_->complete();
    return e_->caps;
}
const Series& Simulation::series() const {
    e_->complete();
    e_->flush_series();
    return e_->series;
}

}  // namespace splbcu
