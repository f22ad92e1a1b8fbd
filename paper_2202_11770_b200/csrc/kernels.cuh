// sm_100a kernels of the sparse D3Q19 LBM step.
//
// Data layout in HBM (per worker):
//   f_old / f_new : 19 direction planes of P doubles (P = n_local rounded up
//                   to 64 sites, 512 B), then the totalSharedFs tail
//                   (reference layout.hpp:47-53 with a padded plane pitch).
//   tab           : 18 direction planes of P u32 — the push destination of
//                   (site s, direction i) as the neighbour's site index
//                   (ToLocal), or a tagged special entry (bounce-back,
//                   shared slot, iolet).  Direction-major so a warp's 32
//                   lanes read 128 contiguous bytes per direction.
// Site order inside a worker: edge group then mid group (decomp.hpp:155-186),
// each split into a plain range (Inner+Wall merged in (z,y,x) order, so row
// neighbours are adjacent and scattered writes coalesce) and an iolet range.
#pragma once

#include <cstdint>

#if defined(__CUDACC__)
#include <cuda.h>  // CUtensorMap (type only; encoding goes through the runtime's driver entry point)
#endif

#include "lattice.hpp"

namespace splbcu {

constexpr uint32_t kSpecial = 0x80000000u;
constexpr uint32_t kOpShift = 29;
constexpr uint32_t kPayload = (1u << 29) - 1;
constexpr uint32_t kOpBounce = 0, kOpShared = 1, kOpIolet = 2;

struct IoletDev {
    double center[3];
    double normal[3];
    double radius;
    int32_t is_velocity;
    int32_t pad;
};

#if defined(__CUDACC__)

// Streaming loads: each f_old / tab element is read once per step.
__device__ __forceinline__ double ld_f(const double* p) { return __ldcs(p); }
__device__ __forceinline__ uint32_t ld_t(const uint32_t* p) { return __ldcs(p); }

// Value streamed into (s, inverse(i)) by an iolet link i (engine.hpp:385-402).
__device__ __forceinline__ double iolet_link_value(int i, double fpost, const Macro& m,
                                                   const IoletDev& g, double staged,
                                                   int x, int y, int z) {
    if (g.is_velocity) {
        const double sw = staged * iolet_weight(g.center, g.normal, g.radius, x, y, z);
        const double ub0 = g.normal[0] * sw, ub1 = g.normal[1] * sw, ub2 = g.normal[2] * sw;
        return fpost - ladd_term(i, m.rho, ub0, ub1, ub2);
    }
    const double un = (m.ux * g.normal[0] + m.uy * g.normal[1]) + m.uz * g.normal[2];
    return feq_one(inv(i), staged, g.normal[0] * un, g.normal[1] * un, g.normal[2] * un);
}

struct IoletArgs {
    const IoletDev* io;
    const double* staged;    // this step's per-iolet value (speed or ghost density)
    const int32_t* coords;   // 3 ints per site of this launch's range, [s - begin]
};

// Fused halo (NVLink P2P): a cut-crossing link's post-collision value is
// stored straight into the neighbour GPU's f_new at its final destination
// (ExchangePlan::final_dest, exchange.hpp:20) instead of the local shared
// tail, so no send/recv and no PostReceive pass is needed.
constexpr int kMaxPeers = 8;
struct HaloArgs {
    double* peer_fn[kMaxPeers];  // neighbours' f_new this step (peer-mapped)
    const uint8_t* slot_peer;    // per shared slot: index into peer_fn
    const uint64_t* slot_dst;    // per shared slot: flat index in that f_new
};

template <bool kP2P>
__device__ __forceinline__ void store_shared(double* fn, uint64_t P, uint32_t slot, double v, const HaloArgs& h) {
    if constexpr (kP2P) h.peer_fn[h.slot_peer[slot]][h.slot_dst[slot]] = v;
    else fn[uint64_t(kQ) * P + slot] = v;
}

// Fused collide + push-stream over sites [begin, end) (update_push,
// engine.hpp:404-433).  One thread per site.
template <bool kIolets, int kThreads, int kMinBlocks, bool kP2P = false>
__global__ void __launch_bounds__(kThreads, kMinBlocks)
lbm_push(const double* __restrict__ fo, double* __restrict__ fn, const uint32_t* __restrict__ tab,
         uint64_t P, uint32_t begin, uint32_t end, double omega, IoletArgs ia, const __grid_constant__ HaloArgs halo) {
    const uint32_t s = begin + blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= end) return;
    double f[kQ];
#pragma unroll
    for (int i = 0; i < kQ; ++i) f[i] = ld_f(fo + uint64_t(i) * P + s);
    uint32_t t[kQ - 1];
#pragma unroll
    for (int i = 0; i < kQ - 1; ++i) t[i] = ld_t(tab + uint64_t(i) * P + s);

    const Macro m = macro_of(f);
    double feq[kQ];
    feq_all(m.rho, m.ux, m.uy, m.uz, feq);
    fn[s] = relax(f[0], feq[0], omega);
#pragma unroll
    for (int i = 1; i < kQ; ++i) {
        double fpost = relax(f[i], feq[i], omega);
        const uint32_t v = t[i - 1];
        uint64_t dst;
        if (v < kSpecial) {
            dst = uint64_t(i) * P + v;
        } else {
            const uint32_t op = (v >> kOpShift) & 3u;
            if (op == kOpShared) {
                if constexpr (kP2P) {
                    store_shared<true>(fn, P, v & kPayload, fpost, halo);
                    continue;
                }
                dst = uint64_t(kQ) * P + (v & kPayload);
            } else {
                dst = uint64_t(inv(i)) * P + s;
                if constexpr (kIolets) {
                    if (op == kOpIolet) {
                        const uint32_t k = v & kPayload;
                        const int32_t* c = ia.coords + 3 * uint64_t(s - begin);
                        fpost = iolet_link_value(i, fpost, m, ia.io[k], ia.staged[k], c[0], c[1], c[2]);
                    }
                }
            }
        }
        fn[dst] = fpost;
    }
}

// ---- pull scheme (update_pull + fill_send_slots, engine.hpp:435-502) ------
// One thread per destination site d.  Population j of d is gathered from the
// site the push step streams it from — the target of d's own link inverse(j)
// in the push table (layout.hpp:243-282 derives GatherSource the same way) —
// recomputing that source's collision as the reference does (its 19 x 19
// gather); wall and iolet links reconstruct it from d's own post-collision
// values.  FromRemote slots are left to the exchange (PostReceive or the
// neighbour's direct store).  Bitwise equal to the push step
// (test_engine.cpp:269-300): the same expression trees on the same inputs.
template <bool kIolets>
__global__ void __launch_bounds__(128)
lbm_pull(const double* __restrict__ fo, double* __restrict__ fn, const uint32_t* __restrict__ tab, uint64_t P,
         uint32_t begin, uint32_t end, double omega, IoletArgs ia) {
    const uint32_t d = begin + blockIdx.x * blockDim.x + threadIdx.x;
    if (d >= end) return;
    double fp[kQ];
    Macro md;
    {
        double f[kQ];
#pragma unroll
        for (int i = 0; i < kQ; ++i) f[i] = ld_f(fo + uint64_t(i) * P + d);
        md = macro_of(f);
        double feq[kQ];
        feq_all(md.rho, md.ux, md.uy, md.uz, feq);
#pragma unroll
        for (int i = 0; i < kQ; ++i) fp[i] = relax(f[i], feq[i], omega);
    }
    fn[d] = fp[0];
#pragma unroll
    for (int j = 1; j < kQ; ++j) {
        const int i = inv(j);
        const uint32_t v = __ldg(tab + uint64_t(i - 1) * P + d);
        double out;
        if (v < kSpecial) {  // FromLocal: the source's collision, recomputed
            double fs[kQ];
#pragma unroll
            for (int q = 0; q < kQ; ++q) fs[q] = __ldg(fo + uint64_t(q) * P + v);
            const Macro ms = macro_of(fs);
            out = relax(fs[j], feq_one(j, ms.rho, ms.ux, ms.uy, ms.uz), omega);
        } else {
            const uint32_t op = (v >> kOpShift) & 3u;
            if (op == kOpShared) continue;  // FromRemote
            out = fp[i];                    // SelfBounce
            if constexpr (kIolets) {
                if (op == kOpIolet) {       // SelfIolet
                    const uint32_t k = v & kPayload;
                    const int32_t* c = ia.coords + 3 * uint64_t(d - begin);
                    out = iolet_link_value(i, fp[i], md, ia.io[k], ia.staged[k], c[0], c[1], c[2]);
                }
            }
        }
        fn[uint64_t(j) * P + d] = out;
    }
}

// fill_send_slots (engine.hpp:489-502): the post-collision value of every
// outgoing shared slot (send site s, direction i) into the send tail, or
// straight into the neighbour's f_new in the fused P2P mode.
template <bool kP2P>
__global__ void lbm_fill_send_slots(const double* __restrict__ fo, double* __restrict__ fn,
                                    const uint64_t* __restrict__ send_pos, uint64_t P, uint32_t n, double omega,
                                    const __grid_constant__ HaloArgs halo) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const uint64_t tp = send_pos[k];  // (i - 1) * P + s
    const int i = int(tp / P) + 1;
    const uint64_t s = tp % P;
    double f[kQ];
#pragma unroll
    for (int q = 0; q < kQ; ++q) f[q] = fo[uint64_t(q) * P + s];
    const Macro m = macro_of(f);
    double feq[kQ];
    feq_all(m.rho, m.ux, m.uy, m.uz, feq);  // feq_all[i] == feq(i, m, usq_term(m)) bit for bit
    double fi = f[1], fe = feq[1];
#pragma unroll
    for (int q = 2; q < kQ; ++q)
        if (q == i) fi = f[q], fe = feq[q];
    store_shared<kP2P>(fn, P, k, relax(fi, fe, omega), halo);
}

// ---- TMA-pipelined persistent variant -------------------------------------
// The plain-site kernel is bound by HBM latency (ncu: long-scoreboard stalls
// dominate at the register-limited occupancy).  This version decouples loads
// from compute: a persistent CTA walks tiles of T sites; one thread streams
// the tile's 19 f-plane segments and 18 table-plane segments into shared
// memory with 1-D bulk async copies (cp.async.bulk, the TMA engine) completing
// on an mbarrier, S stages deep, while the CTA's threads collide+stream the
// previous tile from shared memory and scatter their 19 results to HBM.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ uint64_t evict_first_policy() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t evict_last_policy(float fraction) {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, %1;" : "=l"(p) : "f"(fraction));
    return p;
}
__device__ __forceinline__ void st_hint(double* p, double v, uint64_t policy) {
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(policy) : "memory");
}
// Ampere-style asynchronous copies global -> shared (LDGSTS): register-free
// loads completing per thread on cp.async groups.
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ uint64_t evict_normal_policy() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    return p;
}

template <int T, int S, bool kTabSmem = true>
struct PushTmaSmem {
    static constexpr uint32_t kF = uint32_t(kQ) * T * 8;                   // f tile
    static constexpr uint32_t kT = kTabSmem ? uint32_t(kQ - 1) * T * 4 : 0;  // table tile
    static constexpr uint32_t kStage = kF + kT;
    static constexpr uint32_t kBytes = S * kStage + S * 8;
};

// Sites [begin, end) of the plain (Inner+Wall) range.  Tiles start at
// begin rounded down to 4 sites (16-byte bulk-copy alignment); sites outside
// the range are loaded but neither computed nor stored.  Buffers carry a
// tail pad of T elements so the last tile's copies stay in bounds.
// kHints: bit0 = streaming (.cs) stores, bit1 = no L2 evict-first on the
// bulk loads (tuning knobs; default 0).
template <int T, int S, int kMinBlocks, bool kTabSmem = true, int kHints = 0, bool kP2P = false>
__global__ void __launch_bounds__(T, kMinBlocks)
lbm_push_tma(const double* __restrict__ fo, double* __restrict__ fn, const uint32_t* __restrict__ tab,
             uint64_t P, uint32_t begin, uint32_t end, double omega,
             const __grid_constant__ HaloArgs halo = HaloArgs{}) {
    using L = PushTmaSmem<T, S, kTabSmem>;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + S * L::kStage);
    const uint32_t base = begin & ~3u;
    const uint32_t ntiles = (end - base + T - 1) / T;
    const uint32_t G = gridDim.x;
    const uint32_t tid = threadIdx.x;
    if (tid == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&bar[s], 1);
        mbar_fence_init();
    }
    __syncthreads();
    const uint64_t policy = (kHints & 2) ? evict_normal_policy() : evict_first_policy();
    auto issue = [&](uint32_t k) {
        const uint32_t tile = blockIdx.x + k * G;
        if (tile >= ntiles) return;
        const int st = int(k % S);
        unsigned char* buf = smem + st * L::kStage;
        const uint64_t t0 = uint64_t(base) + uint64_t(tile) * T;
        mbar_expect_tx(&bar[st], L::kStage);
#pragma unroll 1
        for (int i = 0; i < kQ; ++i) bulk_g2s(buf + i * T * 8, fo + uint64_t(i) * P + t0, T * 8, &bar[st], policy);
        if constexpr (kTabSmem) {
#pragma unroll 1
            for (int i = 0; i < kQ - 1; ++i)
                bulk_g2s(buf + L::kF + i * T * 4, tab + uint64_t(i) * P + t0, T * 4, &bar[st], policy);
        }
    };
    if (tid == 0)
        for (uint32_t k = 0; k + 1 < uint32_t(S); ++k) issue(k);
    for (uint32_t k = 0;; ++k) {
        const uint32_t tile = blockIdx.x + k * G;
        if (tile >= ntiles) break;
        if (tid == 0) issue(k + S - 1);
        const int st = int(k % S);
        const uint32_t s = base + tile * T + tid;
        const bool live = s >= begin && s < end;
        uint32_t treg[kTabSmem ? 1 : kQ - 1];
        if constexpr (!kTabSmem) {
            // table straight to registers (coalesced), overlapping the wait
            if (live) {
#pragma unroll
                for (int i = 0; i < kQ - 1; ++i) {
                    if constexpr ((kHints & 4) != 0) treg[i] = __ldg(tab + uint64_t(i) * P + s);
                    else treg[i] = ld_t(tab + uint64_t(i) * P + s);
                }
            }
        }
        mbar_wait(&bar[st], (k / S) & 1u);
        const double* fs = reinterpret_cast<const double*>(smem + st * L::kStage);
        const uint32_t* ts = reinterpret_cast<const uint32_t*>(smem + st * L::kStage + L::kF);
        if (live) {
            double f[kQ];
#pragma unroll
            for (int i = 0; i < kQ; ++i) f[i] = fs[i * T + tid];
            const Macro m = macro_of(f);
            double feq[kQ];
            feq_all(m.rho, m.ux, m.uy, m.uz, feq);
            fn[s] = relax(f[0], feq[0], omega);
#pragma unroll
            for (int i = 1; i < kQ; ++i) {
                const double fpost = relax(f[i], feq[i], omega);
                uint32_t v;
                if constexpr (kTabSmem) v = ts[(i - 1) * T + tid];
                else v = treg[i - 1];
                uint64_t dst;
                if (v < kSpecial) dst = uint64_t(i) * P + v;
                else if (((v >> kOpShift) & 3u) == kOpShared) {
                    if constexpr (kP2P) {
                        store_shared<true>(fn, P, v & kPayload, fpost, halo);
                        continue;
                    }
                    dst = uint64_t(kQ) * P + (v & kPayload);
                } else dst = uint64_t(inv(i)) * P + s;
                if constexpr ((kHints & 1) != 0) __stcs(fn + dst, fpost);
                else fn[dst] = fpost;
            }
        }
        __syncthreads();  // stage st is free for the copy issued next iteration
    }
}

// Base address of each direction plane of f_new (fn + i*P), passed by value
// so per-store address math reads the constant bank instead of recomputing
// 64-bit plane offsets.
struct Planes19 {
    double* p[kQ];
};

// The escape of a run-length table entry (a group with more runs than the
// record holds) reads the u32 table; the condition is warp-uniform there, so
// a branch around the load is free (for the per-lane escapes of the delta
// table a predicated load measured faster: `lbm_push_tmc`).
__device__ __forceinline__ uint32_t escape_load(uint32_t t, bool esc, const uint32_t* p) {
    if (__any_sync(__activemask(), esc)) {
        if (esc) t = __ldg(p);
    }
    return t;
}

// ---- compressed neighbour table (mid-group plain sites) --------------------
// The mid-group plain range has only ToLocal and bounce-back links (shared
// slots occur only at edge sites, iolet links only at iolet sites).  Inside a
// warp's 32 consecutive sites (zyx order) the ToLocal targets of one direction
// are consecutive up to small jumps at row ends, so each (direction, 32-site
// group) stores one u32 base and every site an int16 delta:
//     target = base + lane + delta,   delta == kDeltaBounce -> (s, inv(i)).
// 18 x (2 + 4/32) = 38.25 B/site of index traffic instead of 72.
constexpr int16_t kDeltaBounce = -32768;
constexpr int16_t kDeltaEscape = -32767;

// One warp per (direction, 32-site group) over [begin, end); sets *err when a
// delta does not fit or an unexpected op appears (caller falls back to u32).
__global__ void compress_table(const uint32_t* __restrict__ tab, uint64_t P, uint64_t PG, uint32_t begin,
                               uint32_t end, int16_t* __restrict__ dtab, uint32_t* __restrict__ gbase,
                               unsigned* err) {
    const uint64_t gw = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = int(threadIdx.x & 31);
    const uint32_t g0 = begin >> 5, g1 = (end + 31) >> 5;
    const uint64_t ngroups = g1 - g0;
    if (gw >= ngroups * 18) return;  // whole warp exits together
    const int i1 = int(gw / ngroups);  // direction - 1
    const uint32_t g = g0 + uint32_t(gw % ngroups);
    const uint32_t s = g * 32 + uint32_t(lane);
    const bool live = s >= begin && s < end;
    const uint32_t v = live ? tab[uint64_t(i1) * P + s] : kSpecial;
    const bool local = live && v < kSpecial;
    const unsigned m = __ballot_sync(0xffffffffu, local);
    const int ref = m ? __ffs(int(m)) - 1 : 0;
    const uint32_t vref = __shfl_sync(0xffffffffu, v, ref);
    const int64_t base = m ? int64_t(vref) - ref : 0;
    int16_t d = 0;
    if (local) {
        const int64_t dd = int64_t(v) - base - lane;
        // far targets (e.g. the iolet sites stored after the plain range) take
        // the escape code and are read from the u32 table
        d = (dd < -32766 || dd > 32767) ? kDeltaEscape : int16_t(dd);
    } else if (live) {
        if (((v >> kOpShift) & 3u) != kOpBounce) atomicExch(err, 2u);
        d = kDeltaBounce;
    }
    if (live) dtab[uint64_t(i1) * P + s] = d;
    // the base may be "negative" (target of lane 0 below index 0): stored
    // modulo 2^32, the kernel adds lane + delta in the same arithmetic
    if (lane == 0) gbase[uint64_t(i1) * PG + g] = uint32_t(uint64_t(base));
}

// Tile-major copy of the compressed table (lbm_push_tmc kHints & 16384):
// tile j (sites [j*T, (j+1)*T)) = int16 deltas [18][T] then u32 group bases
// [18][T/32], contiguous, so one bulk copy per tile brings all of it.
template <int T>
__global__ void build_table_tiles(const int16_t* __restrict__ dtab, const uint32_t* __restrict__ gbase, uint64_t P,
                                  uint64_t PG, uint32_t tile0, uint32_t tile1, unsigned char* __restrict__ out) {
    constexpr uint32_t kD = uint32_t(kQ - 1) * T, kB = uint32_t(kQ - 1) * (T / 32);
    constexpr uint32_t kTab = kD * 2 + kB * 4;
    const uint64_t idx = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint32_t per = kD + kB;
    const uint64_t tile = tile0 + idx / per;
    if (tile >= tile1) return;
    const uint32_t e = uint32_t(idx % per);
    unsigned char* o = out + tile * kTab;
    if (e < kD) {
        const uint32_t i = e / T, j = e % T;
        reinterpret_cast<int16_t*>(o)[e] = dtab[uint64_t(i) * P + tile * T + j];
    } else {
        const uint32_t q = e - kD, i = q / (T / 32), g = q % (T / 32);
        reinterpret_cast<uint32_t*>(o + kD * 2)[q] = gbase[uint64_t(i) * PG + tile * (T / 32) + g];
    }
}

// TMA-pipelined persistent plain kernel reading the compressed table.  All
// 32 lanes run the direction loop (bases travel by warp shuffle); only loads
// and stores are predicated on the site being in range.
template <int T, int S, int kMinBlocks, int kHints = 2>
__global__ void __launch_bounds__(T, kMinBlocks)
lbm_push_tmc(const double* __restrict__ fo, double* __restrict__ fn, const int16_t* __restrict__ dtab,
             const uint32_t* __restrict__ gbase, const uint32_t* __restrict__ tab, uint64_t P, uint64_t PG,
             uint32_t begin, uint32_t end, double omega, const __grid_constant__ Planes19 planes) {
    using L = PushTmaSmem<T, S, false>;
    // kHints & 8: the tile's int16 deltas travel with its f planes (bulk
    // copies into the same stage) and the group bases are loaded one tile
    // ahead, so no table load latency is exposed in the direction loop
    // kHints & 16384: the tile's whole compressed table (deltas then group
    // bases, the kGS shared-memory layout) is ONE contiguous block of a
    // tile-major copy of the table (`dtab` then points at it; tiles aligned
    // to T sites), so one bulk copy per tile brings it with the f planes
    constexpr bool kTM = (kHints & 16384) != 0;
    constexpr bool kDS = (kHints & 8) != 0 || kTM;
    // kHints & 128 (with 8): the group bases too — 18 bulk copies of T/32 u32
    // per tile, so the loop body issues no global load at all
    constexpr bool kGS = (kDS && (kHints & 128) != 0) || kTM;
    constexpr uint32_t kDOff = L::kF, kGOff = L::kF + uint32_t(kQ - 1) * T * 2;
    constexpr uint32_t kStage = L::kF + (kDS ? uint32_t(kQ - 1) * T * 2 : 0u) + (kGS ? uint32_t(kQ - 1) * (T / 32) * 4 : 0u);
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + S * kStage);
    // warps cover aligned 32-site groups; kGS: tiles start on 128 sites so the
    // group-base copies are 16-byte aligned
    const uint32_t base = begin & (kTM ? ~uint32_t(T - 1) : (kGS ? ~127u : ~31u));
    const uint32_t ntiles = (end - base + T - 1) / T;
    const uint32_t G = gridDim.x;
    const uint32_t tid = threadIdx.x;
    const int lane = int(tid & 31);
    if (tid == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&bar[s], 1);
        mbar_fence_init();
    }
    __syncthreads();
    const uint64_t policy = (kHints & 2) ? evict_normal_policy() : evict_first_policy();
    // kHints & 32: f_new stores carry an L2 evict-last hint (a fraction 0.5 of
    // them with kHints & 64), so partially written sectors stay in L2 until
    // the slice-later writers complete them
    const uint64_t spolicy = evict_last_policy((kHints & 64) ? 0.5f : 1.0f);
    auto issue = [&](uint32_t k) {
        const uint32_t tile = blockIdx.x + k * G;
        if (tile >= ntiles) return;
        const int st = int(k % S);
        unsigned char* buf = smem + st * kStage;
        const uint64_t t0 = uint64_t(base) + uint64_t(tile) * T;
        mbar_expect_tx(&bar[st], kStage);
#pragma unroll 1
        for (int i = 0; i < kQ; ++i) bulk_g2s(buf + i * T * 8, fo + uint64_t(i) * P + t0, T * 8, &bar[st], policy);
        if constexpr (kTM) {
            constexpr uint32_t kTab = uint32_t(kQ - 1) * T * 2 + uint32_t(kQ - 1) * (T / 32) * 4;
            bulk_g2s(buf + kDOff, reinterpret_cast<const unsigned char*>(dtab) + (t0 / T) * kTab, kTab, &bar[st], policy);
        } else if constexpr (kDS) {
#pragma unroll 1
            for (int i = 0; i < kQ - 1; ++i)
                bulk_g2s(buf + kDOff + i * T * 2, dtab + uint64_t(i) * P + t0, T * 2, &bar[st], policy);
        }
        if constexpr (kGS && !kTM) {
#pragma unroll 1
            for (int i = 0; i < kQ - 1; ++i)
                bulk_g2s(buf + kGOff + i * (T / 32) * 4, gbase + uint64_t(i) * PG + (t0 >> 5), (T / 32) * 4, &bar[st],
                         policy);
        }
    };
    if (tid == 0)
        for (uint32_t k = 0; k + 1 < uint32_t(S); ++k) issue(k);
    auto load_base = [&](uint32_t tile) -> uint32_t {
        const uint32_t sg = base + tile * T + tid;
        return (lane < kQ - 1 && tile < ntiles) ? __ldg(gbase + uint64_t(lane) * PG + (sg >> 5)) : 0u;
    };
    uint32_t bnext = (kDS && !kGS) ? load_base(blockIdx.x) : 0u;
    // kHints & 4096: register prefetch of the next tile's table, issued after
    // this tile's divisions (whose slow-path CALL waits for every load in
    // flight) so it lands during the direction loop and the next TMA wait
    constexpr bool kPF = !kDS && (kHints & 4096) != 0;
    int16_t dn[kQ - 1];
    uint32_t bn = 0;
    auto load_table = [&](uint32_t tile, int16_t* d, uint32_t& b, uint32_t dep) {
        const uint32_t sn = base + tile * T + tid + dep;
        const bool ln = tile < ntiles && sn >= begin && sn < end;
#pragma unroll
        for (int i = 0; i < kQ - 1; ++i) d[i] = ln ? __ldg(dtab + uint64_t(i) * P + sn) : int16_t(0);
        b = (lane < kQ - 1 && tile < ntiles) ? __ldg(gbase + uint64_t(lane) * PG + (sn >> 5)) : 0u;
    };
    if constexpr (kPF) load_table(blockIdx.x, dn, bn, 0u);
    for (uint32_t k = 0;; ++k) {
        const uint32_t tile = blockIdx.x + k * G;
        if (tile >= ntiles) break;
        if (tid == 0) issue(k + S - 1);
        const int st = int(k % S);
        const uint32_t s = base + tile * T + tid;
        const bool live = s >= begin && s < end;
        int16_t dl[kQ - 1];
        uint32_t breg;
        if constexpr (kPF) {
#pragma unroll
            for (int i = 0; i < kQ - 1; ++i) dl[i] = dn[i];
            breg = bn;
            mbar_wait(&bar[st], (k / S) & 1u);
        } else if constexpr (kGS) {
            mbar_wait(&bar[st], (k / S) & 1u);
            const uint32_t* gs = reinterpret_cast<const uint32_t*>(smem + st * kStage + kGOff);
            breg = lane < kQ - 1 ? gs[lane * (T / 32) + (tid >> 5)] : 0u;
            const int16_t* ds = reinterpret_cast<const int16_t*>(smem + st * kStage + kDOff);
#pragma unroll
            for (int i = 0; i < kQ - 1; ++i) dl[i] = ds[i * T + tid];
        } else if constexpr (kDS) {
            breg = bnext;
            bnext = load_base(tile + G);
            mbar_wait(&bar[st], (k / S) & 1u);
            const int16_t* ds = reinterpret_cast<const int16_t*>(smem + st * kStage + kDOff);
#pragma unroll
            for (int i = 0; i < kQ - 1; ++i) dl[i] = ds[i * T + tid];
        } else {
#pragma unroll
            for (int i = 0; i < kQ - 1; ++i) {
                if constexpr ((kHints & 4) != 0) dl[i] = live ? __ldg(dtab + uint64_t(i) * P + s) : int16_t(0);
                else dl[i] = live ? __ldcs(dtab + uint64_t(i) * P + s) : int16_t(0);
            }
            breg = (lane < kQ - 1) ? __ldg(gbase + uint64_t(lane) * PG + (s >> 5)) : 0u;
            mbar_wait(&bar[st], (k / S) & 1u);
        }
        const double* fs = reinterpret_cast<const double*>(smem + st * kStage);
        double f[kQ];
#pragma unroll
        for (int i = 0; i < kQ; ++i) f[i] = fs[i * T + tid];
        const Macro m = macro_of(f);
        if constexpr (kPF) {
            // an always-zero term the compilers cannot fold (a popcount of 32
            // bits is at most 32) ties the prefetch addresses to the three
            // quotients, so the loads are not hoisted above the divisions
            uint32_t pc;
            asm("popc.b32 %0, %1;"
                : "=r"(pc)
                : "r"(uint32_t((__double_as_longlong(m.ux) ^ __double_as_longlong(m.uy) ^
                                __double_as_longlong(m.uz)) >> 32)));
            const uint32_t dep = pc >> 6;
            load_table(tile + G, dn, bn, dep);
        }
        double feq[kQ];
        feq_all(m.rho, m.ux, m.uy, m.uz, feq);
        if constexpr ((kHints & 32) != 0) {
            if (live) st_hint(fn + s, relax(f[0], feq[0], omega), spolicy);
        } else {
            if (live) fn[s] = relax(f[0], feq[0], omega);
        }
#pragma unroll
        for (int i = 1; i < kQ; ++i) {
            const double fpost = relax(f[i], feq[i], omega);
            const uint32_t b = __shfl_sync(0xffffffffu, breg, i - 1);
            const int d = dl[i - 1];
            // branch-free: the rare escape is a predicated load (inline PTX so
            // no divergent block is formed; a warp-uniform branch around it
            // measured 8 % slower from rest), the bounce case a select; plane
            // base addresses come from the constant bank (kernel params)
            uint32_t t = b + uint32_t(lane) + uint32_t(d);
            const uint32_t esc = (d == kDeltaEscape) && live;
            asm("{\n .reg .pred p;\n setp.ne.u32 p, %1, 0;\n @p ld.global.nc.u32 %0, [%2];\n}"
                : "+r"(t)
                : "r"(esc), "l"(tab + uint64_t(i - 1) * P + s));
            const bool bb = d == kDeltaBounce;
            double* dst;
            if constexpr ((kHints & 8192) != 0) {
                // one plane base per direction: a bounce-back target is site s
                // of the inverse plane, i.e. s +- P from plane i (inverse pairs
                // are adjacent indices), a signed 32-bit offset
                const int32_t off = (i & 1) ? int32_t(P) : -int32_t(P);
                dst = planes.p[i] + (bb ? int32_t(s) + off : int32_t(t));
            } else {
                const uintptr_t pb = reinterpret_cast<uintptr_t>(bb ? planes.p[inv(i)] : planes.p[i]);
                dst = reinterpret_cast<double*>(pb) + (bb ? s : t);
            }
            if constexpr ((kHints & 32) != 0) {
                if (live) st_hint(dst, fpost, spolicy);
            } else {
                if (live) *dst = fpost;
            }
        }
        __syncthreads();  // stage st is free for the copy issued next iteration
    }
}

// ---- run-length neighbour table (mid-group plain range) -------------------
// In (z,y,x) site order the ToLocal targets of one direction are consecutive
// along a row: inside a warp's 32-site group, target - lane is constant over
// runs of lanes (a row, or a row's interval between vessel walls) and
// changes only where the source or the target row changes.  Per direction i
// and group g: B = bounce-back lanes (and lanes outside the range), R = lanes
// starting a run (bit 0 always), rd[r] = target - lane of run r; a direction
// whose group has more than kRunK runs is escaped (R = 0: its lanes read the
// u32 table).  Tile-major, T = 256 sites = 8 groups per tile:
//     B[18][8] u32 | R[18][8] u32 | rd[18][8][kRunK] u32   = 3456 B per tile,
// one bulk copy per tile into the stage with the f planes: 13.5 B/site of
// index traffic (the delta table: 38.25), no global load in the direction
// loop.  On the C3 tree 97-99 % of (direction, group)s have <= 4 runs.
constexpr int kRunK = 4;
template <int T>
struct RunTab {
    static constexpr int kG = T / 32;
    static constexpr uint32_t kB = uint32_t(kQ - 1) * kG * 4;
    static constexpr uint32_t kRD = uint32_t(kQ - 1) * kG * kRunK * 4;
    static constexpr uint32_t kBytes = 2 * kB + kRD;
};

// One warp per (tile, direction, group) over tiles [tile0, tile1); err |= 1
// for an op other than ToLocal / bounce-back in the range; *n_esc counts the
// escaped (direction, group)s.
template <int T>
__global__ void build_run_table(const uint32_t* __restrict__ tab, uint64_t P, uint32_t begin, uint32_t end,
                                uint32_t tile0, uint32_t tile1, unsigned char* __restrict__ out, unsigned* err,
                                unsigned* n_esc) {
    using RT = RunTab<T>;
    const uint64_t gw = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t per_tile = uint64_t(kQ - 1) * RT::kG;
    const uint64_t tile = tile0 + gw / per_tile;
    if (tile >= tile1) return;  // whole warp
    const uint32_t rem = uint32_t(gw % per_tile), i1 = rem / RT::kG, g = rem % RT::kG;
    const uint64_t s = tile * T + g * 32 + lane;
    const bool live = s >= begin && s < end;
    const uint32_t v = live ? tab[uint64_t(i1) * P + s] : kSpecial;
    if (live && v >= kSpecial && ((v >> kOpShift) & 3u) != kOpBounce) atomicOr(err, 1u);
    const bool bounce = v >= kSpecial;
    const uint32_t delta = v - lane;
    const uint32_t nb = __ballot_sync(0xffffffffu, !bounce);
    const uint32_t prevmask = nb & ((1u << lane) - 1u);
    const int prev = prevmask ? 31 - __clz(int(prevmask)) : int(lane);
    const uint32_t pd = __shfl_sync(0xffffffffu, delta, prev);
    const bool newrun = !bounce && prevmask != 0 && delta != pd;
    const uint32_t R = __ballot_sync(0xffffffffu, newrun) | 1u;
    const int nr = __popc(R);
    const uint32_t le = lane == 31 ? 0xffffffffu : ((2u << lane) - 1u);
    const int r = __popc(R & le) - 1;
    const bool first = nb != 0 && int(lane) == __ffs(int(nb)) - 1;
    unsigned char* rec = out + tile * RT::kBytes;
    uint32_t* Bs = reinterpret_cast<uint32_t*>(rec);
    uint32_t* Rs = reinterpret_cast<uint32_t*>(rec + RT::kB);
    uint32_t* rd = reinterpret_cast<uint32_t*>(rec + 2 * RT::kB) + (i1 * RT::kG + g) * kRunK;
    const bool esc = nr > kRunK;
    if (lane == 0) {
        Bs[i1 * RT::kG + g] = ~nb;
        Rs[i1 * RT::kG + g] = esc ? 0u : R;
        if (esc) atomicAdd(n_esc, 1u);
    }
    if (lane < uint32_t(kRunK)) rd[lane] = 0u;
    __syncwarp();
    if (!esc && !bounce && (newrun || first)) rd[r] = delta;
}

// Persistent TMA-pipelined plain kernel over the run-length table: one bulk
// copy per tile brings the table with the 19 f planes; the direction loop
// decodes from shared memory (broadcast masks, <= kRunK distinct rd words per
// warp) and stores through the constant-bank plane bases, a bounce-back as
// the signed offset +-P within plane i.
template <int T, int S, int kMinBlocks>
__global__ void __launch_bounds__(T, kMinBlocks)
lbm_push_run(const double* __restrict__ fo, double* __restrict__ fn, const unsigned char* __restrict__ rtab,
             const uint32_t* __restrict__ tab, uint64_t P, uint32_t begin, uint32_t end, double omega,
             const __grid_constant__ Planes19 planes, unsigned* __restrict__ counter = nullptr) {
    using RT = RunTab<T>;
    constexpr uint32_t kF = uint32_t(kQ) * T * 8;
    constexpr uint32_t kStage = kF + RT::kBytes;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + S * kStage);
    uint32_t* tidx = reinterpret_cast<uint32_t*>(bar + S);  // dynamic order: tile of each stage
    const uint32_t base = begin & ~uint32_t(T - 1);  // tiles on the table's absolute grid
    const uint32_t ntiles = (end - base + T - 1) / T;
    const uint32_t G = gridDim.x;
    const uint32_t tid = threadIdx.x;
    const uint32_t lane = tid & 31, warp = tid >> 5;
    const uint32_t le = lane == 31 ? 0xffffffffu : ((2u << lane) - 1u);
    if (tid == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&bar[s], 1);
        mbar_fence_init();
    }
    __syncthreads();
    const uint64_t policy = evict_normal_policy();
    auto issue = [&](uint32_t k) {
        uint32_t tile = blockIdx.x + k * G;
        if (counter) tidx[k % S] = tile = atomicAdd(counter, 1u);
        if (tile >= ntiles) return;
        const int st = int(k % S);
        unsigned char* buf = smem + st * kStage;
        const uint64_t t0 = uint64_t(base) + uint64_t(tile) * T;
        mbar_expect_tx(&bar[st], kStage);
#pragma unroll 1
        for (int i = 0; i < kQ; ++i) bulk_g2s(buf + i * T * 8, fo + uint64_t(i) * P + t0, T * 8, &bar[st], policy);
        bulk_g2s(buf + kF, rtab + (t0 / T) * RT::kBytes, RT::kBytes, &bar[st], policy);
    };
    if (tid == 0)
        for (uint32_t k = 0; k + 1 < uint32_t(S); ++k) issue(k);
    if (counter) __syncthreads();
    for (uint32_t k = 0;; ++k) {
        const uint32_t tile = counter ? tidx[k % S] : blockIdx.x + k * G;
        if (tile >= ntiles) break;
        if (tid == 0) issue(k + S - 1);
        const int st = int(k % S);
        const uint32_t s = base + tile * T + tid;
        const bool live = s >= begin && s < end;
        mbar_wait(&bar[st], (k / S) & 1u);
        const unsigned char* buf = smem + st * kStage;
        const double* fs = reinterpret_cast<const double*>(buf);
        const uint32_t* Bs = reinterpret_cast<const uint32_t*>(buf + kF) + warp;
        const uint32_t* Rs = reinterpret_cast<const uint32_t*>(buf + kF + RT::kB) + warp;
        const uint32_t* rds = reinterpret_cast<const uint32_t*>(buf + kF + 2 * RT::kB) + warp * kRunK;
        double f[kQ];
#pragma unroll
        for (int i = 0; i < kQ; ++i) f[i] = fs[i * T + tid];
        const Macro m = macro_of(f);
        double feq[kQ];
        feq_all(m.rho, m.ux, m.uy, m.uz, feq);
        if (live) fn[s] = relax(f[0], feq[0], omega);
#pragma unroll
        for (int i = 1; i < kQ; ++i) {
            const double fpost = relax(f[i], feq[i], omega);
            const uint32_t Rm = Rs[(i - 1) * RT::kG];
            const uint32_t Bm = Bs[(i - 1) * RT::kG];
            const int r = __popc((Rm | 1u) & le) - 1;
            uint32_t t = rds[(i - 1) * RT::kG * kRunK + r] + lane;
            const uint32_t esc = Rm == 0u && live;
            t = escape_load(t, esc != 0u, tab + uint64_t(i - 1) * P + s);
            const bool bb = Rm == 0u ? t >= kSpecial : ((Bm >> lane) & 1u) != 0u;
            const int32_t off = (i & 1) ? int32_t(P) : -int32_t(P);
            double* dst = planes.p[i] + (bb ? int32_t(s) + off : int32_t(t));
            if (live) *dst = fpost;
        }
        __syncthreads();  // stage st is free for the copy issued next iteration
    }
}

// ---- warp-autonomous push kernel (delta table) ------------------------------
// Each warp walks its own 32-site tiles (persistent, no CTA barrier): the 19
// f-plane segments of tile k+1 are copied into the warp's shared-memory stage
// with 16-byte cp.async (register-free, in flight while tile k computes), the
// compressed table of tile k+1 is loaded into registers one tile ahead (deltas
// packed two per register), and tile k collides and scatters its 19 results.
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}

template <int kWarps, int kMinBlocks>
struct PushW {
    static constexpr uint32_t kStage = uint32_t(kQ) * 32 * 8;  // one warp-tile of f
    static constexpr uint32_t kBytes = 2 * kWarps * kStage;
};

template <int kWarps, int kMinBlocks>
__global__ void __launch_bounds__(kWarps * 32, kMinBlocks)
lbm_push_w(const double* __restrict__ fo, double* __restrict__ fn, const int16_t* __restrict__ dtab,
           const uint32_t* __restrict__ gbase, const uint32_t* __restrict__ tab, uint64_t P, uint64_t PG,
           uint32_t begin, uint32_t end, double omega, const __grid_constant__ Planes19 planes) {
    using L = PushW<kWarps, kMinBlocks>;
    extern __shared__ __align__(128) unsigned char smem[];
    const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    double* stage[2] = {reinterpret_cast<double*>(smem + (2 * wib) * L::kStage),
                        reinterpret_cast<double*>(smem + (2 * wib + 1) * L::kStage)};
    const uint32_t base = begin & ~31u;
    const uint32_t ntiles = (end - base + 31) / 32;
    const uint32_t nw = gridDim.x * kWarps;
    const uint32_t w0 = blockIdx.x * kWarps + wib;
    if (w0 >= ntiles) return;  // whole warp
    constexpr int kD2 = (kQ - 1) / 2;
    uint32_t dA[kD2], dB[kD2];
    uint32_t bA = 0, bB = 0;
    auto load_table = [&](uint32_t k, uint32_t* d, uint32_t& b) {
        const uint32_t tile = w0 + k * nw;
        const uint32_t s = base + tile * 32 + lane;
        const bool live = tile < ntiles && s >= begin && s < end;
#pragma unroll
        for (int i = 0; i < kD2; ++i) {
            const uint32_t lo = live ? uint16_t(__ldg(dtab + uint64_t(2 * i) * P + s)) : 0u;
            const uint32_t hi = live ? uint16_t(__ldg(dtab + uint64_t(2 * i + 1) * P + s)) : 0u;
            d[i] = lo | (hi << 16);
        }
        b = (lane < kQ - 1 && tile < ntiles) ? __ldg(gbase + uint64_t(lane) * PG + (s >> 5)) : 0u;
    };
    // the 19 plane segments of warp-tile k: 304 chunks of 16 B over 32 lanes
    auto copy_tile = [&](uint32_t k) {
        const uint32_t tile = w0 + k * nw;
        if (tile >= ntiles) return;
        const uint64_t t0 = uint64_t(base) + uint64_t(tile) * 32;
        double* st = stage[k & 1];
#pragma unroll
        for (int r = 0; r < 10; ++r) {
            const uint32_t c = uint32_t(r) * 32 + lane;
            if (c < uint32_t(kQ) * 16) {
                const uint32_t pl = c >> 4, off = (c & 15u) * 2;
                cp_async16(st + pl * 32 + off, fo + uint64_t(pl) * P + t0 + off);
            }
        }
    };
    auto step = [&](uint32_t k, const uint32_t* dK, uint32_t bK, uint32_t* dN, uint32_t& bN) -> bool {
        const uint32_t tile = w0 + k * nw;
        if (tile >= ntiles) return false;
        copy_tile(k + 1);
        cp_async_commit();
        load_table(k + 1, dN, bN);
        cp_async_wait<1>();
        __syncwarp();  // every lane's chunks of tile k are in
        const uint32_t s = base + tile * 32 + lane;
        const bool live = s >= begin && s < end;
        const double* st = stage[k & 1];
        double f[kQ];
#pragma unroll
        for (int i = 0; i < kQ; ++i) f[i] = st[i * 32 + lane];
        const Macro m = macro_of(f);
        double feq[kQ];
        feq_all(m.rho, m.ux, m.uy, m.uz, feq);
        if (live) fn[s] = relax(f[0], feq[0], omega);
#pragma unroll
        for (int i = 1; i < kQ; ++i) {
            const double fpost = relax(f[i], feq[i], omega);
            const uint32_t b = __shfl_sync(0xffffffffu, bK, i - 1);
            const int d = (i & 1) ? int(int16_t(dK[(i - 1) / 2] & 0xffffu)) : int(int16_t(dK[(i - 1) / 2] >> 16));
            uint32_t t = b + lane + uint32_t(d);
            const uint32_t esc = (d == kDeltaEscape) && live;
            asm("{\n .reg .pred p;\n setp.ne.u32 p, %1, 0;\n @p ld.global.nc.u32 %0, [%2];\n}"
                : "+r"(t)
                : "r"(esc), "l"(tab + uint64_t(i - 1) * P + s));
            const int32_t off = (i & 1) ? int32_t(P) : -int32_t(P);
            double* dst = planes.p[i] + (d == kDeltaBounce ? int32_t(s) + off : int32_t(t));
            if (live) *dst = fpost;
        }
        __syncwarp();  // stage k & 1 is refilled by tile k+2's copies
        return true;
    };
    load_table(0, dA, bA);
    copy_tile(0);
    cp_async_commit();
    for (uint32_t k = 0;; k += 2) {
        if (!step(k, dA, bA, dB, bB)) break;
        if (!step(k + 1, dB, bB, dA, bA)) break;
    }
    cp_async_wait<0>();
}

// ---- dynamic tile order (delta table, just-in-time table loads) ------------
// lbm_push_tmc<.., 6> with the persistent CTAs taking tiles from a global
// counter instead of the fixed stride blockIdx.x + k * grid: the tiles in
// flight stay within ~one grid's width of the frontier however the CTAs drift
// apart, so the scattered stores of the whole GPU hit a compact window of each
// direction plane (the effect that cutting the bulk range into parts buys).
template <int T, int S, int kMinBlocks>
__global__ void __launch_bounds__(T, kMinBlocks)
lbm_push_dyn(const double* __restrict__ fo, double* __restrict__ fn, const int16_t* __restrict__ dtab,
             const uint32_t* __restrict__ gbase, const uint32_t* __restrict__ tab, uint64_t P, uint64_t PG,
             uint32_t begin, uint32_t end, double omega, unsigned* __restrict__ counter,
             const __grid_constant__ Planes19 planes) {
    using L = PushTmaSmem<T, S, false>;
    constexpr uint32_t kStage = L::kF;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + S * kStage);
    uint32_t* tidx = reinterpret_cast<uint32_t*>(bar + S);  // tile of each stage
    const uint32_t base = begin & ~31u;
    const uint32_t ntiles = (end - base + T - 1) / T;
    const uint32_t tid = threadIdx.x;
    const int lane = int(tid & 31);
    if (tid == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&bar[s], 1);
        mbar_fence_init();
    }
    __syncthreads();
    const uint64_t policy = evict_normal_policy();
    auto issue = [&](uint32_t k) {  // thread 0: take the next tile for iteration k
        const int st = int(k % S);
        const uint32_t tile = atomicAdd(counter, 1u);
        tidx[st] = tile;
        if (tile >= ntiles) return;
        unsigned char* buf = smem + st * kStage;
        const uint64_t t0 = uint64_t(base) + uint64_t(tile) * T;
        mbar_expect_tx(&bar[st], kStage);
#pragma unroll 1
        for (int i = 0; i < kQ; ++i) bulk_g2s(buf + i * T * 8, fo + uint64_t(i) * P + t0, T * 8, &bar[st], policy);
    };
    if (tid == 0)
        for (uint32_t k = 0; k + 1 < uint32_t(S); ++k) issue(k);
    __syncthreads();
    for (uint32_t k = 0;; ++k) {
        const int st = int(k % S);
        const uint32_t tile = tidx[st];
        if (tile >= ntiles) break;
        if (tid == 0) issue(k + S - 1);
        const uint32_t s = base + tile * T + tid;
        const bool live = s >= begin && s < end;
        int16_t dl[kQ - 1];
#pragma unroll
        for (int i = 0; i < kQ - 1; ++i) dl[i] = live ? __ldg(dtab + uint64_t(i) * P + s) : int16_t(0);
        const uint32_t breg = (lane < kQ - 1) ? __ldg(gbase + uint64_t(lane) * PG + (s >> 5)) : 0u;
        mbar_wait(&bar[st], (k / S) & 1u);
        const double* fs = reinterpret_cast<const double*>(smem + st * kStage);
        double f[kQ];
#pragma unroll
        for (int i = 0; i < kQ; ++i) f[i] = fs[i * T + tid];
        const Macro m = macro_of(f);
        double feq[kQ];
        feq_all(m.rho, m.ux, m.uy, m.uz, feq);
        if (live) fn[s] = relax(f[0], feq[0], omega);
#pragma unroll
        for (int i = 1; i < kQ; ++i) {
            const double fpost = relax(f[i], feq[i], omega);
            const uint32_t b = __shfl_sync(0xffffffffu, breg, i - 1);
            const int d = dl[i - 1];
            uint32_t t = b + uint32_t(lane) + uint32_t(d);
            const uint32_t esc = (d == kDeltaEscape) && live;
            asm("{\n .reg .pred p;\n setp.ne.u32 p, %1, 0;\n @p ld.global.nc.u32 %0, [%2];\n}"
                : "+r"(t)
                : "r"(esc), "l"(tab + uint64_t(i - 1) * P + s));
            const bool bb = d == kDeltaBounce;
            const uintptr_t pb = reinterpret_cast<uintptr_t>(bb ? planes.p[inv(i)] : planes.p[i]);
            double* dst = reinterpret_cast<double*>(pb) + (bb ? s : t);
            if (live) *dst = fpost;
        }
        __syncthreads();  // stage st is free; the next stage's tile index is visible
    }
}

// ---- warp-specialised 2-D TMA variant --------------------------------------
// One TMA instruction per tile moves the whole [19 planes x T sites] f box
// (and, optionally, the [18 x T] table box) described by a CUtensorMap over
// the direction-major store.  A dedicated producer warp runs the S-stage ring
// with full/empty mbarriers; the T/32 consumer warps never meet at a CTA
// barrier.  OOB boxes past the plane end are zero-filled by the TMA unit.
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int32_t x, int32_t y, uint64_t* bar,
                                       uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

template <int T, int S, bool kTabSmem>
struct PushWsSmem {
    static constexpr uint32_t kF = uint32_t(kQ) * T * 8;
    static constexpr uint32_t kT = kTabSmem ? uint32_t(kQ - 1) * T * 4 : 0;
    static constexpr uint32_t kStage = kF + kT;
    static constexpr uint32_t kBytes = S * kStage + 2 * S * 8 + 128;  // + barriers + alignment slack
};

template <int T, int S, int kMinBlocks, bool kTabSmem>
__global__ void __launch_bounds__(T + 32, kMinBlocks)
lbm_push_ws(const __grid_constant__ CUtensorMap tm_f, const __grid_constant__ CUtensorMap tm_t,
            double* __restrict__ fn, const uint32_t* __restrict__ tab, uint64_t P, uint32_t begin, uint32_t end,
            double omega) {
    using L = PushWsSmem<T, S, kTabSmem>;
    extern __shared__ unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * L::kStage);
    uint64_t* empty = full + S;
    constexpr int kConsumerWarps = T / 32;
    const uint32_t base = begin & ~3u;
    const uint32_t ntiles = (end - base + T - 1) / T;
    const uint32_t G = gridDim.x;
    const int warp = int(threadIdx.x >> 5), lane = int(threadIdx.x & 31);
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kConsumerWarps);
        }
        mbar_fence_init();
    }
    __syncthreads();
    if (warp == kConsumerWarps) {  // producer
        if (lane == 0) {
            const uint64_t policy = evict_first_policy();
            for (uint32_t k = 0;; ++k) {
                const uint32_t tile = blockIdx.x + k * G;
                if (tile >= ntiles) break;
                const int st = int(k % S);
                if (k >= uint32_t(S)) mbar_wait(&empty[st], ((k / S) - 1) & 1u);
                mbar_expect_tx(&full[st], L::kStage);
                const int32_t x = int32_t(base + tile * T);
                tma_2d(smem + st * L::kStage, &tm_f, x, 0, &full[st], policy);
                if constexpr (kTabSmem) tma_2d(smem + st * L::kStage + L::kF, &tm_t, x, 0, &full[st], policy);
            }
        }
        return;
    }
    const uint32_t tid = threadIdx.x;
    for (uint32_t k = 0;; ++k) {
        const uint32_t tile = blockIdx.x + k * G;
        if (tile >= ntiles) break;
        const int st = int(k % S);
        const uint32_t s = base + tile * T + tid;
        const bool live = s >= begin && s < end;
        uint32_t treg[kTabSmem ? 1 : kQ - 1];
        if constexpr (!kTabSmem) {
            if (live) {
#pragma unroll
                for (int i = 0; i < kQ - 1; ++i) treg[i] = ld_t(tab + uint64_t(i) * P + s);
            }
        }
        mbar_wait(&full[st], (k / S) & 1u);
        const double* fs = reinterpret_cast<const double*>(smem + st * L::kStage);
        const uint32_t* ts = reinterpret_cast<const uint32_t*>(smem + st * L::kStage + L::kF);
        double f[kQ];
        if (live) {
#pragma unroll
            for (int i = 0; i < kQ; ++i) f[i] = fs[i * T + tid];
        }
        uint32_t tv[kQ - 1];
        if constexpr (kTabSmem) {
            if (live) {
#pragma unroll
                for (int i = 0; i < kQ - 1; ++i) tv[i] = ts[i * T + tid];
            }
        }
        // stage consumed: hand it back to the producer before the math
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
        if (live) {
            const Macro m = macro_of(f);
            double feq[kQ];
            feq_all(m.rho, m.ux, m.uy, m.uz, feq);
            fn[s] = relax(f[0], feq[0], omega);
#pragma unroll
            for (int i = 1; i < kQ; ++i) {
                const double fpost = relax(f[i], feq[i], omega);
                uint32_t v;
                if constexpr (kTabSmem) v = tv[i - 1];
                else v = treg[i - 1];
                uint64_t dst;
                if (v < kSpecial) dst = uint64_t(i) * P + v;
                else if (((v >> kOpShift) & 3u) == kOpShared) dst = uint64_t(kQ) * P + (v & kPayload);
                else dst = uint64_t(inv(i)) * P + s;
                fn[dst] = fpost;
            }
        }
    }
}

// ---- AA pattern: one distribution buffer, in place ---------
// State N ("natural", after an even number of steps): F[i][x] = f(x, i).
// Even step (N -> S), purely local: collide at x, store the post-collision
//   g_m(x) (or its iolet BC value) at F[inv(m)][x].
// State S: f(y, i) lives at F[inv(i)][y - c_i] when link inv(i) of y is a
//   fluid link (the source site's swapped slot), else at F[i][y] (the value
//   bounced back / reconstructed at y itself).
// Odd step (S -> N): gather f(y, .) by that rule, collide, store h_i(y) where
//   the push step would (F[i][y + c_i]; bounce-back / iolet -> F[inv(i)][y]).
// Every location is read and written by exactly one site per step, so the
// update is in place; the arithmetic is the push step's, so the bits are the
// reference's.  Cut-crossing links read/write the neighbour GPU's buffer
// (peer-mapped) at the location the P2P push would store to.

// Location of f(y, i) in state S, from the table entry of direction inv(i).
template <bool kP2P>
__device__ __forceinline__ const double* aa_src(const double* F, uint64_t P, uint32_t y, int i, uint32_t vinv,
                                                const HaloArgs& h) {
    if (vinv < kSpecial) return F + uint64_t(inv(i)) * P + vinv;
    if (((vinv >> kOpShift) & 3u) == kOpShared) {
        if constexpr (kP2P) {
            const uint32_t slot = vinv & kPayload;
            return h.peer_fn[h.slot_peer[slot]] + h.slot_dst[slot];
        }
    }
    return F + uint64_t(i) * P + y;  // bounce-back / iolet: reconstructed at y
}

// Even step over sites [begin, end): plain sites need no table at all.
template <bool kIolets>
__global__ void __launch_bounds__(256)
lbm_aa_even(double* __restrict__ F, const uint32_t* __restrict__ tab, uint64_t P, uint32_t begin, uint32_t end,
            double omega, IoletArgs ia) {
    const uint32_t s = begin + blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= end) return;
    double f[kQ];
#pragma unroll
    for (int i = 0; i < kQ; ++i) f[i] = F[uint64_t(i) * P + s];
    const Macro m = macro_of(f);
    double feq[kQ];
    feq_all(m.rho, m.ux, m.uy, m.uz, feq);
    F[s] = relax(f[0], feq[0], omega);
#pragma unroll
    for (int i = 1; i < kQ; ++i) {
        double g = relax(f[i], feq[i], omega);
        if constexpr (kIolets) {
            const uint32_t v = tab[uint64_t(i - 1) * P + s];
            if (v >= kSpecial && ((v >> kOpShift) & 3u) == kOpIolet) {
                const uint32_t k = v & kPayload;
                const int32_t* c = ia.coords + 3 * uint64_t(s - begin);
                g = iolet_link_value(i, g, m, ia.io[k], ia.staged[k], c[0], c[1], c[2]);
            }
        }
        F[uint64_t(inv(i)) * P + s] = g;
    }
}

// Even step, plain sites, TMA-staged loads (the bulk kernel): streaming in,
// streaming out, 304 B/site.
template <int T, int S, int kMinBlocks>
__global__ void __launch_bounds__(T, kMinBlocks)
lbm_aa_even_tma(double* __restrict__ F, uint64_t P, uint32_t begin, uint32_t end, double omega,
                unsigned* __restrict__ counter = nullptr) {
    using L = PushTmaSmem<T, S, false>;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + S * L::kStage);
    uint32_t* tidx = reinterpret_cast<uint32_t*>(bar + S);  // dynamic order: tile of each stage
    const uint32_t base = begin & ~3u;
    const uint32_t ntiles = (end - base + T - 1) / T;
    const uint32_t G = gridDim.x;
    const uint32_t tid = threadIdx.x;
    if (tid == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&bar[s], 1);
        mbar_fence_init();
    }
    __syncthreads();
    const uint64_t policy = evict_normal_policy();
    auto issue = [&](uint32_t k) {
        uint32_t tile = blockIdx.x + k * G;
        if (counter) tidx[k % S] = tile = atomicAdd(counter, 1u);
        if (tile >= ntiles) return;
        const int st = int(k % S);
        unsigned char* buf = smem + st * L::kStage;
        const uint64_t t0 = uint64_t(base) + uint64_t(tile) * T;
        mbar_expect_tx(&bar[st], L::kStage);
#pragma unroll 1
        for (int i = 0; i < kQ; ++i) bulk_g2s(buf + i * T * 8, F + uint64_t(i) * P + t0, T * 8, &bar[st], policy);
    };
    if (tid == 0)
        for (uint32_t k = 0; k + 1 < uint32_t(S); ++k) issue(k);
    if (counter) __syncthreads();
    for (uint32_t k = 0;; ++k) {
        const uint32_t tile = counter ? tidx[k % S] : blockIdx.x + k * G;
        if (tile >= ntiles) break;
        if (tid == 0) issue(k + S - 1);
        const int st = int(k % S);
        const uint32_t s = base + tile * T + tid;
        mbar_wait(&bar[st], (k / S) & 1u);
        const double* fs = reinterpret_cast<const double*>(smem + st * L::kStage);
        if (s >= begin && s < end) {
            double f[kQ];
#pragma unroll
            for (int i = 0; i < kQ; ++i) f[i] = fs[i * T + tid];
            const Macro m = macro_of(f);
            double feq[kQ];
            feq_all(m.rho, m.ux, m.uy, m.uz, feq);
#pragma unroll
            for (int i = 0; i < kQ; ++i) F[uint64_t(inv(i)) * P + s] = relax(f[i], feq[i], omega);
        }
        __syncthreads();
    }
}

// Odd step over sites [begin, end): gather by the state-S rule, collide, store
// like the push step.  One thread per site.
template <bool kIolets, bool kP2P, int kThreads, int kMinBlocks>
__global__ void __launch_bounds__(kThreads, kMinBlocks)
lbm_aa_odd(double* __restrict__ F, const uint32_t* __restrict__ tab, uint64_t P, uint32_t begin, uint32_t end,
           double omega, IoletArgs ia, const __grid_constant__ HaloArgs halo) {
    const uint32_t s = begin + blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= end) return;
    uint32_t t[kQ - 1];
#pragma unroll
    for (int i = 0; i < kQ - 1; ++i) t[i] = __ldg(tab + uint64_t(i) * P + s);
    double f[kQ];
    f[0] = F[s];
#pragma unroll
    for (int i = 1; i < kQ; ++i) f[i] = *aa_src<kP2P>(F, P, s, i, t[inv(i) - 1], halo);
    const Macro m = macro_of(f);
    double feq[kQ];
    feq_all(m.rho, m.ux, m.uy, m.uz, feq);
    F[s] = relax(f[0], feq[0], omega);
#pragma unroll
    for (int i = 1; i < kQ; ++i) {
        double fpost = relax(f[i], feq[i], omega);
        const uint32_t v = t[i - 1];
        double* dst;
        if (v < kSpecial) {
            dst = F + uint64_t(i) * P + v;
        } else {
            const uint32_t op = (v >> kOpShift) & 3u;
            if (op == kOpShared) {
                if constexpr (kP2P) {
                    const uint32_t slot = v & kPayload;
                    dst = halo.peer_fn[halo.slot_peer[slot]] + halo.slot_dst[slot];
                } else {
                    dst = F + uint64_t(kQ) * P + (v & kPayload);  // unreachable: AA needs P2P across workers
                }
            } else {
                dst = F + uint64_t(inv(i)) * P + s;
                if constexpr (kIolets) {
                    if (op == kOpIolet) {
                        const uint32_t k = v & kPayload;
                        const int32_t* c = ia.coords + 3 * uint64_t(s - begin);
                        fpost = iolet_link_value(i, fpost, m, ia.io[k], ia.staged[k], c[0], c[1], c[2]);
                    }
                }
            }
        }
        *dst = fpost;
    }
}

// Odd step over the mid-group plain range with the compressed table: a
// persistent CTA streams each tile's int16 deltas and group bases into shared
// memory with bulk async copies (2 stages) while the previous tile gathers,
// collides and scatters; a table entry serves twice (direction inv(i) for the
// gather of f_i, direction i for the store of h_i).
template <int T, int S, int kMinBlocks>
struct AaOddSmem {
    static constexpr uint32_t kD = uint32_t(kQ - 1) * T * 2;          // deltas
    static constexpr uint32_t kB = uint32_t(kQ - 1) * (T / 32) * 4;   // group bases
    static constexpr uint32_t kStage = (kD + kB + 127) / 128 * 128;
    static constexpr uint32_t kBytes = S * kStage + S * 8;
};

template <int T, int S, int kMinBlocks>
__global__ void __launch_bounds__(T, kMinBlocks)
lbm_aa_odd_tmc(double* __restrict__ F, const int16_t* __restrict__ dtab, const uint32_t* __restrict__ gbase,
               const uint32_t* __restrict__ tab, uint64_t P, uint64_t PG, uint32_t begin, uint32_t end, double omega) {
    using L = AaOddSmem<T, S, kMinBlocks>;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + S * L::kStage);
    const uint32_t base = begin & ~127u;  // 16-byte aligned group-base copies (PG is a multiple of 4)
    const uint32_t ntiles = (end - base + T - 1) / T;
    const uint32_t G = gridDim.x;
    const uint32_t tid = threadIdx.x;
    const int lane = int(tid & 31), warp = int(tid >> 5);
    if (tid == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&bar[s], 1);
        mbar_fence_init();
    }
    __syncthreads();
    const uint64_t policy = evict_normal_policy();
    auto issue = [&](uint32_t k) {
        const uint32_t tile = blockIdx.x + k * G;
        if (tile >= ntiles) return;
        const int st = int(k % S);
        unsigned char* buf = smem + st * L::kStage;
        const uint64_t t0 = uint64_t(base) + uint64_t(tile) * T;
        mbar_expect_tx(&bar[st], L::kD + L::kB);
#pragma unroll 1
        for (int i = 0; i < kQ - 1; ++i) {
            bulk_g2s(buf + i * T * 2, dtab + uint64_t(i) * P + t0, T * 2, &bar[st], policy);
            bulk_g2s(buf + L::kD + i * (T / 32) * 4, gbase + uint64_t(i) * PG + (t0 >> 5), (T / 32) * 4, &bar[st],
                     policy);
        }
    };
    if (tid == 0)
        for (uint32_t k = 0; k + 1 < uint32_t(S); ++k) issue(k);
    for (uint32_t k = 0;; ++k) {
        const uint32_t tile = blockIdx.x + k * G;
        if (tile >= ntiles) break;
        if (tid == 0) issue(k + S - 1);
        const int st = int(k % S);
        const uint32_t s = base + tile * T + tid;
        mbar_wait(&bar[st], (k / S) & 1u);
        const int16_t* ds = reinterpret_cast<const int16_t*>(smem + st * L::kStage);
        const uint32_t* bs = reinterpret_cast<const uint32_t*>(smem + st * L::kStage + L::kD);
        if (s >= begin && s < end) {
            // target of direction j (1..18) from the compressed entry
            auto target = [&](int j, uint64_t& addr, bool& special) {
                const int d = ds[(j - 1) * T + tid];
                if (d == kDeltaBounce) {
                    special = true;
                    addr = 0;
                } else if (d == kDeltaEscape) {
                    special = false;
                    addr = tab[uint64_t(j - 1) * P + s];
                } else {
                    special = false;
                    addr = uint32_t(bs[(j - 1) * (T / 32) + warp] + uint32_t(lane) + uint32_t(d));
                }
            };
            double f[kQ];
            f[0] = F[s];
#pragma unroll
            for (int i = 1; i < kQ; ++i) {
                uint64_t a;
                bool sp;
                target(inv(i), a, sp);
                f[i] = sp ? F[uint64_t(i) * P + s] : F[uint64_t(inv(i)) * P + a];
            }
            const Macro m = macro_of(f);
            double feq[kQ];
            feq_all(m.rho, m.ux, m.uy, m.uz, feq);
            F[s] = relax(f[0], feq[0], omega);
#pragma unroll
            for (int i = 1; i < kQ; ++i) {
                uint64_t a;
                bool sp;
                target(i, a, sp);
                F[sp ? uint64_t(inv(i)) * P + s : uint64_t(i) * P + a] = relax(f[i], feq[i], omega);
            }
        }
        __syncthreads();
    }
}

// Odd step, mid-group plain range, compressed table, one thread per site (no
// CTA barrier: gathers of different CTAs overlap freely).  Bases travel by
// warp shuffle; warps cover aligned 32-site groups.
template <int kThreads, int kMinBlocks>
__global__ void __launch_bounds__(kThreads, kMinBlocks)
lbm_aa_odd_c(double* __restrict__ F, const int16_t* __restrict__ dtab, const uint32_t* __restrict__ gbase,
             const uint32_t* __restrict__ tab, uint64_t P, uint64_t PG, uint32_t begin, uint32_t end, double omega) {
    const uint32_t s = (begin & ~31u) + blockIdx.x * kThreads + threadIdx.x;
    const int lane = int(threadIdx.x & 31);
    const bool live = s >= begin && s < end;
    if (__all_sync(0xffffffffu, !live)) return;  // whole warp outside the range
    int d[kQ - 1];
#pragma unroll
    for (int i = 0; i < kQ - 1; ++i) d[i] = live ? int(__ldg(dtab + uint64_t(i) * P + s)) : int(kDeltaBounce);
    const uint32_t breg = lane < kQ - 1 ? __ldg(gbase + uint64_t(lane) * PG + (s >> 5)) : 0u;
    // direction j's target site; bounce-back -> (s, mirrored plane).  Branch-free:
    // the escape is a predicated load, the bounce a select.
    auto target = [&](int j, bool& bb) -> uint32_t {
        const uint32_t b = __shfl_sync(0xffffffffu, breg, j - 1);
        const int dj = d[j - 1];
        uint32_t t = b + uint32_t(lane) + uint32_t(dj);
        const uint32_t esc = (dj == kDeltaEscape) && live;
        asm("{\n .reg .pred p;\n setp.ne.u32 p, %1, 0;\n @p ld.global.nc.u32 %0, [%2];\n}"
            : "+r"(t)
            : "r"(esc), "l"(tab + uint64_t(j - 1) * P + s));
        bb = dj == kDeltaBounce;
        return bb ? s : t;
    };
    double f[kQ];
    f[0] = live ? F[s] : 1.0;
#pragma unroll
    for (int i = 1; i < kQ; ++i) {
        bool bb;
        const uint32_t t = target(inv(i), bb);
        const double* src = (bb ? F + uint64_t(i) * P : F + uint64_t(inv(i)) * P) + t;
        f[i] = live ? *src : 0.0;
    }
    const Macro m = macro_of(f);
    double feq[kQ];
    feq_all(m.rho, m.ux, m.uy, m.uz, feq);
    if (live) F[s] = relax(f[0], feq[0], omega);
#pragma unroll
    for (int i = 1; i < kQ; ++i) {
        bool bb;
        const uint32_t t = target(i, bb);
        double* dst = (bb ? F + uint64_t(inv(i)) * P : F + uint64_t(i) * P) + t;
        if (live) *dst = relax(f[i], feq[i], omega);
    }
}

// Odd step, mid-group plain range: the gathers as asynchronous copies.
// The odd step reads f_inv(i)(y) from the location its push would write h_i
// to, loc_i(y) = (i, target_i(y)) or (inv(i), y) for a bounce-back link, and
// writes h_i(y) back to that same location — scattered loads AND scattered
// stores, latency-bound as a register gather (one tile of gathers per thread
// in flight, 128 registers: ~0.7 of the copy roofline).  Here a persistent
// CTA runs a software pipeline over tiles of T sites:
//   * the compressed table (int16 deltas + u32 group bases) of tile k+2 is
//     streamed into shared memory by the TMA engine (cp.async.bulk, 3 stages);
//   * the 19 gathers of tile k+1 are issued as cp.async (LDGSTS, 8 B each)
//     straight into shared memory — in flight without holding registers;
//   * tile k collides from shared memory and stores its 19 results to the
//     same locations (addresses recomputed from the staged table).
// Every location is owned by one (site, direction), so the in-place update
// needs no ordering between tiles or CTAs; the arithmetic is the push step's.

template <int T>
struct AaAsyncSmem {
    static constexpr uint32_t kF = uint32_t(kQ) * T * 8;                 // gathered f, one tile
    static constexpr uint32_t kD = uint32_t(kQ - 1) * T * 2;             // int16 deltas
    static constexpr uint32_t kB = uint32_t(kQ - 1) * (T / 32) * 4;      // group bases
    static constexpr uint32_t kTab = (kD + kB + 127) / 128 * 128;
    static constexpr int kFS = 2, kTS = 3;                               // f stages, table stages
    static constexpr uint32_t kBytes = kFS * kF + kTS * kTab + kTS * 8;
};

template <int T, int kMinBlocks>
__global__ void __launch_bounds__(T, kMinBlocks)
lbm_aa_odd_async(double* __restrict__ F, const int16_t* __restrict__ dtab, const uint32_t* __restrict__ gbase,
                 const uint32_t* __restrict__ tab, uint64_t P, uint64_t PG, uint32_t begin, uint32_t end, double omega,
                 const __grid_constant__ Planes19 planes) {
    using L = AaAsyncSmem<T>;
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned char* fsm = smem;                       // [kFS][19][T] doubles
    unsigned char* tsm = smem + L::kFS * L::kF;      // [kTS] x (deltas [18][T], bases [18][T/32])
    uint64_t* bar = reinterpret_cast<uint64_t*>(tsm + L::kTS * L::kTab);
    const uint32_t base = begin & ~127u;  // 16-byte aligned group-base copies (PG is a multiple of 4)
    const uint32_t ntiles = (end - base + T - 1) / T;
    const uint32_t G = gridDim.x;
    const uint32_t tid = threadIdx.x;
    const int lane = int(tid & 31), warp = int(tid >> 5);
    if (tid == 0) {
        for (int s = 0; s < L::kTS; ++s) mbar_init(&bar[s], 1);
        mbar_fence_init();
    }
    __syncthreads();
    const uint64_t policy = evict_normal_policy();
    auto issue_table = [&](uint32_t k) {  // thread 0: TMA of tile k's table
        const uint32_t tile = blockIdx.x + k * G;
        if (tile >= ntiles) return;
        const int st = int(k % L::kTS);
        unsigned char* buf = tsm + st * L::kTab;
        const uint64_t t0 = uint64_t(base) + uint64_t(tile) * T;
        mbar_expect_tx(&bar[st], L::kD + L::kB);
#pragma unroll 1
        for (int i = 0; i < kQ - 1; ++i) {
            bulk_g2s(buf + i * T * 2, dtab + uint64_t(i) * P + t0, T * 2, &bar[st], policy);
            bulk_g2s(buf + L::kD + i * (T / 32) * 4, gbase + uint64_t(i) * PG + (t0 >> 5), (T / 32) * 4, &bar[st],
                     policy);
        }
    };
    // location of direction j (1..18) of site s from a staged table (plane
    // bases from the constant bank, branch-free selects; the rare escape is
    // a predicated load of the u32 table)
    auto loc = [&](const unsigned char* tb, int j, uint32_t s) -> double* {
        const int16_t* ds = reinterpret_cast<const int16_t*>(tb);
        const uint32_t* bs = reinterpret_cast<const uint32_t*>(tb + L::kD);
        const int d = ds[(j - 1) * T + tid];
        uint32_t t = bs[(j - 1) * (T / 32) + warp] + uint32_t(lane) + uint32_t(d);
        const uint32_t esc = d == kDeltaEscape;
        t = escape_load(t, esc != 0u, tab + uint64_t(j - 1) * P + s);
        const bool bb = d == kDeltaBounce;
        const uintptr_t pb = reinterpret_cast<uintptr_t>(bb ? planes.p[inv(j)] : planes.p[j]);
        return reinterpret_cast<double*>(pb) + (bb ? s : t);
    };
    // gathers of tile k into f stage k % kFS (own slots only)
    auto issue_gathers = [&](uint32_t k) {
        const uint32_t tile = blockIdx.x + k * G;
        if (tile >= ntiles) return;
        const uint32_t s = base + tile * T + tid;
        if (s < begin || s >= end) return;
        mbar_wait(&bar[k % L::kTS], (k / L::kTS) & 1u);
        const unsigned char* tb = tsm + (k % L::kTS) * L::kTab;
        double* fs = reinterpret_cast<double*>(fsm + (k % L::kFS) * L::kF);
        cp_async8(fs + tid, F + s);
#pragma unroll
        for (int i = 1; i < kQ; ++i) cp_async8(fs + inv(i) * T + tid, loc(tb, i, s));  // f_inv(i)(s)
    };
    if (tid == 0) {
        issue_table(0);
        issue_table(1);
    }
    issue_gathers(0);
    cp_async_commit();
    for (uint32_t k = 0;; ++k) {
        const uint32_t tile = blockIdx.x + k * G;
        if (tile >= ntiles) break;
        issue_gathers(k + 1);
        cp_async_commit();
        if (tid == 0) issue_table(k + 2);  // into the stage tile k - 1 released
        cp_async_wait<1>();                // this thread's gathers of tile k have landed
        const uint32_t s = base + tile * T + tid;
        if (s >= begin && s < end) {
            const unsigned char* tb = tsm + (k % L::kTS) * L::kTab;
            const double* fs = reinterpret_cast<const double*>(fsm + (k % L::kFS) * L::kF);
            double f[kQ];
#pragma unroll
            for (int i = 0; i < kQ; ++i) f[i] = fs[i * T + tid];
            const Macro m = macro_of(f);
            double feq[kQ];
            feq_all(m.rho, m.ux, m.uy, m.uz, feq);
            F[s] = relax(f[0], feq[0], omega);
#pragma unroll
            for (int i = 1; i < kQ; ++i) *loc(tb, i, s) = relax(f[i], feq[i], omega);
        }
        __syncthreads();  // table stage k % kTS and f stage k % kFS are free
    }
    cp_async_wait<0>();
}

// Odd step, mid-group plain range: warp-autonomous software pipeline.  Each
// warp walks its own 32-site tiles (persistent, no CTA barrier): the
// compressed table of tile k+2 is loaded into registers, the 19 gathers of
// tile k+1 are issued as cp.async straight into the warp's shared-memory
// stage (in flight without holding registers), and tile k collides from its
// stage and scatters to the 19 locations computed one iteration earlier
// (kept as signed offsets from each direction's plane).  Every location is
// owned by one (site, direction): the in-place update needs no ordering.
template <int kWarps, int kMinBlocks>
struct AaOddW {
    static constexpr uint32_t kStage = uint32_t(kQ) * 32 * 8;  // one warp's gathered f
    static constexpr uint32_t kBytes = 2 * kWarps * kStage;
};

template <int kWarps, int kMinBlocks, int kOpt = 1>
__global__ void __launch_bounds__(kWarps * 32, kMinBlocks)
lbm_aa_odd_w(double* __restrict__ F, const int16_t* __restrict__ dtab, const uint32_t* __restrict__ gbase,
             const uint32_t* __restrict__ tab, uint64_t P, uint64_t PG, uint32_t begin, uint32_t end, double omega,
             const __grid_constant__ Planes19 planes, unsigned* __restrict__ counter = nullptr) {
    using L = AaOddW<kWarps, kMinBlocks>;
    extern __shared__ __align__(128) unsigned char smem[];
    const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    double* stage[2] = {reinterpret_cast<double*>(smem + (2 * wib) * L::kStage),
                        reinterpret_cast<double*>(smem + (2 * wib + 1) * L::kStage)};
    const uint32_t base = begin & ~31u;
    const uint32_t ntiles = (end - base + 31) / 32;
    const uint32_t nw = gridDim.x * kWarps;
    const uint32_t w0 = blockIdx.x * kWarps + wib;
    // warp-tile sequence: the fixed stride w0 + k * nw, or (counter) batches
    // of 4 consecutive tiles taken from a global counter (dynamic order: the
    // tiles in flight stay near the frontier however the warps drift apart)
    // (kOpt & 2: lane 0 requests the next batch as soon as it starts one, so
    // the atomic's round trip is off the critical path; the last batch
    // requested lies past the end like the one that stops the warp)
    constexpr uint32_t kBatch = (kOpt & 4) ? 8 : 4;
    constexpr bool kAtomAhead = (kOpt & 2) != 0, kRaw = (kOpt & 1) != 0;
    uint32_t bb0 = 0, bb1 = 0, bi0 = 0xffffffffu, bi1 = 0xffffffffu;
    uint32_t ahead = 0;
    bool have_ahead = false;
    auto grab = [&]() -> uint32_t {
        uint32_t v = 0;
        if (lane == 0) v = atomicAdd(counter, kBatch);
        return v;
    };
    auto tile_at = [&](uint32_t k) -> uint32_t {
        if (!counter) return w0 + k * nw;
        const uint32_t bi = k / kBatch;
        const bool odd = bi & 1u;
        if ((odd ? bi1 : bi0) != bi) {
            uint32_t v;
            if constexpr (kAtomAhead) {
                if (!have_ahead) ahead = grab();
                v = __shfl_sync(0xffffffffu, ahead, 0);
                ahead = grab();
                have_ahead = true;
            } else {
                v = __shfl_sync(0xffffffffu, grab(), 0);
            }
            if (odd) bb1 = v, bi1 = bi;
            else bb0 = v, bi0 = bi;
        }
        return (odd ? bb1 : bb0) + k % kBatch;
    };
    // compressed table of warp-tile k into registers: the 18 int16 deltas
    // (kOpt & 1: one per register, loaded by predicated loads that nothing
    // consumes before the next iteration; else packed two per register — the
    // packing waits for the loads, a full memory latency per tile) and this
    // lane's group base
    constexpr int kD2 = kRaw ? kQ - 1 : (kQ - 1) / 2;
    uint32_t dA[kD2], dB[kD2];
    uint32_t bA = 0, bB = 0;
    auto load_table = [&](uint32_t k, uint32_t* d, uint32_t& b) {
        const uint32_t tile = tile_at(k);
        const uint32_t s = base + tile * 32 + lane;
        const bool live = tile < ntiles && s >= begin && s < end;
        if constexpr (kRaw) {
#pragma unroll
            for (int i = 0; i < kD2; ++i) {
                uint32_t v = uint32_t(int(kDeltaBounce));
                asm("{\n .reg .pred p;\n setp.ne.u32 p, %1, 0;\n @p ld.global.nc.s16 %0, [%2];\n}"
                    : "+r"(v)
                    : "r"(uint32_t(live)), "l"(dtab + uint64_t(i) * P + s));
                d[i] = v;
            }
            uint32_t g = 0;
            asm("{\n .reg .pred p;\n setp.ne.u32 p, %1, 0;\n @p ld.global.nc.u32 %0, [%2];\n}"
                : "+r"(g)
                : "r"(uint32_t(lane < kQ - 1 && tile < ntiles)), "l"(gbase + uint64_t(lane) * PG + (s >> 5)));
            b = g;
        } else {
#pragma unroll
            for (int i = 0; i < kD2; ++i) {
                const uint32_t lo = live ? uint16_t(__ldg(dtab + uint64_t(2 * i) * P + s)) : uint16_t(kDeltaBounce);
                const uint32_t hi = live ? uint16_t(__ldg(dtab + uint64_t(2 * i + 1) * P + s)) : uint16_t(kDeltaBounce);
                d[i] = lo | (hi << 16);
            }
            b = (lane < kQ - 1 && tile < ntiles) ? __ldg(gbase + uint64_t(lane) * PG + (s >> 5)) : 0u;
        }
    };
    // location of direction j of site s: signed offset from plane j's base
    // (a bounce-back lives in the inverse plane at s: s +- P)
    auto loc = [&](const uint32_t* d, uint32_t b, int j, uint32_t s, bool live) -> int32_t {
        const uint32_t bj = __shfl_sync(0xffffffffu, b, j - 1);
        const int dj = kRaw ? int(d[j - 1])
                            : (j & 1) ? int(int16_t(d[(j - 1) / 2] & 0xffffu)) : int(int16_t(d[(j - 1) / 2] >> 16));
        uint32_t t = bj + lane + uint32_t(dj);
        const uint32_t esc = (dj == kDeltaEscape) && live;
        asm("{\n .reg .pred p;\n setp.ne.u32 p, %1, 0;\n @p ld.global.nc.u32 %0, [%2];\n}"
            : "+r"(t)
            : "r"(esc), "l"(tab + uint64_t(j - 1) * P + s));
        const int32_t off = (j & 1) ? int32_t(P) : -int32_t(P);
        return dj == kDeltaBounce ? int32_t(s) + off : int32_t(t);
    };
    int32_t oA[kQ - 1], oB[kQ - 1];  // locations of the tile being stored / being gathered
    // issue the gathers of tile k (table d, b) into stage k & 1; offsets into o
    auto issue = [&](uint32_t k, const uint32_t* d, uint32_t b, int32_t* o) {
        const uint32_t tile = tile_at(k);
        const uint32_t s = base + tile * 32 + lane;
        const bool live = tile < ntiles && s >= begin && s < end;
        double* st = stage[k & 1];
#pragma unroll
        for (int i = 1; i < kQ; ++i) o[i - 1] = loc(d, b, i, s, live);
        if (live) {
            cp_async8(st + lane, F + s);
#pragma unroll
            for (int i = 1; i < kQ; ++i) cp_async8(st + inv(i) * 32 + lane, planes.p[i] + o[i - 1]);  // f_inv(i)(s)
        }
    };
    // iteration k: gathers of tile k+1 (its table in dN), table of tile k+2
    // into dNN, then tile k collides from its stage and stores through oK;
    // two iterations per loop trip swap the register sets without moves
    auto step = [&](uint32_t k, const uint32_t* dN, uint32_t bN, int32_t* oN, uint32_t* dNN, uint32_t& bNN,
                    const int32_t* oK) -> bool {
        const uint32_t tile = tile_at(k);
        if (tile >= ntiles) return false;
        issue(k + 1, dN, bN, oN);
        cp_async_commit();
        load_table(k + 2, dNN, bNN);
        cp_async_wait<1>();  // this lane's gathers of tile k have landed
        const uint32_t s = base + tile * 32 + lane;
        const double* st = stage[k & 1];
        double f[kQ];
#pragma unroll
        for (int i = 0; i < kQ; ++i) f[i] = st[i * 32 + lane];
        const Macro m = macro_of(f);
        double feq[kQ];
        feq_all(m.rho, m.ux, m.uy, m.uz, feq);
        if (s >= begin && s < end) {
            F[s] = relax(f[0], feq[0], omega);
#pragma unroll
            for (int i = 1; i < kQ; ++i) planes.p[i][oK[i - 1]] = relax(f[i], feq[i], omega);
        }
        __syncwarp();  // the stage of tile k is refilled by tile k+2's gathers
        return true;
    };
    load_table(0, dA, bA);
    if (tile_at(0) >= ntiles) return;  // whole warp
    issue(0, dA, bA, oA);
    cp_async_commit();
    load_table(1, dB, bB);
    for (uint32_t k = 0;; k += 2) {
        if (!step(k, dB, bB, oB, dA, bA, oA)) break;
        if (!step(k + 1, dA, bA, oA, dB, bB, oB)) break;
    }
    cp_async_wait<0>();
}

#ifdef SPLBCU_TUNING
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}

// Odd step, the same warp-autonomous pipeline with the compressed table
// staged in shared memory instead of registers: the table of tile k+3 is
// copied (cp.async, 72 x 16 B of deltas + 18 group bases) with the gathers of
// tile k+1, and the 18 locations are decoded from it twice — when tile k+1's
// gathers are issued and when tile k stores — instead of being held.  That
// frees the ~56 registers the register version spends on two table sets and
// two offset sets, for more resident warps (more gathers in flight per SM).
// Measured slower (the decode's shared-memory reads stall the MIO pipe,
// profiles/r02_c3_dev_aa_s.md): tuning build only.
template <int kWarps, int kMinBlocks>
struct AaOddS {
    static constexpr uint32_t kF = uint32_t(kQ) * 32 * 8;               // one warp's gathered f
    static constexpr uint32_t kTD = uint32_t(kQ - 1) * 32 * 2;          // deltas of one tile
    static constexpr uint32_t kT = kTD + 128;                          // + its 18 group bases
    static constexpr uint32_t kWarpBytes = 2 * kF + 4 * kT;
    static constexpr uint32_t kBytes = kWarps * kWarpBytes;
};

template <int kWarps, int kMinBlocks>
__global__ void __launch_bounds__(kWarps * 32, kMinBlocks)
lbm_aa_odd_s(double* __restrict__ F, const int16_t* __restrict__ dtab, const uint32_t* __restrict__ gbase,
             const uint32_t* __restrict__ tab, uint64_t P, uint64_t PG, uint32_t begin, uint32_t end, double omega,
             const __grid_constant__ Planes19 planes, unsigned* __restrict__ counter = nullptr) {
    using L = AaOddS<kWarps, kMinBlocks>;
    extern __shared__ __align__(128) unsigned char smem[];
    const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    unsigned char* const wsm = smem + wib * L::kWarpBytes;
    const uint32_t base = begin & ~31u;  // P is a multiple of 64: whole tiles lie inside the planes
    const uint32_t ntiles = (end - base + 31) / 32;
    const uint32_t nw = gridDim.x * kWarps;
    const uint32_t w0 = blockIdx.x * kWarps + wib;
    constexpr uint32_t kBatch = 4;  // as lbm_aa_odd_w; the look-ahead (3 tiles) spans <= 2 batches
    uint32_t bb0 = 0, bb1 = 0, bi0 = 0xffffffffu, bi1 = 0xffffffffu;
    auto tile_at = [&](uint32_t k) -> uint32_t {
        if (!counter) return w0 + k * nw;
        const uint32_t bi = k / kBatch;
        const bool odd = bi & 1u;
        if ((odd ? bi1 : bi0) != bi) {
            uint32_t v = 0;
            if (lane == 0) v = atomicAdd(counter, kBatch);
            v = __shfl_sync(0xffffffffu, v, 0);
            if (odd) bb1 = v, bi1 = bi;
            else bb0 = v, bi0 = bi;
        }
        return (odd ? bb1 : bb0) + k % kBatch;
    };
    auto fst = [&](uint32_t k) { return reinterpret_cast<double*>(wsm + (k & 1) * L::kF); };
    auto tst = [&](uint32_t k) { return wsm + 2 * L::kF + (k & 3) * L::kT; };
    auto load_table = [&](uint32_t k) {
        const uint32_t tile = tile_at(k);
        if (tile >= ntiles) return;
        const uint32_t tb = base + tile * 32;
        unsigned char* t = tst(k);
#pragma unroll
        for (uint32_t c = lane; c < 4 * (kQ - 1); c += 32)  // row c / 4, 16-byte quarter c % 4
            cp_async16(t + c * 16, dtab + uint64_t(c >> 2) * P + tb + (c & 3) * 8);
        if (lane < kQ - 1) cp_async4(t + L::kTD + lane * 4, gbase + uint64_t(lane) * PG + (tb >> 5));
    };
    // location of direction j of site s (tile k's table): signed offset from
    // plane j's base (a bounce-back lives in the inverse plane at s: s +- P)
    auto loc = [&](uint32_t k, int j, uint32_t s, bool live) -> int32_t {
        const unsigned char* t = tst(k);
        const int dj = reinterpret_cast<const int16_t*>(t)[(j - 1) * 32 + lane];
        const uint32_t bj = reinterpret_cast<const uint32_t*>(t + L::kTD)[j - 1];
        uint32_t tg = bj + lane + uint32_t(dj);
        const uint32_t esc = (dj == kDeltaEscape) && live;
        asm("{\n .reg .pred p;\n setp.ne.u32 p, %1, 0;\n @p ld.global.nc.u32 %0, [%2];\n}"
            : "+r"(tg)
            : "r"(esc), "l"(tab + uint64_t(j - 1) * P + s));
        const int32_t off = (j & 1) ? int32_t(P) : -int32_t(P);
        return dj == kDeltaBounce ? int32_t(s) + off : int32_t(tg);
    };
    auto issue = [&](uint32_t k) {
        const uint32_t tile = tile_at(k);
        const uint32_t s = base + tile * 32 + lane;
        const bool live = tile < ntiles && s >= begin && s < end;
        if (!live) return;
        double* st = fst(k);
        cp_async8(st + lane, F + s);
#pragma unroll
        for (int i = 1; i < kQ; ++i) cp_async8(st + inv(i) * 32 + lane, planes.p[i] + loc(k, i, s, true));
    };
    load_table(0);
    load_table(1);
    cp_async_commit();
    cp_async_wait<0>();
    __syncwarp();
    if (tile_at(0) >= ntiles) return;  // whole warp
    issue(0);
    load_table(2);
    cp_async_commit();
    for (uint32_t k = 0;; ++k) {
        const uint32_t tile = tile_at(k);
        if (tile >= ntiles) break;
        issue(k + 1);       // table k+1 landed with tile k-1's gathers
        load_table(k + 3);  // its stage held table k-1, done
        cp_async_commit();
        cp_async_wait<1>();  // tile k's gathers and table k+2 have landed
        __syncwarp();        // ... for every lane (table rows are copied by other lanes)
        const uint32_t s = base + tile * 32 + lane;
        const double* st = fst(k);
        double f[kQ];
#pragma unroll
        for (int i = 0; i < kQ; ++i) f[i] = st[i * 32 + lane];
        const Macro m = macro_of(f);
        double feq[kQ];
        feq_all(m.rho, m.ux, m.uy, m.uz, feq);
        if (s >= begin && s < end) {
            F[s] = relax(f[0], feq[0], omega);
#pragma unroll
            for (int i = 1; i < kQ; ++i) planes.p[i][loc(k, i, s, true)] = relax(f[i], feq[i], omega);
        }
        __syncwarp();  // f stage k & 1 and table stage k & 3 are refilled next
    }
    cp_async_wait<0>();
}
#endif  // SPLBCU_TUNING

// Gather the 19 populations of site s in the current AA state (state N:
// plain reads; state S: the rule above).
template <bool kP2P>
__device__ __forceinline__ void aa_gather(const double* F, const uint32_t* tab, uint64_t P, uint32_t s, bool state_s,
                                          const HaloArgs& h, double f[kQ]) {
    if (!state_s) {
#pragma unroll
        for (int i = 0; i < kQ; ++i) f[i] = F[uint64_t(i) * P + s];
        return;
    }
    f[0] = F[s];
#pragma unroll
    for (int i = 1; i < kQ; ++i) f[i] = *aa_src<kP2P>(F, P, s, i, tab[uint64_t(inv(i) - 1) * P + s], h);
}

template <bool kP2P>
__global__ void lbm_aa_capture(const double* __restrict__ F, const uint32_t* __restrict__ tab, uint64_t P,
                               uint32_t n, int state_s, const __grid_constant__ HaloArgs h, double* __restrict__ out4) {
    const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n) return;
    double fl[kQ];
    aa_gather<kP2P>(F, tab, P, s, state_s != 0, h, fl);
    const Macro m = macro_of(fl);
    double* o = out4 + 4 * uint64_t(s);
    o[0] = m.rho;
    o[1] = m.ux;
    o[2] = m.uy;
    o[3] = m.uz;
}

// f in the reference's meaning for every (site, direction): 19 planes of n.
template <bool kP2P>
__global__ void lbm_aa_export(const double* __restrict__ F, const uint32_t* __restrict__ tab, uint64_t P, uint32_t n,
                              int state_s, const __grid_constant__ HaloArgs h, double* __restrict__ out) {
    const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n) return;
    double fl[kQ];
    aa_gather<kP2P>(F, tab, P, s, state_s != 0, h, fl);
#pragma unroll
    for (int i = 0; i < kQ; ++i) out[uint64_t(i) * P + s] = fl[i];
}

// Inverse of lbm_aa_export: scatter f(s, i) to its location in the current
// state (own sites only; a cut-crossing source lives on the neighbour).
__global__ void lbm_aa_import(double* __restrict__ F, const uint32_t* __restrict__ tab, uint64_t P, uint32_t n,
                              int state_s, const double* __restrict__ in) {
    const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n) return;
    if (!state_s) {
        for (int i = 0; i < kQ; ++i) F[uint64_t(i) * P + s] = in[uint64_t(i) * P + s];
        return;
    }
    F[s] = in[s];
    for (int i = 1; i < kQ; ++i) {
        const uint32_t vinv = tab[uint64_t(inv(i) - 1) * P + s];
        if (vinv < kSpecial) F[uint64_t(inv(i)) * P + vinv] = in[uint64_t(i) * P + s];
        else if (((vinv >> kOpShift) & 3u) != kOpShared) F[uint64_t(i) * P + s] = in[uint64_t(i) * P + s];
    }
}

template <bool kP2P>
__global__ void lbm_aa_observe(const double* __restrict__ F, const uint32_t* __restrict__ tab, uint64_t P,
                               uint32_t n_obs, int state_s, const __grid_constant__ HaloArgs h, const uint32_t* __restrict__ obs_site,
                               const uint16_t* __restrict__ obs_iolet, const IoletDev* __restrict__ io,
                               double* __restrict__ out_row) {
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n_obs) return;
    const uint32_t s = obs_site[j];
    double fl[kQ];
    aa_gather<kP2P>(F, tab, P, s, state_s != 0, h, fl);
    const Macro m = macro_of(fl);
    const IoletDev& g = io[obs_iolet[j]];
    double* o = out_row + 3 * uint64_t(j);
    o[0] = sqrt((m.ux * m.ux + m.uy * m.uy) + m.uz * m.uz);
    o[1] = kCs2 * m.rho;
    o[2] = (m.ux * g.normal[0] + m.uy * g.normal[1]) + m.uz * g.normal[2];
}

// PostReceive re-allocation (engine.hpp:534-542): fn[recv_dest[k]] = fo[tail + k].
__global__ void lbm_post_receive(const double* __restrict__ fo_tail, double* __restrict__ fn,
                                 const uint64_t* __restrict__ recv_flat, uint32_t n) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n) fn[recv_flat[k]] = fo_tail[k];
}

// f_old = equilibrium(rho0, 0) (engine.hpp:254-259); eq computed on the host.
struct Eq19 {
    double v[kQ];
};
__global__ void lbm_init_equilibrium(double* __restrict__ f, uint64_t P, uint32_t n, Eq19 eq) {
    const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n) return;
#pragma unroll
    for (int i = 0; i < kQ; ++i) f[uint64_t(i) * P + s] = eq.v[i];
}

// Moments of every site (fields_of_worker, engine.hpp:583-597), internal order.
__global__ void lbm_capture_moments(const double* __restrict__ f, uint64_t P, uint32_t n,
                                    double* __restrict__ out4) {
    const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n) return;
    double fl[kQ];
#pragma unroll
    for (int i = 0; i < kQ; ++i) fl[i] = f[uint64_t(i) * P + s];
    const Macro m = macro_of(fl);
    double* o = out4 + 4 * uint64_t(s);
    o[0] = m.rho;
    o[1] = m.ux;
    o[2] = m.uy;
    o[3] = m.uz;
}

// Per iolet boundary site: |u|, cs2*rho, u.n (record_observation,
// engine.hpp:557-581).  One row of n_obs triples.
__global__ void lbm_iolet_observe(const double* __restrict__ f, uint64_t P, uint32_t n_obs,
                                  const uint32_t* __restrict__ obs_site,
                                  const uint16_t* __restrict__ obs_iolet,
                                  const IoletDev* __restrict__ io, double* __restrict__ out_row) {
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n_obs) return;
    const uint32_t s = obs_site[j];
    double fl[kQ];
#pragma unroll
    for (int i = 0; i < kQ; ++i) fl[i] = f[uint64_t(i) * P + s];
    const Macro m = macro_of(fl);
    const IoletDev& g = io[obs_iolet[j]];
    double* o = out_row + 3 * uint64_t(j);
    o[0] = sqrt((m.ux * m.ux + m.uy * m.uy) + m.uz * m.uz);
    o[1] = kCs2 * m.rho;
    o[2] = (m.ux * g.normal[0] + m.uy * g.normal[1]) + m.uz * g.normal[2];
}

// ---- iolet series on the device (assemble_series, engine.hpp:602-629) ------
// Observation rows of every worker (worker w's rows at src + per*w, each row
// tot[w] entries of 3 doubles) are first gathered into iolet-major order
// (entry j of the CSR ent_* lists, ascending global site per iolet), then one
// warp per (iolet, row) runs the reference's sequential reduction.
__global__ void series_gather(const double* __restrict__ src, uint64_t per, const uint32_t* __restrict__ tot,
                              const uint16_t* __restrict__ ent_w, const uint32_t* __restrict__ ent_idx,
                              uint32_t n_ent, uint32_t rows, double* __restrict__ dst) {
    const uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= uint64_t(n_ent) * rows) return;
    const uint32_t j = uint32_t(t % n_ent), r = uint32_t(t / n_ent);
    const uint32_t w = ent_w[j];
    const double* v = src + per * w + 3 * (uint64_t(r) * tot[w] + ent_idx[j]);
    double* o = dst + 3 * t;
    o[0] = v[0];
    o[1] = v[1];
    o[2] = v[2];
}

// Sequential in entry order, as the host loop: vmax = std::max(vmax, v0),
// psum += v1, qsum += v2; then (vmax, psum / n, qsum).  One warp per
// (iolet, row), launched as 32-thread blocks.  The lanes stage chunks of
// kChunk entries in shared memory, loading the next chunk into registers
// while every lane runs the same ordered add chain over the current one with
// broadcast reads, so the sums are bit-identical to the host's.  The max is
// order-free: (v < x) ? x : v from +0.0 keeps the first of equal values and
// skips NaN, so each lane folds its own entries and the lanes are folded.
__global__ void __launch_bounds__(32) series_chain(const double* __restrict__ g, const uint32_t* __restrict__ kdev,
                                                   const uint32_t* __restrict__ ent_be, uint32_t n_dev, uint32_t n_io,
                                                   uint32_t rows, uint32_t n_ent, double* __restrict__ out) {
    constexpr int kPer = 8, kChunk = 32 * kPer;  // a chunk's chain (~kChunk DADD latencies) covers a load
    __shared__ double c1[kChunk], c2[kChunk];
    const uint32_t warp = blockIdx.x;
    const int lane = threadIdx.x;
    if (warp >= n_dev * rows) return;
    const uint32_t k = kdev[warp % n_dev], r = warp / n_dev;
    const uint32_t b = ent_be[2 * k], e = ent_be[2 * k + 1];
    const double* base = g + 3 * (uint64_t(r) * n_ent);
    double vmax = 0.0, psum = 0.0, qsum = 0.0;
    double a0[kPer], a1[kPer], a2[kPer];
    auto load = [&](uint32_t c) {
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
            const uint32_t x = c + uint32_t(u * 32 + lane);
            if (x < e) {
                const double* v = base + 3 * uint64_t(x);
                a0[u] = v[0], a1[u] = v[1], a2[u] = v[2];
            } else {
                a0[u] = 0.0, a1[u] = 0.0, a2[u] = 0.0;
            }
        }
    };
    load(b);
    for (uint32_t c = b; c < e; c += kChunk) {
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
            vmax = (vmax < a0[u]) ? a0[u] : vmax;
            c1[u * 32 + lane] = a1[u];
            c2[u * 32 + lane] = a2[u];
        }
        __syncwarp();
        load(c + kChunk);
        if (e - c >= uint32_t(kChunk)) {
#pragma unroll 32
            for (int l = 0; l < kChunk; ++l) {
                psum += c1[l];
                qsum += c2[l];
            }
        } else {
            for (uint32_t l = 0; l < e - c; ++l) {
                psum += c1[l];
                qsum += c2[l];
            }
        }
        __syncwarp();
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double x = __shfl_xor_sync(0xffffffffu, vmax, o);
        vmax = (vmax < x) ? x : vmax;
    }
    if (lane == 0) {
        double* o = out + 3 * (uint64_t(r) * n_io + k);
        o[0] = vmax;
        o[1] = psum / double(e - b);
        o[2] = qsum;
    }
}

#endif  // __CUDACC__

}  // namespace splbcu
