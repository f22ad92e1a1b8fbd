/*
 * splbcu.h — C-ABI of the B200-native sparse D3Q19 LBM engine.
 *
 * This is the drop-in boundary for the reference's hot path.  The reference
 * (`splb`, /root/reference/proj/include/splb) has no FFI: its boundary is the
 * header-only C++ class `splb::Simulation` (engine.hpp:121-205) plus the
 * domain builders it consumes (geometry.hpp:64-363) and the decomposition it
 * exposes to tests (decomp.hpp:16-188).  Each entry point below names the
 * reference interface it replaces.  Plain pointers and sizes only; no torch or
 * CUDA types.  `include/splbcu.hpp` rebuilds the reference's C++ class surface
 * on top of these calls (same names, same exception types).
 *
 * Conventions
 *  - Every function that can fail returns an int status (SPLBCU_OK = 0).  The
 *    message of the last failure on the calling thread is returned by
 *    splbcu_last_error(); the C++ wrapper rethrows it as the matching
 *    splb:: exception type (common.hpp:11-28 of the reference).
 *  - Arrays passed in are borrowed for the duration of the call; handles own
 *    everything they allocate (host and device).
 *  - Indices: global site indices are u32 (the reference's CrossLink/
 *    PartitionAssignment width, layout.hpp:335-339, decomp.hpp:18).
 *  - Handles are not re-entrant (the reference's Simulation is not either).
 */
#ifndef SPLBCU_H
#define SPLBCU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (map to the reference exception taxonomy) ------------ */
enum {
    SPLBCU_OK = 0,
    SPLBCU_ERR_CONFIG = 1,     /* splb::ConfigError   (common.hpp:22-24)     */
    SPLBCU_ERR_RUNTIME = 2,    /* splb::Error         (common.hpp:11-13)     */
    SPLBCU_ERR_COMM = 3,       /* splb::Error "exchange failure: ..."        */
    SPLBCU_ERR_GEOMETRY = 4,   /* splb::GeometryError (common.hpp:17-19)     */
    SPLBCU_ERR_DEGENERATE = 5, /* splb::DegenerateState (common.hpp:14-16)   */
    SPLBCU_ERR_CUDA = 6        /* CUDA/NCCL failure (reported as splb::Error) */
};

/* enums mirrored from the reference, same numeric values */
enum { SPLBCU_LINK_FLUID = 0, SPLBCU_LINK_WALL = 1, SPLBCU_LINK_INLET = 2,
       SPLBCU_LINK_OUTLET = 3 };                          /* geometry.hpp:14 */
enum { SPLBCU_TYPE_INNER = 0, SPLBCU_TYPE_WALL = 1, SPLBCU_TYPE_INLET = 2,
       SPLBCU_TYPE_OUTLET = 3, SPLBCU_TYPE_INLET_WALL = 4,
       SPLBCU_TYPE_OUTLET_WALL = 5 };                     /* geometry.hpp:26 */
enum { SPLBCU_IOLET_INLET = 0, SPLBCU_IOLET_OUTLET = 1 }; /* geometry.hpp:45 */
enum { SPLBCU_LAYOUT_AOS = 0, SPLBCU_LAYOUT_SOA = 1 };    /* layout.hpp:12   */
enum { SPLBCU_SCHEME_PUSH = 0, SPLBCU_SCHEME_PULL = 1 };  /* engine.hpp:23   */
enum { SPLBCU_SEQ_CLASSIC = 0, SPLBCU_SEQ_REORDERED = 1 };/* engine.hpp:27   */
enum { SPLBCU_BC_PRESSURE = 0, SPLBCU_BC_VELOCITY = 1 };  /* engine.hpp:38   */
enum { SPLBCU_OP_TO_LOCAL = 0, SPLBCU_OP_TO_SHARED = 1, SPLBCU_OP_BOUNCE_BACK = 2,
       SPLBCU_OP_IOLET = 3 };                             /* layout.hpp:84   */

/* Iolet geometry (geometry.hpp:44-52). */
typedef struct splbcu_iolet {
    int32_t kind;      /* SPLBCU_IOLET_* */
    double center[3];  /* grid units */
    double normal[3];  /* unit, points into the fluid */
    double radius;
} splbcu_iolet;

/* One boundary condition entry (engine.hpp:37-44 BCSet::Entry + the
 * boundary.hpp:18-74 TimeTable it carries). */
typedef struct splbcu_bc {
    int32_t kind;          /* SPLBCU_BC_* */
    const double* times;   /* n_nodes ascending node times */
    const double* values;  /* n_nodes node values */
    uint32_t n_nodes;
    double period;         /* 0 = aperiodic (clamp) */
} splbcu_bc;

/* EngineParams (engine.hpp:46-57) plus the B200 placement fields. */
typedef struct splbcu_params {
    double tau;
    double rho0;
    double dt_s;
    int32_t layout;             /* layout of host-visible stores/maps (AoS/SoA) */
    int32_t scheme;             /* 0 push (update_push), 1 pull (update_pull +
                                   fill_send_slots, engine.hpp:435-502; bitwise
                                   identical to push, engine.hpp:20-22).  With
                                   storage = 1 the AA scheme runs either way. */
    int32_t sequence;           /* classic/reordered exchange order */
    int32_t workers;            /* logical workers (slabs) */
    uint64_t capture_period;    /* 0 disables field captures */
    int32_t observe_iolets;     /* per-step iolet time series */
    double exchange_timeout_s;  /* engine.hpp:92-101: a run fails when no step
                                   completes for this long (dead or stuck
                                   neighbour, one process per GPU) */
    /* B200 extension: devices the workers are placed on, round robin.
     * n_devices == 0 means {current device}. */
    int32_t n_devices;
    const int32_t* device_ids;
    /* B200 extension: halo exchange between workers.  0 = NCCL send/recv of
     * the shared tail (one process per GPU) or peer copies (in-process), then
     * PostReceive; 1 = fused NVLink P2P: the edge kernels store cut-crossing
     * links straight into the neighbour's f_new (§8f.4 of SURVEY.md). */
    int32_t halo_mode;
    /* B200 extension: distribution storage.  0 = two buffers, push step
     * (f_old -> f_new, reference layout.hpp:19-62); 1 = one buffer updated in
     * place with the AA pattern (even steps local, odd steps gather/scatter;
     * §8f.3): half the HBM, identical bits. */
    int32_t storage;
} splbcu_params;

typedef struct splbcu_domain splbcu_domain;       /* splb::SparseDomain */
typedef struct splbcu_partition splbcu_partition; /* splb::PartitionAssignment */
typedef struct splbcu_sim splbcu_sim;             /* splb::Simulation */

/* ---- errors / build info -------------------------------------------------- */
const char* splbcu_last_error(void);
const char* splbcu_version(void);
void splbcu_params_default(splbcu_params* p); /* engine.hpp:46-57 defaults */

/* ---- lattice known-answer helpers (lattice.hpp:151-191, boundary.hpp:38-132);
 *      host arithmetic identical to the device kernels' expression order. -- */
void splbcu_equilibrium(double rho, const double u[3], double out19[19]);
int splbcu_moments(const double f19[19], double* rho, double u[3]);
int splbcu_bgk_collide(const double f19[19], double tau, double out19[19]);
int splbcu_timetable_at(const double* times, const double* values, uint32_t n,
                        double period, double t, double* out);
double splbcu_iolet_weight(const splbcu_iolet* io, const int32_t coords[3]);

/* ---- domain (geometry.hpp) ------------------------------------------------ */
/* classify_sites (geometry.hpp:139-208): raw voxels (3*n int32, any order) →
 * classified, type-major (z,y,x)-sorted domain. */
int splbcu_domain_classify(const int32_t* voxels, uint64_t n_voxels,
                           const splbcu_iolet* iolets, uint32_t n_iolets,
                           double voxel_size, splbcu_domain** out);
/* build_pipe (geometry.hpp:285-308). */
int splbcu_domain_build_pipe(int32_t radius, int32_t length, double voxel_size,
                             splbcu_domain** out);
/* build_bifurcation (geometry.hpp:313-363). */
int splbcu_domain_build_bifurcation(int32_t trunk_radius, int32_t branch_radius,
                                    int32_t trunk_length, int32_t branch_length,
                                    double voxel_size, splbcu_domain** out);
/* New generators for the scaling configs (no reference equivalent; both
 * produce domains that pass validate_domain): a recursive bifurcating vessel
 * tree (C3) and a dense rectangular channel with disc iolets (C4). */
int splbcu_domain_build_tree(int32_t root_radius, int32_t root_length,
                             int32_t levels, double radius_ratio,
                             double length_ratio, double voxel_size,
                             splbcu_domain** out);
int splbcu_domain_build_channel(int32_t nx, int32_t ny, int32_t nz,
                                double voxel_size, splbcu_domain** out);
/* A SparseDomain given field by field (geometry.hpp:64-73); validated with
 * validate_domain (geometry.hpp:212-271).  link_kind/link_iolet are 18*n,
 * links[i-1] of site s at [18*s + i-1]. type_ranges = 6 (begin,end) pairs. */
int splbcu_domain_from_arrays(uint64_t n_sites, const int32_t* coords,
                              const uint8_t* types, const uint8_t* link_kind,
                              const uint16_t* link_iolet,
                              const splbcu_iolet* iolets, uint32_t n_iolets,
                              const uint64_t* type_ranges, double voxel_size,
                              splbcu_domain** out);
int splbcu_domain_validate(const splbcu_domain* d);
/* SPLB v1 geometry file (geometry_io.hpp:44-129). */
int splbcu_domain_read(const char* path, splbcu_domain** out);
int splbcu_domain_write(const splbcu_domain* d, const char* path);
uint64_t splbcu_domain_n_sites(const splbcu_domain* d);
uint32_t splbcu_domain_n_iolets(const splbcu_domain* d);
double splbcu_domain_voxel_size(const splbcu_domain* d);
/* Copies out the domain; any output pointer may be NULL. */
int splbcu_domain_export(const splbcu_domain* d, int32_t* coords, uint8_t* types,
                         uint8_t* link_kind, uint16_t* link_iolet,
                         splbcu_iolet* iolets, uint64_t* type_ranges);
void splbcu_domain_free(splbcu_domain* d);

/* ---- geometry sources (slab-local construction) -------------
 * A source is a generator evaluated one z-slice at a time; the builders above
 * are splbcu_source_build(splbcu_source_*(...)).  A distributed simulation
 * created from a source (splbcu_sim_create_dist_source) classifies only its
 * own slab plus one halo slice per side when the reference partition
 * (decomp.hpp:65-121) is a z-slab split, instead of every rank holding the
 * whole SparseDomain (the reference's Simulation ctor, engine.hpp:114-140).
 * Same argument checks and error texts as the builders. */
typedef struct splbcu_source splbcu_source;
int splbcu_source_pipe(int32_t radius, int32_t length, double voxel_size, splbcu_source** out);
int splbcu_source_bifurcation(int32_t trunk_radius, int32_t branch_radius, int32_t trunk_length,
                              int32_t branch_length, double voxel_size, splbcu_source** out);
int splbcu_source_tree(int32_t root_radius, int32_t root_length, int32_t levels, double radius_ratio,
                       double length_ratio, double voxel_size, splbcu_source** out);
int splbcu_source_channel(int32_t nx, int32_t ny, int32_t nz, double voxel_size, splbcu_source** out);
/* The whole domain (classify_sites over every slice). */
int splbcu_source_build(const splbcu_source* s, splbcu_domain** out);
/* Host-side view of what rank `worker` of `n_workers` builds (for tests and
 * tools; computes every worker's slice counts in-process).  Returns 1 in
 * *slab when the partition is a z-slab split, else 0 and nothing else.  The
 * window is a domain (sites in global order restricted to the window);
 * splbcu_window_info gives its global indices; *part the worker's part
 * (site lists are window indices; other parts empty). */
int splbcu_source_window(const splbcu_source* s, int32_t n_workers, int32_t worker, int32_t* slab,
                         splbcu_domain** window, splbcu_partition** part);
int splbcu_window_info(const splbcu_domain* window, uint64_t* n_global, int32_t* own_lo, int32_t* own_hi,
                       uint64_t* global_index /* n_sites of the window, or NULL */);
void splbcu_source_free(splbcu_source* s);

/* ---- decomposition (decomp.hpp:16-188) ------------------------------------ */
int splbcu_partition_create(const splbcu_domain* d, int32_t n_workers,
                            splbcu_partition** out);
/* owner[n] and local_index[n] per global site; any pointer may be NULL. */
int splbcu_partition_global(const splbcu_partition* p, int32_t* owner,
                            uint32_t* local_index);
/* Worker part shape: number of sites, n_edge, number of neighbours. */
int splbcu_partition_part_shape(const splbcu_partition* p, int32_t w,
                                uint32_t* n_sites, uint32_t* n_edge,
                                uint32_t* n_neighbors);
/* Worker part: sites (global, worker-local order), edge/mid ranges (6 pairs
 * each, local indices), neighbours ascending.  Any pointer may be NULL. */
int splbcu_partition_part(const splbcu_partition* p, int32_t w, uint32_t* sites,
                          uint64_t* edge_ranges, uint64_t* mid_ranges,
                          int32_t* neighbors);
double splbcu_partition_imbalance(const splbcu_partition* p); /* decomp.hpp:30 */
void splbcu_partition_free(splbcu_partition* p);

/* ---- simulation (engine.hpp:121-205) -------------------------------------- */
/* Simulation(SparseDomain, BCSet, EngineParams) (engine.hpp:123-140): all
 * workers in this process, placed on params->device_ids round robin;
 * halo exchange between workers by device-to-device / peer copies. */
int splbcu_sim_create(const splbcu_domain* d, const splbcu_bc* bcs,
                      uint32_t n_bcs, const splbcu_params* params,
                      splbcu_sim** out);
/* One process per GPU: this process owns worker `rank` of params->workers ==
 * nranks on device params->device_ids[0]; the halo exchange is NCCL send/recv
 * over NVLink on a communicator built from `nccl_id` (128 bytes from
 * splbcu_nccl_unique_id on rank 0, broadcast by the caller). */
int splbcu_nccl_unique_id(uint8_t out128[128]);
int splbcu_sim_create_dist(const splbcu_domain* d, const splbcu_bc* bcs,
                           uint32_t n_bcs, const splbcu_params* params,
                           int32_t rank, int32_t nranks,
                           const uint8_t nccl_id[128], splbcu_sim** out);
/* As splbcu_sim_create_dist, over a geometry source: slab-local construction
 * (each rank classifies only its own slices + one halo slice per side) when
 * the partition is a z-slab split, else the whole domain is built.  Results
 * are bit-identical to splbcu_sim_create_dist on splbcu_source_build(s). */
int splbcu_sim_create_dist_source(const splbcu_source* src, const splbcu_bc* bcs,
                                  uint32_t n_bcs, const splbcu_params* params,
                                  int32_t rank, int32_t nranks,
                                  const uint8_t nccl_id[128], splbcu_sim** out);
/* 1 when this rank holds only its window of the domain (then
 * splbcu_sim_partition returns NULL); sites of the whole domain. */
int32_t splbcu_sim_slab_local(const splbcu_sim* s);
uint64_t splbcu_sim_n_sites(const splbcu_sim* s);
/* run(nSteps) (engine.hpp:155-197).  The steps are enqueued and the
 * PREVIOUS run is completed before returning (so consecutive calls keep the
 * GPU busy); every accessor below completes the run in flight first, so the
 * results are those of a synchronous engine.  A run with captures, and every
 * run under SPLBCU_SYNC_RUN=1, completes before returning.  An exchange
 * failure is reported by this call or, at the latest, by the next one. */
int splbcu_sim_run(splbcu_sim* s, uint64_t n_steps);
uint64_t splbcu_sim_steps_run(const splbcu_sim* s);
double splbcu_sim_step_loop_seconds(const splbcu_sim* s);
/* Device-measured seconds of the step loop (CUDA events, max over local
 * workers' streams) — the number the bench reports. */
double splbcu_sim_device_loop_seconds(const splbcu_sim* s);
/* snapshot_fields() (engine.hpp:200-205): 4*n doubles (rho,ux,uy,uz) in domain
 * order (n = splbcu_sim_n_sites); in dist mode assembled across ranks
 * (collective: every rank must call it). */
int splbcu_sim_snapshot(splbcu_sim* s, double* out4n);
/* Workers owned by this handle (all in-process; one in dist mode). */
int32_t splbcu_sim_n_workers(const splbcu_sim* s);
int32_t splbcu_sim_worker_is_local(const splbcu_sim* s, int32_t w);
/* store(w) (engine.hpp:149, layout.hpp:19-62): n_sites, shared_size. */
int splbcu_sim_store_shape(const splbcu_sim* s, int32_t w, uint32_t* n_sites,
                           uint32_t* shared_size);
/* Host copy of f_old (which=0) or f_new (which=1) of worker w in the
 * reference's DistributionStore layout (params.layout, reference local site
 * order, 19*n + shared entries). */
int splbcu_sim_get_f(splbcu_sim* s, int32_t w, int32_t which, double* host);
int splbcu_sim_set_f(splbcu_sim* s, int32_t w, int32_t which, const double* host);
/* map(w) (engine.hpp:150, layout.hpp:113-140), exported from the device-built
 * table into the reference's encoding (reference local order, params.layout).
 * dest/op/iolet: 18*n_local; recv_dest, send_src_site, send_src_dir:
 * shared_size; seg_*: n_segments.  Any pointer may be NULL. */
int splbcu_sim_map_shape(const splbcu_sim* s, int32_t w, uint32_t* n_local,
                         uint32_t* shared_size, uint32_t* n_segments);
int splbcu_sim_export_map(splbcu_sim* s, int32_t w, uint32_t* dest, uint8_t* op,
                          uint16_t* iolet, uint32_t* recv_dest,
                          uint32_t* send_src_site, uint8_t* send_src_dir,
                          int32_t* seg_neighbor, uint32_t* seg_base,
                          uint32_t* seg_count);
/* map(w).sources (layout.hpp:104-119, 237-282): the pull-side source of every
 * slot [site*18 + (j-1)] in the reference encoding — src_site (local index;
 * FromLocal only, else the site itself / 0), op (GatherOp: 0 FromLocal,
 * 1 FromRemote, 2 SelfBounce, 3 SelfIolet) and iolet id.  Arrays of 18*n. */
int splbcu_sim_export_sources(splbcu_sim* s, int32_t worker, uint32_t* src_site,
                              uint8_t* op, uint16_t* iolet);
/* assignment() (engine.hpp:143): the partition the simulation uses (borrowed,
 * valid for the simulation's lifetime); NULL when slab-local. */
const splbcu_partition* splbcu_sim_partition(const splbcu_sim* s);
/* cache() (engine.hpp:144, 59-68): captures. */
uint64_t splbcu_sim_n_captures(const splbcu_sim* s);
int splbcu_sim_capture(const splbcu_sim* s, uint64_t k, uint64_t* step,
                       double* fields4n);
/* series() (engine.hpp:145, 70-78): rows and per-iolet columns.  series_rows
 * completes the pending reduction; on failure it returns 0 and records the
 * error (splbcu_last_error). */
uint64_t splbcu_sim_series_rows(const splbcu_sim* s);
int splbcu_sim_series(const splbcu_sim* s, uint32_t iolet, double* max_speed,
                      double* pressure, double* flow);
/* Output formats (snapshot.hpp:12-82): the captures as the reference's
 * snapshots.bin (per capture: u64 step, then 4*n f64 in domain order) and the
 * iolet series as its timeseries.csv text.  series_csv writes at most cap
 * bytes (NUL-terminated when room) and always reports the full length. */
int splbcu_sim_write_snapshots(const splbcu_sim* s, const char* path);
int splbcu_sim_series_csv(const splbcu_sim* s, double dt_s, char* buf, size_t cap,
                          size_t* len);
/* B200 instrumentation (no reference equivalent): CUDA-event timing of every
 * fused plain-site collide+stream launch, on the stream it is launched on. */
int splbcu_sim_set_kernel_timing(splbcu_sim* s, int32_t on);
int splbcu_sim_kernel_stats(const splbcu_sim* s, double* plain_seconds,
                            uint64_t* plain_launches, uint64_t* plain_sites);
/* Number of kernels this handle launched inside run() so far. */
uint64_t splbcu_sim_launch_count(const splbcu_sim* s);
/* The kernel the bulk (Inner+Wall mid-range) plain launch uses now, chosen
 * online: 0 just-in-time table loads, 1 table prefetch after the
 * divisions, -1 another (forced variant or uncompressed table). */
int32_t splbcu_sim_bulk_kernel(const splbcu_sim* s);
/* Bytes the iolet series moves device -> host per step (0 unless
 * observe_iolets): reduced rows plus the entries of iolets the host reduces. */
uint64_t splbcu_sim_series_d2h_bytes(const splbcu_sim* s);
void splbcu_sim_destroy(splbcu_sim* s);

#ifdef __cplusplus
}
#endif
#endif /* SPLBCU_H */
