// B200 engine: the reference's splb::Simulation (engine.hpp:121-650)
// re-designed around GPU-resident workers.
#pragma once

#include <memory>
#include <string>
#include <vector>

#include "host.hpp"

namespace splbcu {

struct BCEntry {
    int kind = 0;  // 0 pressure, 1 velocity
    TimeTable table;
};

struct Params {
    double tau = 0.9, rho0 = 1.0, dt_s = 1.0;
    int layout = 0, scheme = 0, sequence = 0, workers = 1;
    uint64_t capture_period = 0;
    bool observe_iolets = false;
    double exchange_timeout_s = 30.0;
    int halo_mode = 0;  // 0: NCCL send/recv (dist) or peer copies; 1: fused P2P stores
    int storage = 0;    // 0: two buffers (push); 1: one buffer, AA pattern in place
    std::vector<int> devices;
};

struct Capture {
    uint64_t step = 0;
    std::vector<double> fields;
};

struct Series {
    uint64_t rows = 0;
    std::vector<std::vector<double>> max_speed, pressure, flow;
};

// Exported StreamingMap in the reference encoding (layout.hpp:113-140).
struct ExportedMap {
    uint32_t n_local = 0, shared_size = 0;
    std::vector<uint32_t> dest;
    std::vector<uint8_t> op;
    std::vector<uint16_t> iolet;
    std::vector<uint32_t> recv_dest, send_site;
    std::vector<uint8_t> send_dir;
    std::vector<int> seg_neighbor;
    std::vector<uint32_t> seg_base, seg_count;
    // pull side (GatherSource, layout.hpp:104-108), [site*18 + j-1]
    std::vector<uint32_t> src_site;
    std::vector<uint8_t> src_op;
    std::vector<uint16_t> src_iolet;
};

class Engine;  // defined in engine.cu

class Simulation {
  public:
    // In-process: all workers in this process.
    Simulation(const Domain& d, std::vector<BCEntry> bcs, Params p);
    // One process per GPU with NCCL (rank owns worker `rank`).
    Simulation(const Domain& d, std::vector<BCEntry> bcs, Params p, int rank, int nranks,
               const void* nccl_id);
    // Distributed engine over a geometry source: slab-local construction
    // when the partition is a z-slab split (nccl_id null: in-process, whole domain).
    Simulation(const Source& src, std::vector<BCEntry> bcs, Params p, int rank, int nranks,
               const void* nccl_id);
    ~Simulation();
    bool slab_local() const;  // this rank holds only its window of the domain
    uint64_t n_sites() const; // sites of the whole domain
    uint64_t series_d2h_bytes() const;

    void run(uint64_t n);
    uint64_t steps_run() const;
    double step_loop_seconds() const;
    double device_loop_seconds() const;
    double plain_kernel_seconds() const;
    uint64_t plain_kernel_launches() const;
    uint64_t plain_kernel_sites() const;
    void set_kernel_timing(bool on);
    uint64_t launch_count() const;
    int bulk_kernel() const;
    void snapshot(double* out4n);
    int n_workers() const;
    bool is_local(int w) const;
    void store_shape(int w, uint32_t* n, uint32_t* shared) const;
    void get_f(int w, int which, double* host);
    void set_f(int w, int which, const double* host);
    ExportedMap export_map(int w);
    const Partition& partition() const;
    const std::vector<Capture>& captures() const;
    const Series& series() const;

  private:
    std::unique_ptr<Engine> e_;
};

std::string nccl_unique_id(void* out128);

}  // namespace splbcu
