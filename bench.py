#!/usr/bin/env python3
"""MSUPS of the fused D3Q19 sparse LBM step on B200 (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload c2|c3|c1|c4]

Default workload at every N: config C3 — a 1.07e8-site bifurcating vessel
tree (BASELINE configs[2], the config the metric "MSUPS at 1/2/4/8 B200" is
quoted on), pressure iolets, strong scaling (the same total work at every N,
so the driver's per-N values give the strong-scaling efficiency directly).
N>1: torchrun, one process per GPU, slab decomposition, fused NVLink P2P halo.
Storage: the AA single buffer by default (same bits as the reference's
two-buffer push, half the HBM, faster on the vessel trees: DESIGN §6b); the
dense C4 channel defaults to the two-buffer push kernels (`--storage two`),
which are faster there.
At N=1 the line also carries `secondary`: config C2 — build_pipe(48, 1400)
(10,130,400 sites), 60-bpm pulsatile velocity inlet (proj/configs/
pipe_beat.cfg), outlet p=1/3, tau 0.8, dt 5e-4 s — kernel-only value and
roofline (`--workload c2` makes it the primary line).

value  : sites*steps / device time of the step loop (CUDA events on the
         launching streams, max over ranks), inputs resident in HBM.
e2e    : the same metric through the public C-ABI call sequence a user makes
         (Simulation.run(1) per step with the iolet series on: per-step BC
         staging H2D and the observation row D2H), host wall clock.
roofline: the bulk plain-site fused kernels (AA: lbm_aa_even_tma /
         lbm_aa_odd_w, 304 / 342.25 B/site -> 323.125 per step; two buffers:
         lbm_push_dyn, 342.25 B/site: 19*8 read + 19*8 write + 18*(2+4/32)
         compressed index), algorithmic bytes per launch / CUDA-event launch
         time; frac_376 restates it in SURVEY §8d's 376 B/site.
cpu_baseline: the unmodified reference (oracle/_ref) on this host's cores,
         bounded sample of the same workload (rank 0, N=1 only).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

BYTES_PER_SITE = 19 * 8 + 19 * 8 + 18 * 4  # 376
DESIGN_BYTES_PER_SITE = 19 * 8 + 19 * 8 + 18 * (2 + 4 / 32)  # 342.25: compressed-table kernel
CS2 = 1.0 / 3.0
BEAT = ([(0.0, 0.008), (0.05, 0.012), (0.1, 0.024), (0.15, 0.036), (0.2, 0.04), (0.25, 0.036), (0.3, 0.026),
         (0.35, 0.016), (0.4, 0.01), (0.5, 0.007), (0.6, 0.006), (0.75, 0.0055), (0.9, 0.006)], 1.0)
DT_BEAT = CS2 * (0.8 - 0.5) * 0.001 * 0.001 / 0.0002  # config.hpp:42-46 on pipe_beat.cfg


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


C4W_SITES_PER_GPU = 3.5e8


def workload(M, name, scale=1.0, source=False, world=1):
    """Returns (domain, bcs, params, description).  source=True returns the
    geometry as a Source instead (slab-local construction on each rank)."""
    def geo(kind, *args):
        return getattr(M.Source, kind)(*args) if source else getattr(M, "build_" + kind)(*args)

    if name == "c2":
        L = max(4, int(round(1400 * scale)))
        d = geo("pipe", 48, L)
        bcs = M.BCSet([M.BCEntry(M.VELOCITY, M.TimeTable(*BEAT)), M.BCEntry(M.PRESSURE, M.TimeTable.constant(CS2))])
        return d, bcs, dict(tau=0.8, dt_s=DT_BEAT), f"C2 pipe R=48 L={L}, 60-bpm velocity inlet, p_out=1/3, tau=0.8"
    if name == "c1":
        d = geo("pipe", 16, 128)
        dp = 0.02 * 4.0 * (CS2 * 0.4) * 128 / 256.0
        bcs = M.BCSet([M.BCEntry(M.PRESSURE, M.TimeTable.constant(CS2 + dp / 2)),
                       M.BCEntry(M.PRESSURE, M.TimeTable.constant(CS2 - dp / 2))])
        return d, bcs, dict(tau=0.9, dt_s=1.0), "C1 Poiseuille pipe R=16 L=128, pressure iolets, tau=0.9"
    if name == "c3":
        levels = 6  # R0=80, L0=800: 107,037,564 sites, 64 outlets
        d = geo("tree", 80, max(8, int(round(800 * scale))), levels, 0.8, 0.8)
        n_out = 2 ** levels
        ents = [M.BCEntry(M.PRESSURE, M.TimeTable.constant(CS2 * 1.001))]
        ents += [M.BCEntry(M.PRESSURE, M.TimeTable.constant(CS2 * 0.999)) for _ in range(n_out)]
        return d, M.BCSet(ents), dict(tau=0.8, dt_s=1.0), f"C3 bifurcating tree R0=80 L0={max(8, int(round(800 * scale)))}, {levels} levels, pressure iolets"
    if name == "c5":
        # sparse vasculature, ~1e9 sites: R0=160, L0=1600, 7 levels
        # -> 1.01e9 sites at scale 1, ~1.2 % of its bounding box, 129 iolets
        levels = 7
        L0 = max(8, int(round(1600 * scale)))
        d = geo("tree", 160, L0, levels, 0.8, 0.8)
        ents = [M.BCEntry(M.PRESSURE, M.TimeTable.constant(CS2 * 1.001))]
        ents += [M.BCEntry(M.PRESSURE, M.TimeTable.constant(CS2 * 0.999)) for _ in range(2 ** levels)]
        return d, M.BCSet(ents), dict(tau=0.8, dt_s=1.0), f"C5 sparse vascular tree R0=160 L0={L0}, {levels} levels, pressure iolets"
    if name in ("c4", "c4w"):
        # c4w: weak scaling (BASELINE configs[3]) — the channel grows along z
        # with the GPU count, C4W_SITES_PER_GPU sites per GPU (two f buffers +
        # u32 and compressed tables: ~414 B/site, ~145 GB of the 180 GB HBM)
        nz = int(round(2400 * scale)) if name == "c4" else int(round(C4W_SITES_PER_GPU / 65536 * world * scale))
        d = geo("channel", 256, 256, nz)
        bcs = M.BCSet([M.BCEntry(M.PRESSURE, M.TimeTable.constant(CS2 * 1.001)),
                       M.BCEntry(M.PRESSURE, M.TimeTable.constant(CS2 * 0.999))])
        return d, bcs, dict(tau=0.8, dt_s=1.0), f"C4 dense channel 256x256x{nz}"
    raise SystemExit(f"unknown workload {name}")


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu):
        self.gpu, self.rows, self.proc = gpu, [], None
        self.t0 = self.t1 = None

    def __enter__(self):
        self.t0 = time.perf_counter()
        if self.gpu is None:
            return self
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # the sampler is running before the timed region starts (nvidia-smi
            # takes a moment to start): a short region still gets its samples
            deadline = time.perf_counter() + 5.0
            while not self.rows and time.perf_counter() < deadline and self.proc.poll() is None:
                time.sleep(0.005)
        except Exception:
            self.proc = None
        self.t0 = time.perf_counter()
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append((time.perf_counter(), [x.strip() for x in line.split(",")]))

    def __exit__(self, *a):
        self.t1 = time.perf_counter()
        if self.proc:
            time.sleep(0.06)  # the sample in flight at the end of the region
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self):
        """Samples taken inside the timed region (read within one sampling
        period after its end: nvidia-smi reports the state at the query)."""
        rows = [r for t, r in self.rows if self.t0 is not None and self.t0 <= t <= (self.t1 or t) + 0.05]
        self.rows_in = rows
        sm = [float(r[1]) for r in rows if len(r) >= 7 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if len(r) >= 7 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows if len(r) >= 7 for k in range(4) if r[3 + k] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm)}


# Bounded samples of the bench geometries for the reference engine, as
# (generator, args, description).  The reference has no tree/channel builder:
# oracle/geometry_gen.py restates the product's voxelisation in numpy and the
# reference's own classify_sites classifies it (tests/test_host.py pins that
# this equals the product's build_tree / build_channel), so the reference
# process never maps the product library.
REF_SAMPLES = {
    # reference arm: as large as the reference's setup allows within a few
    # minutes (its Simulation ctor runs ~5 s per 1e6 sites)
    "arm": {"c3": ("tree", (48, 240, 6, 0.8, 0.8), "C3-shaped tree sample R0=48 L0=240, 6 levels, 65 pressure iolets"),
            "c5": ("tree", (32, 480, 7, 0.8, 0.8), "C5-shaped tree sample R0=32 L0=480, 7 levels, 129 pressure iolets"),
            "c4": ("channel", (192, 192, 300), "C4-shaped channel sample 192x192x300")},
    # cpu_baseline beside our N=1 line: ~10-30 s of CPU work in total
    "baseline": {"c3": ("tree", (32, 160, 6, 0.8, 0.8), "C3-shaped tree sample R0=32 L0=160, 6 levels, 65 pressure iolets"),
                 "c5": ("tree", (32, 320, 7, 0.8, 0.8), "C5-shaped tree sample R0=32 L0=320, 7 levels, 129 pressure iolets"),
                 "c4": ("channel", (128, 128, 200), "C4-shaped channel sample 128x128x200")},
}


def cpu_reference_run(name, steps_cap, seconds, scale, warmup=1, sample="baseline"):
    """The unmodified reference (oracle/_ref) on all host cores, on a bounded
    sample of workload `name`; returns (MSUPS, cores, steps, sites, desc)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import impls
    R = impls.reference()
    if name in REF_SAMPLES[sample]:
        import geometry_gen as G
        kind, gargs, desc = REF_SAMPLES[sample][name]
        vox, io = getattr(G, kind)(*gargs)
        d = G.classify(R, vox, io)
        del vox
        ents = [R.BCEntry(R.PRESSURE, R.TimeTable.constant(CS2 * 1.001))]
        ents += [R.BCEntry(R.PRESSURE, R.TimeTable.constant(CS2 * 0.999)) for _ in io[1:]]
        bcs, p = R.BCSet(ents), dict(tau=0.8, dt_s=1.0)
    else:
        d, bcs, p, desc = workload(R, name, scale)
    cores = os.cpu_count() or 1
    sim = R.Simulation(d, bcs, R.EngineParams(workers=cores, layout=R.SOA, **p))
    sim.run(max(1, warmup))  # untimed warm-up steps
    t0 = sim.step_loop_seconds()
    steps = 0
    while steps < steps_cap and (sim.step_loop_seconds() - t0) < seconds:
        sim.run(1)
        steps += 1
    T = sim.step_loop_seconds() - t0
    return d.n_sites() * steps / T / 1e6, cores, steps, d.n_sites(), desc


BULK_KERNELS = {0: "void lbm_push_dyn<256, 2, 2>", 1: "void lbm_push_tmc<256, 2, 2, 4102>",
                2: "void lbm_push_run<256, 2, 2>", 3: "void lbm_push_tmc<256, 2, 2, 6>"}
RUN_BYTES_PER_SITE = 19 * 8 + 19 * 8 + 3456 / 256  # 317.5: run-length table kernel
# AA single buffer: even steps 304 B/site (no table), odd steps
# the compressed-table gather/scatter 342.25 -> 323.125 per step on average
AA_BYTES_PER_SITE = (19 * 8 * 2 + DESIGN_BYTES_PER_SITE) / 2
AA_KERNELS = "AA pair: void lbm_aa_even_tma<256, 2, 2> + void lbm_aa_odd_w<4, 3, 1>"


def load_profile_traffic(name, kernel=None, developed=False):
    """DRAM bytes per site of the bulk plain kernel from the committed ncu
    capture of this workload (profiles/ncu_summary.json), or None.  Entries of
    the same workload ("c3", "c3_jit", "c3_dev_jit", ...) captured on the
    kernel the engine's online choice launched (`kernel`) and in the same
    flow state (developed: keys containing "_dev") are preferred."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            s = json.load(f)
    except Exception:
        return None, None
    cands = [k for k in s if k == name or k.startswith(name + "_")]
    cands.sort(key=lambda k: (("_dev" in k) != developed, s[k].get("kernel") != kernel))
    if cands:
        return s[cands[0]].get("traffic_bytes_per_site"), cands[0]
    return None, None


def timed_loop(sim, n, steps, warmup, bps, barrier, max_over_ranks, gpu, name, developed=False, aa=False):
    """W untimed steps, then K steps timed by CUDA events on the launching
    streams (max over ranks), with per-launch events on the bulk plain kernel
    and nvidia-smi clocks sampled during the timed region."""
    sim.run(warmup)
    barrier()
    sim.set_kernel_timing(True)
    k0 = sim.kernel_stats()
    l0 = sim.launch_count()
    d0 = sim.device_loop_seconds()
    # rank 0 samples its GPU (the line it prints); one nvidia-smi per node
    # keeps the driver queries off the other ranks' launch paths.  The
    # sampler is up before the barrier, so every rank enters the timed steps
    # together (a rank waiting for nvidia-smi to start would otherwise hold
    # its neighbours' steps at the halo exchange inside their timed region).
    clk = ClockSampler(gpu if int(os.environ.get("RANK", "0")) == 0 else None).__enter__()
    barrier()
    clk.t0 = time.perf_counter()
    try:
        sim.run(steps)
        sim.device_loop_seconds()  # run() returns while its last steps execute: wait inside the sampled window
    finally:
        clk.__exit__(None, None, None)
    barrier()
    dev_s = max_over_ranks(sim.device_loop_seconds() - d0)
    k1 = sim.kernel_stats()
    launches = sim.launch_count() - l0
    sim.set_kernel_timing(False)
    value = n * steps / dev_s / 1e6
    ks, kl, kn = k1[0] - k0[0], k1[1] - k0[1], k1[2] - k0[2]
    hbm, src = peaks()
    kernel = AA_KERNELS if aa else BULK_KERNELS.get(sim.bulk_kernel())
    if not aa and sim.bulk_kernel() == 2 and bps == DESIGN_BYTES_PER_SITE:
        bps = RUN_BYTES_PER_SITE  # the online choice launched the run-length table kernel
    traffic, traffic_key = load_profile_traffic(name + "_dev_aa" if aa else name, kernel, developed)
    # The default kernel reads a compressed table (int16 deltas + a u32 base per
    # 32 sites): its algorithmic bytes are 304 + 18*(2 + 4/32) = 342.25 B/site
    # (AA storage: even steps 304, odd steps 342.25 -> 323.125 on average).
    # `achieved`/`frac` use those bytes (the DRAM rate the kernel really
    # sustains); `achieved_376`/`frac_376` restate it in SURVEY §8d's
    # 376 B/site (the reference data layout), which can exceed 1.0 because the
    # kernel moves fewer bytes than that layout.
    achieved = (kn / kl) * bps / (ks / kl) / 1e9 if kl else None
    achieved_376 = (kn / kl) * BYTES_PER_SITE / (ks / kl) / 1e9 if kl else None
    roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
            "frac": achieved / hbm if achieved else None,
            "traffic": (traffic * kn / kl) if (traffic and kl) else None,
            "peak_source": src,
            "kernel": ("lbm_aa_even_tma / lbm_aa_odd_w (AA single buffer: even steps in place, odd steps "
                       "gather/scatter)") if aa else
                      "lbm_push_dyn / lbm_push_tmc / lbm_push_run (Inner+Wall fused collide+stream, TMA-pipelined)",
            "kernel_template": kernel, "traffic_source": traffic_key,
            "bytes_per_site": bps, "achieved_376": achieved_376,
            "frac_376": achieved_376 / hbm if achieved_376 else None,
            "sites_per_launch": kn / kl if kl else None, "avg_launch_ms": ks / kl * 1e3 if kl else None,
            "kernel_share": ks / dev_s if dev_s else None}
    return value, dev_s, launches, roof, clk



def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    name = args.workload or "c3"
    scale = 1.0 if name == "c2" else 0.25
    v, cores, steps, n, desc = cpu_reference_run(name, max(args.steps, 1), 60.0, scale, args.warmup, "arm")
    line = {"impl": "reference", "metric": "MSUPS", "value": v, "unit": "MSUPS", "n_gpus": args.gpus,
            "steps": steps, "warmup": args.warmup, "ms_per_step": n / (v * 1e6) * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": desc, "sites": n, "parallelism": f"{cores} CPU worker threads"},
            "cpu_baseline": {"value": v, "unit": "MSUPS", "cores": cores, "kind": "reference",
                             "sample": f"{steps} steps of {desc} ({n} sites)"},
            "e2e": {"value": v, "unit": "MSUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def spawn_ranks(n):
    """`python bench.py --gpus N` outside torchrun: relaunch this command as
    N ranks (one per GPU, rendezvous on 127.0.0.1), the way the driver's
    scaling run launches it; rank 0 prints the line."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    rc = subprocess.call(cmd)
    if rc != 0:
        raise SystemExit(rc)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=None)
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-secondary", action="store_true", help="N=1: skip the C2 kernel-only line")
    ap.add_argument("--quick", action="store_true", help="kernel-only number (tuning runs)")
    ap.add_argument("--storage", default=None, choices=["two", "aa"],
                    help="one buffer updated in place (AA pattern: the same bits in half the memory; the "
                         "default for the vessel trees C1-C3/C5, faster there at N = 1 / 2 / 4, DESIGN §6b) "
                         "or two buffers (the reference's f_old / f_new push; the default for the dense C4 "
                         "channel)")
    ap.add_argument("--scheme", default="push", choices=["push", "pull"],
                    help="push (fused collide + scatter) or the reference's pull gather (update_pull)")
    ap.add_argument("--halo", default="p2p", choices=["nccl", "p2p"],
                    help="N>1 halo exchange: NCCL send/recv + PostReceive, or fused NVLink P2P stores")
    ap.add_argument("--develop", type=int, default=3000,
                    help="untimed steps before the warm-up so the headline is measured in a developed flow "
                         "(0: from rest); the from-rest number is reported beside it")
    ap.add_argument("--geometry", default="source", choices=["source", "domain"],
                    help="N>1: each rank classifies only its own slab of the generator (source) "
                         "or every rank builds the whole domain")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        return run_reference_arm(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # launched without torchrun: spawn one rank per GPU ourselves
        return spawn_ranks(args.gpus)
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world} ranks were launched")

    import paper_2202_11770_b200 as P

    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    name = args.workload or "c3"
    if world > 1:
        import torch
        import torch.distributed as td
        torch.cuda.set_device(local)
        td.init_process_group("nccl", device_id=torch.device("cuda", local))

    def make_sim(params):
        """In-process engine at N=1; at N>1 one worker per rank, joined by a
        fresh NCCL communicator (unique id from rank 0, broadcast by torch)."""
        if world == 1:
            return P.Simulation(d, bcs, params)
        import torch
        import torch.distributed as td
        td.barrier()
        uid = P.Simulation.nccl_unique_id() if rank == 0 else bytes(128)
        t = torch.tensor(list(uid), dtype=torch.uint8, device="cuda")
        td.broadcast(t, 0)
        return P.Simulation.distributed(d, bcs, params, rank, world, bytes(t.cpu().tolist()))

    t_setup = time.time()
    slab_src = world > 1 and args.geometry == "source"
    d, bcs, p, desc = workload(P, name, args.scale, source=slab_src, world=world)
    halo_mode = 1 if args.halo == "p2p" else 0
    if args.storage is None:
        # per workload, as measured: the AA pair is faster on the
        # vessel trees (C3 at N = 1/2/4, C5), the two-buffer push on the dense
        # C4 channel (18,787 vs 18,217 at N=1, 75,059 vs 71,659 at N=4)
        args.storage = "two" if name in ("c4", "c4w") else "aa"
    storage = 1 if args.storage == "aa" else 0
    scheme = P.PULL if args.scheme == "pull" else P.PUSH
    sim = make_sim(P.EngineParams(workers=world, devices=[local], halo_mode=halo_mode, storage=storage, scheme=scheme,
                                  **p))
    n = sim.n_sites()
    sim_slab = sim.slab_local()
    setup_s = time.time() - t_setup

    def barrier():
        if world > 1:
            import torch.distributed as td
            td.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        import torch
        import torch.distributed as td
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        td.all_reduce(t, op=td.ReduceOp.MAX)
        return float(t.item())

    bps = AA_BYTES_PER_SITE if args.storage == "aa" else DESIGN_BYTES_PER_SITE

    def develop(sim, steps, chunk=None):
        """Untimed steps that take the flow from rest to a developed state
        (chunked so observation buffers stay small)."""
        left = steps
        while left > 0:
            k = min(left, chunk or left)
            sim.run(k)
            left -= k

    # from rest (f = equilibrium(rho0, 0) everywhere): secondary number
    rest = None
    if args.develop > 0:
        rv, rdev, _, rroof, rclk = timed_loop(sim, n, args.steps, args.warmup, bps, barrier, max_over_ranks, local,
                                              name)
        rest = {"value": rv, "unit": "MSUPS", "ms_per_step": rdev / args.steps * 1e3,
                "frac": rroof["frac"], "kernel_template": rroof["kernel_template"], "clocks": rclk.summary(),
                "note": f"the first {args.warmup + args.steps} steps from rest"}
        develop(sim, args.develop)
        barrier()
    state = f"developed flow: {args.develop + (args.warmup + args.steps if rest else 0)} untimed steps first" \
        if args.develop > 0 else "from rest"
    value, dev_s, launches, roof, clk = timed_loop(sim, n, args.steps, args.warmup, bps, barrier, max_over_ranks, local,
                                                  name, developed=args.develop > 0, aa=storage == 1)

    if args.quick:
        if rank == 0:
            print(json.dumps({"value": value, "roofline": roof, "launches": launches, "clocks": clk.summary(),
                              "from_rest": rest}))
        return
    # e2e through the public API: run(1) per step with the iolet series on,
    # in the same (developed) state as the device-timed number
    sim.close()
    params_e = P.EngineParams(workers=world, devices=[local], observe_iolets=True, halo_mode=halo_mode,
                              storage=storage, scheme=scheme, **p)
    sim = make_sim(params_e)
    develop(sim, args.develop, chunk=100)
    for _ in range(args.warmup):
        sim.run(1)
    barrier()
    e2e_steps = max(50, min(args.steps, 200))  # a window long enough that the final series() read is not a fixed cost
    dd0 = sim.device_loop_seconds()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        sim.run(1)
    t_ser = time.perf_counter()
    ser = sim.series()  # completes the last row (the host part of the reduction is lazy)
    t_end = time.perf_counter()
    barrier()
    e2e_s = max_over_ranks(time.perf_counter() - t0)
    # diagnostics: the same window's device time of the steps (CUDA events, as
    # `value`) and the final series() call's share of the wall time
    e2e_dev_s = max_over_ranks(sim.device_loop_seconds() - dd0)
    series_call_s = max_over_ranks(t_end - t_ser)
    # the series row's device -> host bytes (reduced values + the entries of
    # the iolets the host reduces)
    d2h = sim.series_d2h_bytes()
    e2e = {"value": n * e2e_steps / e2e_s / 1e6, "unit": "MSUPS",
           "h2d_bytes_per_step": 8 * len(bcs.entries), "d2h_bytes_per_step": d2h,
           "note": "Simulation.run(1) per step via the C-ABI with the iolet series on: per-step BC values "
                   "H2D, the step, the series row (all-gathered across ranks, reduced in the reference's order) "
                   "D2H, host wall clock; " + state,
           "device_value": n * e2e_steps / e2e_dev_s / 1e6 if e2e_dev_s > 0 else None,
           "final_series_call_ms": series_call_s * 1e3}
    sim.close()

    secondary = None
    if world == 1 and name != "c2" and not args.no_secondary:
        # BASELINE configs[1] (the 1e7-site pulsatile pipe), kernel-only
        d, bcs, p, desc2 = workload(P, "c2")
        sim = P.Simulation(d, bcs, P.EngineParams(workers=1, devices=[local], storage=storage, **p))
        n2 = sim.n_sites()
        develop(sim, args.develop)
        v2, dev2, _, roof2, clk2 = timed_loop(sim, n2, max(args.steps, 50), args.warmup, bps, barrier,
                                              max_over_ranks, local, "c2", developed=args.develop > 0)
        sim.close()
        del d
        secondary = {"workload": desc2, "sites": n2, "value": v2, "unit": "MSUPS", "state": state,
                     "ms_per_step": dev2 / max(args.steps, 50) * 1e3, "roofline": roof2, "clocks": clk2.summary()}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            v, cores, steps, cn, cdesc = cpu_reference_run(name, 1000, 12.0, 0.1 if name == "c2" else 0.05)
            cpu = {"value": v, "unit": "MSUPS", "cores": cores, "kind": "reference",
                   "sample": f"{steps} steps of {cdesc} ({cn} sites)"}
        except Exception as ex:  # the reference shim may be absent
            cpu = {"value": None, "unit": "MSUPS", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {ex}"}

    if rank == 0:
        line = {"metric": "MSUPS", "value": value, "unit": "MSUPS", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": dev_s / args.steps * 1e3, "higher_is_better": True,
                "scaling": "weak" if name == "c4w" else "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": desc, "sites": n, "parallelism": f"slab decomposition x{world}",
                           "scheme": args.scheme, "storage": "AA single buffer" if storage else "two buffers",
                           "halo": (("NCCL send/recv + PostReceive" if halo_mode == 0 else "fused NVLink P2P stores")
                                    if world > 1 else "none"),
                           "l2": f"bytes moved per step (f read + written, table) {n * bps / 1e9:.1f} GB >> 126 MB L2; "
                                 "no flush needed",
                           "setup_s": round(setup_s, 2), "state": state,
                           "geometry": ("slab-local (each rank classifies its own slices)" if sim_slab
                                        else "whole domain on every rank")},
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": int(launches),
                "clocks": clk.summary()}
        if rest:
            line["from_rest"] = rest
        if secondary:
            line["secondary"] = secondary
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as td
        td.destroy_process_group()


if __name__ == "__main__":
    main()
