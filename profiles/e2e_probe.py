"""Where the end-to-end run(1) time goes (profiling aid, not a bench line).

Runs the bench workload under torchrun like bench.py and times, per step,
run(1) with the iolet series off and on, next to the device step time.
    python -m torch.distributed.run --nproc-per-node N profiles/e2e_probe.py [workload]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main():
    import torch
    import torch.distributed as td
    import paper_2202_11770_b200 as P
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    name = sys.argv[1] if len(sys.argv) > 1 else ("c2" if world == 1 else "c3")
    if world > 1:
        torch.cuda.set_device(local)
        td.init_process_group("nccl", device_id=torch.device("cuda", local))
    g, bcs, p, desc = bench.workload(P, name, 1.0, source=world > 1)

    def make(observe):
        prm = P.EngineParams(workers=world, devices=[local], halo_mode=1, observe_iolets=observe, **p)
        if world == 1:
            return P.Simulation(g, bcs, prm)
        td.barrier()
        uid = P.Simulation.nccl_unique_id() if rank == 0 else bytes(128)
        t = torch.tensor(list(uid), dtype=torch.uint8, device="cuda")
        td.broadcast(t, 0)
        return P.Simulation.distributed(g, bcs, prm, rank, world, bytes(t.cpu().tolist()))

    out = {}
    for observe in (False, True):
        sim = make(observe)
        sim.run(5)
        if world > 1:
            td.barrier()
        d0 = sim.device_loop_seconds()
        l0 = sim.step_loop_seconds()
        t0 = time.perf_counter()
        K = 30
        for _ in range(K):
            sim.run(1)
        wall = (time.perf_counter() - t0) / K
        rec = dict(wall_ms=wall * 1e3, device_ms=(sim.device_loop_seconds() - d0) / K * 1e3,
                   loop_ms=(sim.step_loop_seconds() - l0) / K * 1e3)
        # one run(K): the same steps with a single host round trip
        if world > 1:
            td.barrier()
        t0 = time.perf_counter()
        sim.run(K)
        rec["runK_ms_per_step"] = (time.perf_counter() - t0) / K * 1e3
        if world > 1:
            allr = [None] * world
            td.all_gather_object(allr, rec)
            rec = {k: [round(r[k], 4) for r in allr] for k in rec}
        out[observe] = rec
        sim.close()
    if rank == 0:
        print(desc, world, json.dumps(out), flush=True)
    if world > 1:
        td.destroy_process_group()


if __name__ == "__main__":
    main()
