"""The fused P2P edge kernel in one process: C3 split into 2 workers on 2
devices (in-process, NVLink peer stores), developed flow, the target step
inside an NVTX range for ncu (a multi-rank job cannot be replayed by ncu)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import bench  # noqa: E402
import paper_2202_11770_b200 as P  # noqa: E402
d, bcs, p, desc = bench.workload(P, sys.argv[1] if len(sys.argv) > 1 else "c3")
sim = P.Simulation(d, bcs, P.EngineParams(workers=2, devices=[0, 1], halo_mode=1, **p))
sim.run(int(sys.argv[2]) if len(sys.argv) > 2 else 1000)
torch.cuda.nvtx.range_push("target")
sim.run(1)
torch.cuda.nvtx.range_pop()
sim.snapshot_fields()
print("profiled", desc, flush=True)
