"""One step of a workload in a developed flow, inside an NVTX range named
"target", for ncu:  ncu --nvtx --nvtx-include "target/" --set full ... \
    python tools/prof_target.py --workload c3 --develop 3000 [--storage aa] [--steps 2]
(the engine's own kernels of the development steps are not captured)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402  (NVTX)

import bench  # noqa: E402
import paper_2202_11770_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c3")
ap.add_argument("--develop", type=int, default=3000)
ap.add_argument("--storage", default="two")
ap.add_argument("--scheme", default="push")
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--variant", default=None)
a = ap.parse_args()
if a.variant:
    os.environ["SPLBCU_PLAIN_VARIANT"] = a.variant
d, bcs, p, desc = bench.workload(P, a.workload)
sim = P.Simulation(d, bcs, P.EngineParams(storage=1 if a.storage == "aa" else 0,
                                          scheme=P.PULL if a.scheme == "pull" else P.PUSH, **p))
sim.run(a.develop)
torch.cuda.nvtx.range_push("target")
sim.run(a.steps)
torch.cuda.nvtx.range_pop()
print("profiled", desc, sim.n_sites(), "sites, steps", sim.steps_run(), flush=True)
