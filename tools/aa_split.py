"""AA storage: even-step vs odd-step bulk-kernel time on a workload (developed
flow), from the engine's per-launch CUDA events.
  python tools/aa_split.py [--workload c3] [--develop 3000] [--storage aa|two]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2202_11770_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c3")
ap.add_argument("--develop", type=int, default=3000)
ap.add_argument("--storage", default="aa")
ap.add_argument("--steps", type=int, default=20)
a = ap.parse_args()
d, bcs, p, desc = bench.workload(P, a.workload)
sim = P.Simulation(d, bcs, P.EngineParams(storage=1 if a.storage == "aa" else 0, **p))
n = sim.n_sites()
sim.run(a.develop)
sim.set_kernel_timing(True)
out = {"even": [], "odd": []}
for k in range(a.steps):
    par = "odd" if (sim.steps_run() & 1) else "even"
    s0 = sim.kernel_stats()
    sim.run(1)
    s1 = sim.kernel_stats()
    out[par].append((s1[0] - s0[0], s1[2] - s0[2]))
res = {}
for par, v in out.items():
    t = sum(x[0] for x in v)
    sites = sum(x[1] for x in v)
    res[par] = {"ms": t / len(v) * 1e3, "msups": sites / t / 1e6}
res["workload"], res["sites"], res["storage"] = desc, n, a.storage
print(json.dumps(res))
