"""e2e A/B: Simulation.run(1) x K with the series on, async run() (default) vs
SPLBCU_SYNC_RUN=1 (each run completes before returning), same process/box.
  python tools/e2e_ab.py [--workload c3] [--develop 3000] [--steps 50]"""
import argparse, json, os, subprocess, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c3")
ap.add_argument("--develop", type=int, default=3000)
ap.add_argument("--steps", type=int, default=50)
ap.add_argument("--child", action="store_true")
ap.add_argument("--observe", type=int, default=1)
a = ap.parse_args()
if not a.child:
    for rep in range(2):
        for sync in ((False, True) if a.observe else (False,)):
            env = dict(os.environ)
            env.pop("SPLBCU_SYNC_RUN", None)
            if sync:
                env["SPLBCU_SYNC_RUN"] = "1"
            out = subprocess.run([sys.executable, __file__, "--child", "--workload", a.workload, "--develop",
                                  str(a.develop), "--steps", str(a.steps), "--observe", str(a.observe)], env=env,
                                 capture_output=True, text=True)
            print(json.dumps({"sync": sync, "rep": rep, **json.loads(out.stdout.strip().splitlines()[-1])}), flush=True)
    sys.exit(0)
import bench
import paper_2202_11770_b200 as P
d, bcs, p, desc = bench.workload(P, a.workload)
sim = P.Simulation(d, bcs, P.EngineParams(observe_iolets=bool(a.observe), **p))
n = sim.n_sites()
left = a.develop
while left > 0:
    k = min(100, left); sim.run(k); left -= k
for _ in range(5):
    sim.run(1)
sim.series()
d0 = sim.device_loop_seconds()
l0 = sim.step_loop_seconds()
t0 = time.perf_counter()
for _ in range(a.steps):
    sim.run(1)
sim.series()
e2e = time.perf_counter() - t0
dev = sim.device_loop_seconds() - d0
loop = sim.step_loop_seconds() - l0
print(json.dumps({"observe": a.observe, "e2e_msups": n * a.steps / e2e / 1e6, "device_msups": n * a.steps / dev / 1e6,
                  "host_loop_msups": n * a.steps / loop / 1e6}))
