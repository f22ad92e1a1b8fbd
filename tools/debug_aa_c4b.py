"""AA with 3 workers on the C4-shaped channel: which sites / directions differ
after 1 step from the 1-worker push engine (debug)."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "oracle")]
import cases, impls  # noqa
P = impls.product()
nx, ny, nz = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
d = P.build_channel(nx, ny, nz)
bcs = lambda: P.BCSet([P.BCEntry(P.PRESSURE, P.TimeTable.constant(cases.CS2 * 1.001)),
                       P.BCEntry(P.PRESSURE, P.TimeTable.constant(cases.CS2 * 0.999))])
noise = cases.noise_for(d.n_sites(), 20240808, 0.01)
def fields(kw, steps):
    s = P.Simulation(d, bcs(), P.EngineParams(devices=[0], tau=0.8, dt_s=1.0, **kw))
    cases.apply_noise(P, s, noise)
    s.run(steps)
    snap = s.snapshot_fields().reshape(-1, 4)
    pa = s.assignment()
    own = np.zeros(d.n_sites(), np.int32)
    for w in range(pa.n_workers):
        own[pa.parts[w].sites] = w
    s.close()
    return snap, own
e = d.export()
z = e["coords"][:, 2]
for steps in (1, 2):
    ref, _ = fields(dict(workers=1), steps)
    for rep in range(3):
        for kw in (dict(workers=3, storage=1), dict(workers=3, storage=1, devices=[0])):
            got, own = fields(kw, steps)
            bad = np.where((got != ref).any(1))[0]
            zs = np.unique(z[bad]) if len(bad) else []
            print(steps, rep, kw, "bad sites", len(bad), "z:", list(zs)[:12], "owners:", np.bincount(own[bad], minlength=3).tolist() if len(bad) else [], flush=True)
            break
