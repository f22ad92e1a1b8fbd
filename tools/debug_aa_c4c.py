"""AA 3 workers on the 48x40x120 channel: isolate the mismatch (debug)."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "oracle")]
import cases, impls  # noqa
P = impls.product()
d = P.build_channel(48, 40, 120)
bcs = lambda: P.BCSet([P.BCEntry(P.PRESSURE, P.TimeTable.constant(cases.CS2 * 1.001)),
                       P.BCEntry(P.PRESSURE, P.TimeTable.constant(cases.CS2 * 0.999))])
noise = cases.noise_for(d.n_sites(), 20240808, 0.01)
mode = sys.argv[1]
def sim(kw):
    return P.Simulation(d, bcs(), P.EngineParams(devices=[0], tau=0.8, dt_s=1.0, **kw))
ref = sim(dict(workers=1)); cases.apply_noise(P, ref, noise)
s = sim(dict(workers=3, storage=1)); cases.apply_noise(P, s, noise)
def cmp(tag):
    a, b = ref.snapshot_fields().reshape(-1, 4), s.snapshot_fields().reshape(-1, 4)
    bad = np.where((a != b).any(1))[0]
    print(mode, tag, "bad sites", len(bad), flush=True)
cmp("after noise")
# store round trip per worker
pa = s.assignment(); pr = ref.assignment()
for w in range(3):
    f = s.store(w).f_old()
    n = len(pa.parts[w].sites)
    fr = ref.store(0).f_old()[:19 * d.n_sites()].reshape(-1, 19)
    mine = f[:19 * n].reshape(n, 19)
    want = fr[pr.local_index[pa.parts[w].sites]]
    print(mode, "store w", w, "mismatch entries", int((mine != want).sum()), flush=True)
for k in range(1, 4):
    ref.run(1); s.run(1)
    cmp(f"after {k} steps")
