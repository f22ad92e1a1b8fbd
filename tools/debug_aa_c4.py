"""AA 3-slab parity on the C4-shaped channel sample, by feature (debug)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "oracle")]
import cases, impls  # noqa
P = impls.product()
d = P.build_channel(48, 40, 120)
io = d.iolets
def bcs():
    return P.BCSet([P.BCEntry(P.PRESSURE, P.TimeTable.constant(cases.CS2 * 1.001)),
                    P.BCEntry(P.PRESSURE, P.TimeTable.constant(cases.CS2 * 0.999))])
noise = cases.noise_for(d.n_sites(), 20240808, 0.01)
def dig(kw, runs, cap=0, obs=False, noisy=True):
    s = P.Simulation(d, bcs(), P.EngineParams(devices=[0], tau=0.8, dt_s=1.0, capture_period=cap, observe_iolets=obs, **kw))
    if noisy: cases.apply_noise(P, s, noise)
    for r in runs: s.run(r)
    out = (cases.h(s.snapshot_fields()), [(c.step, cases.h(c.fields)) for c in s.cache()],
           {k: [cases.h(a) for a in v] for k, v in s.series().items() if k != "rows"})
    s.close()
    return out
for name, cap, obs, runs, noisy in (("plain", 0, False, (60,), True), ("split", 0, False, (20, 40), True),
                                    ("obs", 0, True, (20, 40), True), ("cap", 30, False, (20, 40), True),
                                    ("both", 30, True, (20, 40), True), ("rest", 0, False, (60,), False),
                                    ("short", 0, False, (1,), True), ("two", 0, False, (2,), True)):
    ref = dig(dict(workers=1), runs, cap, obs, noisy)
    res = []
    for kw in (dict(workers=3, storage=1), dict(workers=1, storage=1), dict(workers=2, storage=1), dict(workers=3, storage=1, halo_mode=1),
               dict(workers=3, halo_mode=1)):
        got = dig(kw, runs, cap, obs, noisy)
        res.append((str(kw), got[0] == ref[0], got[1] == ref[1], got[2] == ref[2]))
    print(name, res, flush=True)
