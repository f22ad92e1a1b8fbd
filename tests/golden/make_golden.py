"""Generates tests/golden/* from the UNMODIFIED reference.

The reference (header-only C++ under /root/reference/proj/include) is
compiled in place by oracle/Makefile into oracle/_ref/libsplbref.so and driven
through the same C-ABI mirror as the B200 engine (tests/impls.py).  Run here
(not on the GPU box):  python tests/golden/make_golden.py

Outputs
  golden.json  known-answer values + sha256 of canonicalised arrays
  golden.npz   small arrays (captures/series of the small parity cases)
Floating arrays are hashed after `a + 0.0` so -0.0 and +0.0 (equal under the
reference's ==) hash alike.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import impls  # noqa: E402
import cases  # noqa: E402


from cases import domain_digest, h, map_digest, partition_digest, run_digest  # noqa: E402


def main():
    R = impls.reference()
    out = {"kat": {}, "domains": {}, "partitions": {}, "maps": {}, "runs": {}}
    arrays = {}
    # ---- lattice / boundary known answers (test_lattice.cpp, test_boundary.cpp)
    out["kat"]["eq_rest"] = R.equilibrium(1.0, [0, 0, 0]).tolist()
    out["kat"]["eq_01"] = R.equilibrium(1.0, [0.1, 0.0, 0.0]).tolist()
    rng = np.random.default_rng(20240811)
    F = rng.uniform(0.01, 1.0, size=(64, 19))
    arrays["kat_f"] = F
    arrays["kat_collide_08"] = np.stack([R.bgk_collide(f, 0.8) for f in F])
    arrays["kat_moments"] = np.stack([np.r_[R.moments(f)[0], R.moments(f)[1]] for f in F])
    st = rng.uniform(0.5, 2.0, size=(64, 1))
    su = rng.uniform(-0.0577, 0.0577, size=(64, 3))
    arrays["kat_eq_in"] = np.hstack([st, su])
    arrays["kat_eq"] = np.stack([R.equilibrium(r[0], r[1:]) for r in arrays["kat_eq_in"]])
    tt = {}
    for name, tab in cases.TABLES.items():
        ts = np.linspace(-0.3, 2.7, 61)
        tt[name] = [R.TimeTable(tab[0], tab[1]).at(float(t)) for t in ts]
    out["kat"]["tables"] = tt
    io = R.Iolet(0, [0.375, 0.5, -0.5], [0.0, 0.0, 1.0], 8.0)
    out["kat"]["weights"] = [R.iolet_weight(io, c) for c in cases.WEIGHT_COORDS]

    # ---- domains, partitions, maps, runs
    for name, spec in cases.DOMAINS.items():
        d = cases.make_domain(R, spec)
        out["domains"][name] = domain_digest(d)
        for W in cases.PARTITION_WORKERS.get(name, []):
            out["partitions"][f"{name}/W{W}"] = partition_digest(R.partition(d, W))
    for key, run in cases.MAP_CASES.items():
        d = cases.make_domain(R, cases.DOMAINS[run["domain"]])
        s = R.Simulation(d, cases.make_bcs(R, run["bcs"]), R.EngineParams(workers=run["W"], layout=run["layout"]))
        out["maps"][key] = [map_digest(s.map(w)) for w in range(run["W"])]
    for key, run in cases.RUNS.items():
        res = cases.execute_run(R, run)
        out["runs"][key] = run_digest(res)
        if res["snapshot"].size <= 20000:
            arrays[f"run_{key}_snapshot"] = res["snapshot"]
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    print("wrote", len(out["domains"]), "domains,", len(out["partitions"]), "partitions,",
          len(out["maps"]), "maps,", len(out["runs"]), "runs")


if __name__ == "__main__":
    main()
