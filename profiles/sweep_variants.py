#!/usr/bin/env python3
"""Tuning sweep of the plain-kernel launch variants (SPLBCU_PLAIN_VARIANT).

  python profiles/sweep_variants.py --workload c3 --variants 0,43,49 [--steps 20]

One domain per workload, one engine per variant (the engine reads the
variable at construction), kernel-only MSUPS and the bulk kernel's CUDA-event
roofline fraction, one JSON line per (workload, variant).  Tuning evidence
only: bench.py's line is the measured number.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_2202_11770_b200 as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c3")
    ap.add_argument("--variants", default="0")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--tree", default=None, help="R0,L0,levels: a C3-style tree of another size (workload 'tree')")
    ap.add_argument("--pre", type=int, default=0, help="untimed steps before warm-up (developed flow)")
    args = ap.parse_args()
    for name in args.workload.split(","):
        if name == "tree":
            r0, l0, lv = (int(x) for x in args.tree.split(","))
            d = P.build_tree(r0, l0, lv, 0.8, 0.8)
            ents = [P.BCEntry(P.PRESSURE, P.TimeTable.constant(bench.CS2 * 1.001))]
            ents += [P.BCEntry(P.PRESSURE, P.TimeTable.constant(bench.CS2 * 0.999)) for _ in range(2 ** lv)]
            bcs, p = P.BCSet(ents), dict(tau=0.8, dt_s=1.0)
        else:
            d, bcs, p, desc = bench.workload(P, name, args.scale)
        for v in args.variants.split(","):
            os.environ["SPLBCU_PLAIN_VARIANT"] = v
            sim = P.Simulation(d, bcs, P.EngineParams(workers=1, devices=[0], **p))
            sim_n = sim.n_sites()
            if args.pre:
                sim.run(args.pre)
            val, dev_s, launches, roof, clk = bench.timed_loop(sim, sim.n_sites(), args.steps, args.warmup,
                                                               bench.DESIGN_BYTES_PER_SITE, lambda: None,
                                                               lambda x: x, 0, name)
            sim.close()
            print(json.dumps({"workload": name, "scale": args.scale, "sites": sim_n, "variant": int(v), "pre": args.pre, "value": round(val, 1),
                              "frac": roof["frac"], "avg_launch_ms": roof["avg_launch_ms"],
                              "clocks": clk.summary()}), flush=True)


if __name__ == "__main__":
    main()
