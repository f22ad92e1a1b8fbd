"""Small engine runs for compute-sanitizer (memcheck / racecheck / synccheck):
  smoke  3 workers, push, peer-copy halo (the __graft_entry__.smoke case)
  p2p3   3 workers, fused NVLink-P2P halo stores, flag-ordered
  aa3    3 workers, AA single buffer updated in place (odd steps gather/scatter
         across workers)
  pull3  3 workers, pull scheme (update_pull + fill_send_slots)
Each is checked bit-exactly against the golden digests of the reference.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import json  # noqa: E402

import cases  # noqa: E402
import impls  # noqa: E402

golden = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))
P = impls.product()
key = "bif_W3_soa_reordered"
kw = {"smoke": {}, "p2p3": dict(halo_mode=1), "aa3": dict(storage=1), "pull3": dict(halo_mode=1)}[sys.argv[1]]
run = dict(cases.RUNS[key])
if sys.argv[1] == "pull3":
    run["scheme"] = 1
res = cases.execute_run(P, run, devices=[0], **kw)
ok = cases.run_digest(res) == golden["runs"][key]
res["sim"].close()
print(sys.argv[1], "bit-exact" if ok else "MISMATCH")
sys.exit(0 if ok else 1)
