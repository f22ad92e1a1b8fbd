mkdir -p gpurun_out/dbg
timeout 900 python tools/debug_aa_c4.py > gpurun_out/dbg/aa_c4.log 2>&1
timeout 900 python tools/e2e_ab.py --workload c3 > gpurun_out/dbg/e2e_ab_c3.jsonl 2>&1
timeout 600 python tools/e2e_ab.py --workload c2 > gpurun_out/dbg/e2e_ab_c2.jsonl 2>&1
