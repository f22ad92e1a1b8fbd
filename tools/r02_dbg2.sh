mkdir -p gpurun_out/dbg2
timeout 600 python tools/debug_aa_c4b.py 48 40 120 > gpurun_out/dbg2/aa_c4.log 2>&1
timeout 600 python tools/debug_aa_c4b.py 16 12 30 > gpurun_out/dbg2/aa_c4_small.log 2>&1
