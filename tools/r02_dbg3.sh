mkdir -p gpurun_out/dbg3
timeout 300 python tools/debug_aa_c4c.py default > gpurun_out/dbg3/default.log 2>&1
SPLBCU_SYNC_RUN=1 timeout 300 python tools/debug_aa_c4c.py syncrun > gpurun_out/dbg3/syncrun.log 2>&1
CUDA_LAUNCH_BLOCKING=1 timeout 600 python tools/debug_aa_c4c.py blocking > gpurun_out/dbg3/blocking.log 2>&1
