mkdir -p gpurun_out/aaprof
/usr/local/cuda/bin/ncu --nvtx --nvtx-include "target/" -k regex:lbm_aa --launch-count 4 --set full --import-source on \
  --clock-control none -o gpurun_out/aaprof/c3_dev_aa_final -f python tools/prof_target.py --workload c3 --storage aa --steps 2 > gpurun_out/aaprof/ncu.log 2>&1
