mkdir -p gpurun_out/aaprof2
for v in 88 89; do
SPLBCU_PLAIN_VARIANT=$v /usr/local/cuda/bin/ncu --nvtx --nvtx-include "target/" -k regex:lbm_aa_odd_s --launch-count 1 --set full --import-source on \
  --clock-control none -o gpurun_out/aaprof2/c3_dev_aa_s$v -f python tools/prof_target.py --workload c3 --storage aa --steps 2 > gpurun_out/aaprof2/ncu$v.log 2>&1
done
