# AA split timing + ncu captures in a developed flow (C3): push bulk part, AA even/odd
mkdir -p gpurun_out/prof
python tools/aa_split.py --workload c3 > gpurun_out/prof/aa_split_c3.json 2>&1
python tools/aa_split.py --workload c3 --storage two > gpurun_out/prof/two_split_c3.json 2>&1
python tools/aa_split.py --workload c2 > gpurun_out/prof/aa_split_c2.json 2>&1
NCU=/usr/local/cuda/bin/ncu
$NCU --nvtx --nvtx-include "target/" -k regex:lbm_push_tmc --launch-count 1 --set full --import-source on \
  --clock-control none -o gpurun_out/prof/c3_dev_push -f python tools/prof_target.py --workload c3 > gpurun_out/prof/ncu_push.log 2>&1
$NCU --nvtx --nvtx-include "target/" -k regex:lbm_aa --launch-count 4 --set full --import-source on \
  --clock-control none -o gpurun_out/prof/c3_dev_aa -f python tools/prof_target.py --workload c3 --storage aa --steps 2 > gpurun_out/prof/ncu_aa.log 2>&1
$NCU --nvtx --nvtx-include "target/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/prof/c3_dev_launches.csv python tools/prof_target.py --workload c3 --steps 2 > gpurun_out/prof/ncu_launches.log 2>&1
