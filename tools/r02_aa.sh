mkdir -p gpurun_out/aa
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "aa or partition or online or pull or eight" > gpurun_out/aa/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/aa/pytest.log
python tools/aa_split.py --workload c3 > gpurun_out/aa/split_c3.json 2>&1
SPLBCU_PLAIN_VARIANT=64 python tools/aa_split.py --workload c3 > gpurun_out/aa/split_c3_v64.json 2>&1
python tools/aa_split.py --workload c2 > gpurun_out/aa/split_c2.json 2>&1
/usr/local/cuda/bin/ncu --nvtx --nvtx-include "target/" -k regex:lbm_aa_odd_async --launch-count 1 --set full --import-source on \
  --clock-control none -o gpurun_out/aa/c3_dev_aa_async -f python tools/prof_target.py --workload c3 --storage aa --steps 2 > gpurun_out/aa/ncu.log 2>&1
