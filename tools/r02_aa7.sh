mkdir -p gpurun_out/aa7
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_full_size.py -m gpu -q -p no:cacheprovider -k "aa or AA" > gpurun_out/aa7/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/aa7/pytest.log
for v in 0 92 0 92; do
  SPLBCU_PLAIN_VARIANT=$v timeout 300 python tools/aa_split.py --workload c3 | sed "s/^/{\"variant\": $v, \"r\": /; s/$/}/" >> gpurun_out/aa7/split_c3.jsonl 2>&1
done
timeout 300 python tools/aa_split.py --workload c2 | sed "s/^/{\"variant\": 0, \"r\": /; s/$/}/" >> gpurun_out/aa7/split_c2.jsonl 2>&1
/usr/local/cuda/bin/ncu --nvtx --nvtx-include "target/" -k regex:lbm_aa_odd_w --launch-count 1 --set full --import-source on \
  --clock-control none -o gpurun_out/aa7/c3_dev_aa_raw -f python tools/prof_target.py --workload c3 --storage aa --steps 2 > gpurun_out/aa7/ncu.log 2>&1
