mkdir -p gpurun_out/aa12
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "aa_odd" > gpurun_out/aa12/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/aa12/pytest.log
for v in 0 105 106 0 105 106; do
  SPLBCU_PLAIN_VARIANT=$v timeout 300 python tools/aa_split.py --workload c3 | sed "s/^/{\"variant\": $v, \"r\": /; s/$/}/" >> gpurun_out/aa12/split_c3.jsonl 2>&1
done
