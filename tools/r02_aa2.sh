mkdir -p gpurun_out/aa2
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "aa_odd or eight or store_set" > gpurun_out/aa2/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/aa2/pytest.log
for v in 0 72 73; do
  SPLBCU_PLAIN_VARIANT=$v python tools/aa_split.py --workload c3 | sed "s/^/{\"variant\": $v, \"r\": /; s/$/}/" >> gpurun_out/aa2/split_c3.jsonl 2>&1
done
for v in 0 73; do
  SPLBCU_PLAIN_VARIANT=$v python tools/aa_split.py --workload c2 | sed "s/^/{\"variant\": $v, \"r\": /; s/$/}/" >> gpurun_out/aa2/split_c2.jsonl 2>&1
done
