mkdir -p gpurun_out/aa3
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "aa_odd or store_set or eight" > gpurun_out/aa3/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/aa3/pytest.log
for v in 0 80 0 80; do
  SPLBCU_PLAIN_VARIANT=$v python tools/aa_split.py --workload c3 | sed "s/^/{\"variant\": $v, \"r\": /; s/$/}/" >> gpurun_out/aa3/split_c3.jsonl 2>&1
done
timeout 600 python bench.py --workload c3 --storage aa --steps 20 --warmup 5 --quick > gpurun_out/aa3/aa_c3.log 2>&1
