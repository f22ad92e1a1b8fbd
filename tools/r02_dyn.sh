mkdir -p gpurun_out/dyn
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_full_size.py -m gpu -q -p no:cacheprovider -k "variants or chunked or c3_full" > gpurun_out/dyn/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/dyn/pytest.log
for c in 0 13500000 6750000; do
  SPLBCU_BULK_CHUNK=$c timeout 900 python profiles/sweep_variants.py --workload c3 --variants 76,43 --pre 3000 --steps 20 | sed "s/^/{\"chunk\": $c, \"r\": /; s/$/}/" >> gpurun_out/dyn/dev_c3.jsonl 2>&1
done
for c in 0 6750000; do
  SPLBCU_BULK_CHUNK=$c timeout 900 python profiles/sweep_variants.py --workload c3 --variants 76,43 --steps 20 | sed "s/^/{\"chunk\": $c, \"r\": /; s/$/}/" >> gpurun_out/dyn/rest_c3.jsonl 2>&1
done
