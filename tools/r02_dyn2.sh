mkdir -p gpurun_out/dyn2
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "variants or chunked or online" > gpurun_out/dyn2/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/dyn2/pytest.log
timeout 1200 python profiles/sweep_variants.py --workload c3,c2 --variants 77,71,0 --pre 3000 --steps 20 > gpurun_out/dyn2/dev_run.jsonl 2>&1
for v in 0 78; do
  SPLBCU_PLAIN_VARIANT=$v python tools/aa_split.py --workload c3 | sed "s/^/{\"variant\": $v, \"r\": /; s/$/}/" >> gpurun_out/dyn2/aa_split_c3.jsonl 2>&1
done
