mkdir -p gpurun_out/sweep4
for c in 3375000 4500000 6750000 9000000 13500000 6750000; do
  SPLBCU_BULK_CHUNK=$c timeout 900 python profiles/sweep_variants.py --workload c3 --variants 43,59,24 --pre 3000 --steps 20 | sed "s/^/{\"chunk\": $c, \"r\": /; s/$/}/" >> gpurun_out/sweep4/chunk_dev_c3.jsonl 2>&1
done
for c in 4500000 6750000 13500000; do
  SPLBCU_BULK_CHUNK=$c timeout 900 python profiles/sweep_variants.py --workload c3 --variants 43,59 --steps 20 | sed "s/^/{\"chunk\": $c, \"r\": /; s/$/}/" >> gpurun_out/sweep4/chunk_rest_c3.jsonl 2>&1
  SPLBCU_BULK_CHUNK=$c timeout 900 python profiles/sweep_variants.py --workload c2,c4 --variants 43,71 --pre 3000 --steps 20 | sed "s/^/{\"chunk\": $c, \"r\": /; s/$/}/" >> gpurun_out/sweep4/chunk_dev_c2c4.jsonl 2>&1
done
