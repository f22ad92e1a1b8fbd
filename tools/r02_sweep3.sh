mkdir -p gpurun_out/sweep3
for c in 6750000 13500000 27000000; do
  SPLBCU_BULK_CHUNK=$c timeout 900 python profiles/sweep_variants.py --workload c3 --variants 43,59 --pre 3000 --steps 20 | sed "s/^/{\"chunk\": $c, \"r\": /; s/$/}/" >> gpurun_out/sweep3/chunk_dev_c3.jsonl 2>&1
done
SPLBCU_LIB=$PWD/paper_2202_11770_b200/libsplbcu_tuning.so timeout 900 python profiles/sweep_variants.py --workload c3 --variants 52,53,54,43 --pre 3000 --steps 20 > gpurun_out/sweep3/hints_dev_c3.jsonl 2>&1
