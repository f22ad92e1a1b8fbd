# Part-size sweep of the bulk range (SPLBCU_BULK_CHUNK) on C3, both bulk kernels
mkdir -p gpurun_out
for C in 13500000 9000000 6750000 4500000; do
  SPLBCU_BULK_CHUNK=$C timeout 300 python profiles/sweep_variants.py --workload c3 --variants 43,59 --steps 20 --warmup 3 2>&1 | grep '^{' | sed "s/^{/{\"chunk\": $C, /" >> gpurun_out/chunk_sweep2.log
done
echo done >> gpurun_out/chunk_sweep2.log
