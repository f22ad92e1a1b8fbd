mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "chunked" > gpurun_out/t6.log 2>&1; echo rc=$? >> gpurun_out/t6.log
for C in 0 27000000 13500000 54000000; do
  SPLBCU_BULK_CHUNK=$C timeout 300 python profiles/sweep_variants.py --workload c3 --variants 43,59 --steps 20 --warmup 3 2>&1 | grep '^{' | sed "s/^{/{\"chunk\": $C, /" >> gpurun_out/chunk_sweep.log
done
echo done >> gpurun_out/chunk_sweep.log
