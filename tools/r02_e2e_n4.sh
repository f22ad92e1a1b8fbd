mkdir -p gpurun_out/e2en4
for rep in 1 2; do
  timeout 900 python bench.py --gpus 4 --steps 20 --warmup 5 --no-secondary > gpurun_out/e2en4/series_first_$rep.log 2>&1
  SPLBCU_NO_SERIES_FIRST=1 timeout 900 python bench.py --gpus 4 --steps 20 --warmup 5 --no-secondary > gpurun_out/e2en4/overlap_$rep.log 2>&1
done
