mkdir -p gpurun_out/e2e2
for rep in 1 2; do
  timeout 900 python bench.py --gpus 4 --steps 20 --warmup 5 --no-secondary > gpurun_out/e2e2/n4_overlap_$rep.log 2>&1
  SPLBCU_SERIES_FIRST=1 timeout 900 python bench.py --gpus 4 --steps 20 --warmup 5 --no-secondary > gpurun_out/e2e2/n4_first_$rep.log 2>&1
done
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 --no-secondary --no-cpu > gpurun_out/e2e2/n1_overlap.log 2>&1
SPLBCU_SERIES_FIRST=1 timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 --no-secondary --no-cpu > gpurun_out/e2e2/n1_first.log 2>&1
