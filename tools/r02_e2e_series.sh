# N=1 series reduction on the edge stream vs behind the steps (SPLBCU_SERIES_ON_MAIN)
mkdir -p gpurun_out/e2es
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/e2es/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/e2es/pytest_gpu.log
for i in 1 2; do
  timeout 900 python bench.py --no-cpu --no-secondary > gpurun_out/e2es/side_$i.log 2>&1
  SPLBCU_SERIES_ON_MAIN=1 timeout 900 python bench.py --no-cpu --no-secondary > gpurun_out/e2es/main_$i.log 2>&1
done
