# dist: series reduction on its own stream beside the next run (default) vs before it (SPLBCU_SERIES_SIDE_OFF)
mkdir -p gpurun_out/side4
timeout 1500 python -m pytest tests/test_dist.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider \
  -k "dist or nccl or dead or eight or multi or p2p or store_set" > gpurun_out/side4/pytest_multi.log 2>&1
echo "pytest rc=$?" >> gpurun_out/side4/pytest_multi.log
for i in 1 2; do
  timeout 900 python bench.py --gpus 4 > gpurun_out/side4/side_n4_$i.log 2>&1
  SPLBCU_SERIES_SIDE_OFF=1 timeout 900 python bench.py --gpus 4 > gpurun_out/side4/off_n4_$i.log 2>&1
done
timeout 900 python bench.py --gpus 2 > gpurun_out/side4/side_n2.log 2>&1
