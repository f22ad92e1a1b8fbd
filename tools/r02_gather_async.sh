# fused-P2P dist: observation all-gather + series behind the next run (default) vs before it (SPLBCU_GATHER_SYNC)
mkdir -p gpurun_out/gasync
timeout 1500 python -m pytest tests/test_dist.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider \
  -k "dist or nccl or dead or eight or multi or p2p or store_set" > gpurun_out/gasync/pytest_multi.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gasync/pytest_multi.log
for i in 1 2; do
  timeout 900 python bench.py --gpus 4 --no-cpu > gpurun_out/gasync/async_n4_$i.log 2>&1
  SPLBCU_GATHER_SYNC=1 timeout 900 python bench.py --gpus 4 --no-cpu > gpurun_out/gasync/sync_n4_$i.log 2>&1
done
timeout 900 python bench.py --gpus 2 --no-cpu > gpurun_out/gasync/async_n2.log 2>&1
