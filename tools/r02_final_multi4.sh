mkdir -p gpurun_out/fm4
timeout 1800 python -m pytest tests/test_dist.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider \
  -k "dist or nccl or dead or eight or multi or p2p or store_set or aa" > gpurun_out/fm4/pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/fm4/pytest.log
timeout 900 python bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/fm4/bench_c3_n4.log 2>&1
timeout 900 python bench.py --gpus 4 --steps 20 --warmup 5 --storage aa --quick > gpurun_out/fm4/bench_c3_n4_aa.log 2>&1
