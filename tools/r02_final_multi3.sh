# final 4-GPU session with the dynamic-order bulk kernel
mkdir -p gpurun_out/fm3
timeout 1800 python -m pytest tests/test_dist.py tests/test_gpu_parity.py tests/test_bench_geometries.py -m gpu -q -p no:cacheprovider \
  -k "dist or nccl or dead or eight or multi or p2p or store_set or bench_geom or c3_tree or c4_channel or c5_tree" > gpurun_out/fm3/pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/fm3/pytest.log
for n in 4 2; do
  timeout 900 python bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/fm3/bench_c3_n$n.log 2>&1
done
timeout 900 python bench.py --gpus 4 --steps 50 --warmup 5 --scale 0.5 --quick > gpurun_out/fm3/bench_c3half_n4.log 2>&1
timeout 900 python bench.py --gpus 1 --steps 50 --warmup 5 --scale 0.5 --quick > gpurun_out/fm3/bench_c3half_n1.log 2>&1
timeout 1200 python bench.py --gpus 4 --workload c5 --steps 20 --warmup 5 --quick > gpurun_out/fm3/bench_c5_n4.log 2>&1
for n in 1 2 4; do
  timeout 1200 python bench.py --gpus $n --workload c4w --steps 20 --warmup 5 --develop 1000 --quick > gpurun_out/fm3/bench_c4w_n$n.log 2>&1
done
