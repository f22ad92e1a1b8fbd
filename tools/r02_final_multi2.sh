# final 4-GPU check: every multi-GPU test with the final build, bench N=4 and N=2
mkdir -p gpurun_out/fmulti2
timeout 1800 python -m pytest tests/test_dist.py tests/test_gpu_parity.py tests/test_bench_geometries.py -m gpu -q -p no:cacheprovider \
  > gpurun_out/fmulti2/pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/fmulti2/pytest.log
for n in 4 2; do
  timeout 900 python bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/fmulti2/bench_c3_n$n.log 2>&1
done
