# 4-GPU session on the AA-default state: multi-GPU tests, C5 and C4 weak with AA storage
mkdir -p gpurun_out/fmulti2
timeout 1500 python -m pytest tests/test_dist.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider \
  -k "dist or nccl or dead or eight or multi or p2p or store_set" > gpurun_out/fmulti2/pytest_multi.log 2>&1
echo "pytest rc=$?" >> gpurun_out/fmulti2/pytest_multi.log
timeout 1200 python bench.py --gpus 4 --workload c5 --steps 20 --warmup 5 --quick > gpurun_out/fmulti2/bench_c5_n4_aa.log 2>&1
for n in 1 4; do
  timeout 1200 python bench.py --gpus $n --workload c4w --steps 20 --warmup 5 --develop 1000 --quick > gpurun_out/fmulti2/bench_c4w_n${n}_aa.log 2>&1
done
