# 4-GPU session: multi-GPU tests, C3 strong scaling (developed), small slabs, C5, C4 weak scaling
mkdir -p gpurun_out/multi
nvidia-smi topo -m > gpurun_out/multi/topo.txt 2>&1
timeout 1500 python -m pytest tests/test_dist.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider \
  -k "dist or nccl or dead or eight or multi or p2p" > gpurun_out/multi/pytest_multi.log 2>&1
echo "pytest rc=$?" >> gpurun_out/multi/pytest_multi.log
for n in 2 4; do
  timeout 900 python bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/multi/bench_c3_n$n.log 2>&1
done
# small slabs: C3 at half length (5.4e7 sites, 1.35e7 per GPU at N=4), N=1 and N=4
for n in 1 4; do
  timeout 900 python bench.py --gpus $n --steps 50 --warmup 5 --scale 0.5 --quick > gpurun_out/multi/bench_c3half_n$n.log 2>&1
done
timeout 1200 python bench.py --gpus 4 --workload c5 --steps 20 --warmup 5 --quick > gpurun_out/multi/bench_c5_n4.log 2>&1
for n in 1 2 4; do
  timeout 1200 python bench.py --gpus $n --workload c4w --steps 20 --warmup 5 --develop 1000 --quick > gpurun_out/multi/bench_c4w_n$n.log 2>&1
done
